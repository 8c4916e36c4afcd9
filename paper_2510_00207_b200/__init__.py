"""B200-native FlowMoE block hot path (arXiv 2510.00207).

The compute lives in libflowmoe.so (C ABI: include/flowmoe.h, test hooks include/flowmoe_test.h; CUDA sm_100a);
``flowmoe`` is the thin ctypes binding.
"""
from .flowmoe import (BlockShape, BlockTensors, ExpertOpt, FlowMoE, FlowMoEError, Grads, Optimizer,  # noqa: F401
                      Params,
                      get_unique_id, kernel_launches, lib, test_gemm, to_device,
                      to_host_f64, torch_dtype)
