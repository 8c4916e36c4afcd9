#!/bin/bash
# One compute-sanitizer tool (TOOL=memcheck|racecheck|synccheck) over small GEMM, attention,
# routing and peer-memory (simulated world) unit tests.  One tool per gpurun call
# (B200_PROFILING.md).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/sanitize; mkdir -p $O
T=${TOOL:-memcheck}
SEL='test_gemm_tc_layouts_vs_fp64 and shape0 and (0-0 or 1-1) or test_gemm_tc_epilogues or (test_block_parity_forced_routing and (bf16_small or bf16_ragged or c1_f32)) or (test_token_chunk_parity and tok_bf16_ragged) or (test_routing_crafted_ties and bf16_small) or (test_block_parity_cta_pair_gemms and bf16_small)'
timeout 2400 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$SEL" > $O/$T.log 2>&1
echo "$T parity rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" $O/$T.log | tail -5
if [ "$T" = "memcheck" ] || [ "$T" = "synccheck" ]; then
timeout 1800 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_gpu_group.py -q -p no:cacheprovider -x -k "block_parity and c1_f32 or chunked_allreduce and 4112" > $O/${T}_group.log 2>&1
echo "$T group rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" $O/${T}_group.log | tail -5
fi
