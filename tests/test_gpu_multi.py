"""Multi-GPU parity (P = 2 or 4 ranks, NCCL A2A + chunked AR) against the oracle's
P simulated workers.  Needs >= 2 GPUs (gpurun --gpus 2|4)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"c1_f32": 1e-4, "c1_f32_p2p": 1e-4, "bf16_p": 2e-2}  # other bf16_p_* variants: bf16 tol


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("P", [2, 4])
def test_multi_gpu_parity(P):
    if _ngpus() < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + P),
           os.path.join(ROOT, "tests", "mp_parity_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("MP_RESULTS ")]
    assert line, out.stdout[-3000:]
    per_rank = json.loads(line[0][len("MP_RESULTS "):])
    for rank, res in enumerate(per_rank):
        for case, r in res.items():
            if case.startswith("sched_"):  # measured schedule properties
                v = dict(r["violations"])
                if case == "sched_nccl":  # NCCL kernels of the A2A and AR communicators share
                    v.pop("priority", None)  # the copy engines / SMs: reported, not asserted
                if v:
                    pytest.fail(f"rank {rank} {case}: {json.dumps(r)}")
                for prop in ("eq3", "eq4", "eq5", "eq6", "6a", "6c", "6e", "priority"):
                    assert r["checked"].get(prop, 0) > 0, (rank, case, prop, r["checked"])
                continue
            if case.startswith("stack_"):  # 3-block chain, checked block by block
                assert r.pop("stack_bitwise"), (rank, case)
                tol = 1e-4 if "f32" in case else 2e-2
            else:
                assert r.pop("routing_exact"), (rank, case)
                tol = TOL.get(case, TOL["bf16_p"])
            bad = {k: v for k, v in r.items() if not v <= tol}
            assert not bad, (rank, case, bad)
