"""world_size-2 gloo tests on CPU for the multi-process host logic: the expert-
parallel A2A data layout the library implements with NCCL send/recv
([E][C][M] owner side <-> [E/P][P][C][M] expert side), checked with real
torch.distributed all_to_all on gloo against the oracle's simulated A2A; and the
bench --impl reference arm under torchrun (rank 0 alone prints)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
import oracle as o
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
E, C, M = 4, 3, 5
El = E // P
sends = [np.arange(E * C * M, dtype=np.float64).reshape(E, C, M) + 1000 * p for p in range(P)]
# dispatch: rows of expert e = q*El + el go to rank q; received as [El][P][C][M]
send = torch.from_numpy(sends[rank]).reshape(P, El * C * M).contiguous()
recv = torch.empty_like(send)
dist.all_to_all_single(recv, send)
expert_side = recv.reshape(P, El, C, M).permute(1, 0, 2, 3).contiguous().numpy()
ref = o.alltoall(sends, P)[rank]            # [P(src)][El][C][M]
ok1 = np.array_equal(expert_side, ref.transpose(1, 0, 2, 3))
# combine: expert side [El][P][C][M] back to owners as [E][C][M]
back_send = torch.from_numpy(expert_side).permute(1, 0, 2, 3).contiguous().reshape(P, El * C * M)
back = torch.empty_like(back_send)
dist.all_to_all_single(back, back_send)
ok2 = np.array_equal(back.reshape(E, C, M).numpy(), sends[rank])
res = [None] * P
dist.all_gather_object(res, bool(ok1 and ok2))
if rank == 0:
    print("GLOO_OK", json.dumps(res))
dist.destroy_process_group()
'''


def _torchrun(script_args, port):
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
            "--master-addr", "127.0.0.1", "--master-port", str(port)] + script_args


def test_a2a_layout_roundtrip_gloo(tmp_path):
    p = tmp_path / "w.py"
    p.write_text(WORKER.format(root=ROOT))
    out = subprocess.run(_torchrun([str(p)], 29710), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("GLOO_OK")]
    assert line and json.loads(line[0].split(" ", 1)[1]) == [True, True]


def test_bench_reference_arm_rank0_only(tmp_path):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run(_torchrun([os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                                    "--steps", "2", "--warmup", "1", "--config", "c1"], 29720),
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
