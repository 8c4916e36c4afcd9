"""Interval arithmetic of the exposed-communication metric (no GPU)."""
import json

from paper_2510_00207_b200.timeline import analyze


def test_exposed_comm_interval_math(tmp_path):
    ev = [
        {"cat": "kernel", "name": "gemm_tc_kernel<256, 4>", "ts": 0, "dur": 10},
        {"cat": "kernel", "name": "ncclDevKernel_SendRecv", "ts": 5, "dur": 10},    # 5 exposed (10..15)
        {"cat": "kernel", "name": "attn_fwd_tc_kernel<64>", "ts": 20, "dur": 10},
        {"cat": "kernel", "name": "ncclDevKernel_AllReduce", "ts": 22, "dur": 4},   # hidden
        {"cat": "kernel", "name": "ncclDevKernel_AllReduce", "ts": 35, "dur": 5},   # 5 exposed
    ]
    p = tmp_path / "t.json"
    p.write_text(json.dumps({"traceEvents": ev}))
    r = analyze(str(p), 1)
    assert r["comm_busy_us_per_iter"] == 19
    assert r["exposed_comm_us_per_iter"] == 10
    assert abs(r["exposed_comm_frac_of_comm"] - 10 / 19) < 1e-12
    assert r["span_us_per_iter"] == 40
    assert r["idle_us_per_iter"] == 40 - 30
