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


def test_kernel_groups_and_transfer_only_exposure(tmp_path):
    """Per-group busy time is the union of the group's intervals (overlapping lanes count
    once), the sum counts every launch; a peer-memory exchange kernel is counted as
    communication only over its transfer time (bytes / link bandwidth) in the
    transfer-only exposure — its tail is a wait for the peers."""
    ev = [
        {"cat": "kernel", "name": "void fm::gemm_tc_kernel<256, 4, 1>(fm::TcParams)", "ts": 0, "dur": 10},
        {"cat": "kernel", "name": "void fm::gemm_tc_kernel<128, 6, 1>(fm::TcParams)", "ts": 5, "dur": 10},  # overlaps
        {"cat": "kernel", "name": "void fm::gate_topk_kernel<__nv_bfloat16, 16>(...)", "ts": 20, "dur": 2},
        # exchange kernel 20 us long, but 770 GB/s moves 7700 B in 10 ns... use 7.7 MB -> 10 us
        {"cat": "kernel", "name": "void fm::a2a_p2p_send_wait_kernel(fm::P2PArgs)", "ts": 30, "dur": 20},
    ]
    p = tmp_path / "t.json"
    p.write_text(json.dumps({"traceEvents": ev}))
    r = analyze(str(p), 1, a2a_bytes=7.7e6, link_gbs=770.0)
    g = r["groups"]
    assert g["gemm"]["launches_per_iter"] == 2
    assert g["gemm"]["sum_us_per_iter"] == 20 and g["gemm"]["busy_us_per_iter"] == 15
    assert g["gate_topk"]["busy_us_per_iter"] == 2 and g["a2a"]["busy_us_per_iter"] == 20
    assert r["exposed_comm_us_per_iter"] == 20               # the whole kernel, nothing overlaps it
    assert abs(r["exposed_transfer_us_per_iter"] - 10) < 1e-9  # only the 10 us transfer
    assert abs(r["exposed_transfer_frac_of_transfer"] - 1.0) < 1e-12
