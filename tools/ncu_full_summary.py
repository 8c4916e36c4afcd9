"""Key counters of every kernel in an `ncu --set full` report: duration, DRAM bytes and
throughput, tensor-pipe activity (tcgen05), SM throughput, registers, dynamic smem.
Usage: python tools/ncu_full_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import re
import subprocess
import sys

M = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd_GB": "dram__bytes_read.sum",
    "dram_wr_GB": "dram__bytes_write.sum",
    "dram_rd_TBps": "dram__bytes_read.sum.per_second",
    "tensor_pipe_%": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm_thru_%": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
    "smem_dyn_KB": "launch__shared_mem_per_block_dynamic",
}
SCALE = {"us": 1, "usecond": 1, "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "Gbyte": 1, "Mbyte": 1e-3,
         "Kbyte": 1e-6, "byte": 1e-9, "Tbyte/s": 1, "Gbyte/s": 1e-3, "%": 1, "": 1, "Kbyte/block": 1,
         "byte/block": 1e-3, "register/thread": 1}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"{'kernel':44s} " + " ".join(f"{k:>13s}" for k in M))
    for r in data:
        name = re.sub(r"^void ", "", r[idx["Kernel Name"]])
        name = re.match(r"([\w:]+(?:<[^()]*?>)?)", name).group(1)[:44]
        vals = []
        for k, m in M.items():
            if m not in idx:
                vals.append("n/a")
                continue
            v = r[idx[m]].replace(",", "")
            try:
                vals.append(f"{float(v) * SCALE.get(units[idx[m]], 1):.4g}")
            except ValueError:
                vals.append(v)
        print(f"{name:44s} " + " ".join(f"{v:>13s}" for v in vals))


if __name__ == "__main__":
    main(sys.argv[1])
