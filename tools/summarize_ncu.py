"""Summarise an `ncu --set full` report into a small JSON for profiles/.

usage: python tools/summarize_ncu.py REPORT.ncu-rep OUT.json "capture command" [flops_per_launch]
"""
import csv
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
    # INT8 tcgen05 kernel (Ozaki MTTKRP): tensor / conversion / FP64 pipe activity
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
]


def main():
    rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    flops = float(sys.argv[4]) if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k + (f" [{u[i]}]" if u[i] else "")] = r[i]
        stalls = {x.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): float(r[i])
            for i, x in enumerate(h)
            if x.startswith("smsp__average_warps_issue_stalled") and x.endswith(
                "per_issue_active.ratio") and r[i] and float(r[i]) > 0.2}
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        launches.append(d)

    def mb(d, k):
        for key, v in d.items():
            if key.startswith(k):
                scale = 1e6 if "[Mbyte]" in key else (1e9 if "[Gbyte]" in key else 1e3
                                                        if "[Kbyte]" in key else 1.0)
                return float(v) * scale
        return 0.0

    res = {"capture": cmd, "launches": launches}
    tr = [mb(d, "dram__bytes_read.sum") + mb(d, "dram__bytes_write.sum") for d in launches]
    if tr:
        res["dram_bytes_per_launch"] = sum(tr) / len(tr)
    if flops:
        res["algorithmic_flops_per_launch"] = flops
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))


if __name__ == "__main__":
    main()
