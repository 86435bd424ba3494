"""Summarise an ncu --set full report of the step kernel (run here, no GPU):
    python tools/ncu_summary.py gpurun_out/prof_tc.ncu-rep [--top 25] [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    recs, units = raw(path)
    summary = []
    for rec in recs:
        d = {"kernel": rec.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in rec:
                d[k] = rec[k]
                print(f"{k:70s} {units.get(k, ''):>10s} {rec[k]}")
        stalls = {k: float(v) for k, v in rec.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")}
        for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
            print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v:.3f}")
        d["stalls"] = stalls
        summary.append(d)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        hdr = rows[1]
        data = rows[2:]
        iss, iex, isrc = (hdr.index("Warp Stall Sampling (All Samples)"),
                          hdr.index("Instructions Executed"), hdr.index("Source"))
        tot = sum(float(r[iss] or 0) for r in data) or 1
        print(f"total stall samples {tot:.0f}, warp instructions {sum(float(r[iex] or 0) for r in data):.0f}")
        for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:top]:
            print(f"  {float(r[iss]) / tot * 100:5.1f}%  {r[iex]:>9s}  {r[isrc][:80]}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
