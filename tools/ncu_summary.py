"""Summarise an `ncu --set full` report of the NTT passes into profiles/ (JSON): per kernel duration,
DRAM bytes, issue activity, pipe utilisation, occupancy and the top warp-stall reasons."""
import csv
import io
import json
import subprocess
import sys


def f(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def summarise(rep, limb_transforms):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    U = {h[i]: scale.get(units[i], 1.0) for i in range(len(h))}
    out = []
    tot_bytes = 0.0
    for r in data:
        d = {h[i]: r[i] for i in range(len(h))}
        ps = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and f(v) is not None and not k.endswith("not_issued")}
        tot = sum(ps.values()) or 1.0
        rd = (f(d.get("dram__bytes_read.sum", "0")) or 0.0) * U.get("dram__bytes_read.sum", 1.0)
        wr = (f(d.get("dram__bytes_write.sum", "0")) or 0.0) * U.get("dram__bytes_write.sum", 1.0)
        tot_bytes += rd + wr
        out.append({
            "kernel": d["Kernel Name"].split("(")[0],
            "duration_us": (f(d.get("gpu__time_duration.sum", "0")) or 0) * U.get("gpu__time_duration.sum", 1e-3),
            "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
            "issue_active_pct": f(d.get("sm__inst_issued.avg.pct_of_peak_sustained_active", "")),
            "pipe_fp64_cycles_pct": f(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "")),
            "inst_pipe_fp64_pct": f(d.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "")),
            "pipe_fma_pct": f(d.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "")),
            "pipe_alu_pct": f(d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "")),
            "warps_active_pct": f(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "")),
            "registers": f(d.get("launch__registers_per_thread", "")),
            "instructions": f(d.get("smsp__inst_executed.sum", "")),
            "top_stalls_pct": {k: round(100 * v / tot, 1) for k, v in sorted(ps.items(), key=lambda x: -x[1])[:6]},
        })
    return {"source": rep, "kernels": out, "dram_bytes_total": tot_bytes,
            "dram_bytes_per_limb_transform": tot_bytes / limb_transforms if limb_transforms else None}


if __name__ == "__main__":
    rep, lt, dst = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    s = summarise(rep, lt)
    json.dump(s, open(dst, "w"), indent=1)
    print(json.dumps(s, indent=1)[:3000])
