"""Summarise an ncu --set full report (.ncu-rep) into the counters DESIGN.md cites.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]

Capture with the pipe counters `--set full` leaves out (tools/gpu_r02.sh):
  ncu --set full --metrics sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fmaheavy.sum,
      sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,
      sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,
      sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg ...
B200 has no XU "cycles active" counter; the XU (MUFU) utilisation is derived: one warp
MUFU instruction occupies its SM sub-partition's 4-lane XU for 8 cycles, i.e. an SM
retires at most 0.5 warp XU instructions per cycle (measured 15.96 lanes/clk/SM,
profiles/r02_pipe_peaks.json), so xu_pct = inst_executed_pipe_xu / SMs / (0.5 x active cycles).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__waves_per_multiprocessor",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_xu.sum", "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_fmaheavy.sum", "sm__inst_executed_pipe_fmalite.sum", "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed_pipe_fp64.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__warps_eligible.avg.per_cycle_active",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kernels.append(d)
    return kernels


def summarise(d):
    s = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
    for k in KEYS:
        if k in d:
            v, u = d[k]
            try:
                v = float(v.replace(",", ""))
            except ValueError:
                pass
            s[k] = v if not u else [v, u]
    stalls = {}
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                fv = float(v)
            except ValueError:
                continue
            if fv > 0.01:
                stalls[h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = fv
    s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    xu, cyc = _num(s.get("sm__inst_executed_pipe_xu.sum")), _num(s.get("sm__cycles_active.avg"))
    if xu is not None and cyc:
        s["derived_xu_pct_of_peak_active"] = 100.0 * xu / SMS / (0.5 * cyc)
    return s


SMS = 148


def _num(v):
    if isinstance(v, list):
        v = v[0]
    return v if isinstance(v, float) else None


if __name__ == "__main__":
    res = [summarise(d) for d in load(sys.argv[1])]
    txt = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt)
    print(txt)
