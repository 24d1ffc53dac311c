"""Summarise one-kernel ncu captures (.ncu-rep) into a JSON object per report:
python scripts/ncu_summarize.py TASKS gpurun_out/prof_pair.ncu-rep [...]
(TASKS = tasks per launch, for instructions per task)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu_time_ns": "gpu__time_duration.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
}
STALL = "smsp__pcsamp_warps_issue_stalled_"


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def summarize(rep, tasks):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = dict(zip(head, vals))
    unit = dict(zip(head, units))
    r = {"report": rep}
    for k, m in KEYS.items():
        if m in col:
            v = num(col[m])
            u = unit.get(m, "")
            if v is not None and k == "gpu_time_ns":
                v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)
            if v is not None and k.startswith("dram_bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
            r[k] = v
    if r.get("inst_executed"):
        r["instructions_per_task"] = r["inst_executed"] / tasks
    st = {h[len(STALL):]: num(col[h]) for h in head
          if h.startswith(STALL) and not h.endswith("_not_issued") and num(col[h])}
    tot = sum(st.values()) or 1.0
    r["stall_top"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:7]}
    return r


if __name__ == "__main__":
    tasks = float(sys.argv[1])
    print(json.dumps([summarize(p, tasks) for p in sys.argv[2:]], indent=1))
