"""Summarise ncu captures of book_kernel into profiles/ncu_summary.json (dev tool).

  python tools/ncu_summary.py TAG W1:rep1:benchlog1 [W2:rep2:benchlog2 ...]

Each capture is `ncu --set full -k regex:book_kernel -s 3 -c 1 ... python
bench.py --workload W ...`; the bench line printed by that (profiled, so
slow) run gives the messages of one step exactly (value x ms_per_step),
which turns ncu's per-launch counters into per-message figures.  bench.py
reads the entry of its workload (inst_per_msg -> the issue-rate roofline,
dram_bytes_per_msg -> roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STALLS = ["wait", "long_scoreboard", "short_scoreboard", "barrier", "not_selected", "no_instruction",
          "branch_resolving", "math_pipe_throttle", "mio_throttle", "lg_throttle", "dispatch_stall"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1, "msecond": 1, "s": 1e3, "second": 1e3, "nsecond": 1e-6}


def main():
    tag = sys.argv[1]
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        summary = json.load(open(path))
    except Exception:
        summary = {}
    summary.setdefault("workloads", {})
    for spec in sys.argv[2:]:
        w, rep, log = spec.split(":")
        d, units = raw(rep)
        line = next(json.loads(x) for x in open(log) if x.startswith("{"))
        msgs = line["value"] * line["ms_per_step"] / 1e3
        f = lambda k: float(d[k]) * SCALE.get(units.get(k, ""), 1)  # noqa: E731
        inst = f("smsp__inst_executed.sum")
        dram = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
        e = {
            "kernel": d.get("Kernel Name") or d.get("Function Name"),
            "capture": f"ncu --set full --clock-control none --import-source on -k regex:book_kernel -s 3 -c 1 "
                       f"python bench.py --workload {w} --steps 2 --warmup 3 --no-cpu --no-extra ({tag})",
            "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
            "registers_per_thread": d.get("launch__registers_per_thread"),
            "msgs_per_launch": msgs,
            "duration_ms_ncu": f("gpu__time_duration.sum"),
            "inst_executed": inst,
            "inst_per_msg": inst / msgs,
            "dram_bytes_read": f("dram__bytes_read.sum"), "dram_bytes_write": f("dram__bytes_write.sum"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "stalls_per_issue": {s: round(f(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"), 3)
                                 for s in STALLS
                                 if f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" in d},
        }
        e["dram_bytes_per_msg"] = dram / msgs
        summary["workloads"][w] = e
        print(w, json.dumps({k: e[k] for k in ("inst_per_msg", "dram_bytes_per_msg", "issue_active_pct",
                                                 "warps_active_pct", "duration_ms_ncu")}))
    json.dump(summary, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
