"""Summarise ncu reports into profiles/ (text per capture + ncu_summary.json).

Usage: python tools/ncu_summarize.py <tag> <report.ncu-rep> [<tag> <report> ...]
Writes profiles/<round>_<tag>.txt with the headline metrics of every
captured launch and the top source lines by warp-stall samples, and merges
{tag: {dram_bytes_per_launch, duration_us, ...}} into profiles/ncu_summary.json
(bench.py reads the "find" / "update" / "filter" entries for roofline.traffic).
"""

import collections
import csv
import json
import os
import subprocess
import sys

ROUND = os.environ.get("GS_ROUND", "r01")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "profiles")
SRC_FILES = ",".join(os.path.join(REPO, "paper_1503_08294_b200", "csrc", f)
                     for f in ("update_kernel.cuh", "engine.cu", "common.cuh", "find.cu",
                               "filter.cu", "sample.cu"))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU inst %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle",
          "membar", "not_selected", "dispatch_stall", "branch_resolving", "mio_throttle",
          "lg_throttle", "no_instruction"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
        "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def source_hot(rep, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--resolve-source-file", SRC_FILES],
                         capture_output=True, text=True).stdout
    agg = collections.defaultdict(float)
    src = {}
    cur = None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 5 or r[2] != "-":
            continue
        try:
            key = (cur, int(r[0]))
            agg[key] += float(r[4] or 0)
            src[key] = r[1].strip()
        except ValueError:
            pass
    tot = sum(agg.values()) or 1.0
    return [(k, v / tot * 100, src[k]) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]]


def to_num(v, u):
    try:
        return float(v) * UNIT.get(u, 1.0)
    except (TypeError, ValueError):
        return None


def main():
    args = sys.argv[1:]
    os.makedirs(OUT, exist_ok=True)
    summ_path = os.path.join(OUT, "ncu_summary.json")
    try:
        summary = json.load(open(summ_path))
    except (OSError, ValueError):
        summary = {}
    for tag, rep in zip(args[0::2], args[1::2]):
        launches = raw(rep)
        lines = [f"# ncu --set full: {tag}  (report {os.path.basename(rep)}; {len(launches)} launch(es))",
                 "# cold-cache unless the tag says warm; per-launch values", ""]
        durs, dram = [], []
        for i, (d, u) in enumerate(launches):
            lines.append(f"## launch {i}: {d.get('Kernel Name', '?')[:110]}")
            for k, label in METRICS:
                if k in d:
                    lines.append(f"  {label:28s} {d[k]} {u.get(k, '')}")
            st = []
            for name in STALLS:
                k = f"smsp__average_warps_issue_stalled_{name}_per_issue_active.ratio"
                if k in d:
                    try:
                        st.append((float(d[k]), name))
                    except ValueError:
                        pass
            lines.append("  stalls per issued instruction: " +
                         ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6]))
            durs.append(to_num(d.get("gpu__time_duration.sum"), u.get("gpu__time_duration.sum")))
            r_ = to_num(d.get("dram__bytes_read.sum"), u.get("dram__bytes_read.sum")) or 0.0
            w_ = to_num(d.get("dram__bytes_write.sum"), u.get("dram__bytes_write.sum")) or 0.0
            dram.append(r_ + w_)
            lines.append("")
        lines.append("## hottest source lines (share of warp-stall samples, all launches)")
        for (f, ln), pct, text in source_hot(rep):
            lines.append(f"  {pct:5.1f}%  {f}:{ln}  {text[:90]}")
        with open(os.path.join(OUT, f"{ROUND}_{tag}.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        durs = [x for x in durs if x is not None]
        summary[tag] = {"report": os.path.basename(rep), "launches": len(launches),
                        "duration_us_mean": sum(durs) / len(durs) if durs else None,
                        "dram_bytes_per_launch": sum(dram) / len(dram) if dram else None}
        print(f"{tag}: {len(launches)} launches, mean {summary[tag]['duration_us_mean']} us, "
              f"dram/launch {summary[tag]['dram_bytes_per_launch']}")
    with open(summ_path, "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
