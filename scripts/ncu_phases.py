"""Stall samples / instructions of k_search or k_backup grouped by phase (vp_phases.cuh line ranges).

    python scripts/ncu_phases.py gpurun_out/prof_x.ncu-rep
"""
import csv
import subprocess
import sys

PHASES = [  # (file, first line, last line, phase) -- vp_phases.cuh / vp_common.cuh layout
    ("vp_phases.cuh", 264, 345, "draw: CDF scan / build"),
    ("vp_phases.cuh", 346, 386, "draw: TMA staging"),
    ("vp_phases.cuh", 584, 680, "draw: staging / cache protocol"),
    ("vp_phases.cuh", 385, 408, "group sums"),
    ("vp_phases.cuh", 410, 460, "lazy rows + id alloc"),
    ("vp_phases.cuh", 505, 531, "root draw"),
    ("vp_phases.cuh", 681, 700, "arrive / leaf list"),
    ("vp_phases.cuh", 755, 1000, "search body (claims, stats, creation)"),
    ("vp_phases.cuh", 50, 68, "claims"),
    ("vp_phases.cuh", 70, 126, "backup delivery"),
    ("vp_phases.cuh", 127, 243, "LSE"),
    ("vp_phases.cuh", 994, 1150, "backup body"),
    ("vp_common.cuh", 27, 57, "RNG"),
    ("vp_common.cuh", 58, 180, "hash / atomics"),
    ("vp_models.cuh", 1, 10000, "model step / heuristic"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr = None, None
    agg = {}
    ts = ti = 0
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            i = int(r[hdr.index("Instructions Executed")])
            ln = int(r[0])
        except (ValueError, IndexError):
            continue
        name = next((p for f, a, b, p in PHASES if f == cur and a <= ln <= b), f"other ({cur})")
        x = agg.setdefault(name, [0, 0])
        x[0] += s
        x[1] += i
        ts += s
        ti += i
    print(f"# {path}: {ts} stall samples, {ti} warp instructions")
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{100.0 * s / max(ts, 1):5.1f}% stalls  {100.0 * i / max(ti, 1):5.1f}% inst  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
