"""Per-source-line totals (warp instructions executed, stall samples) of an ncu report.

    python scripts/ncu_lines.py gpurun_out/prof_x.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, res = None, []
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue  # only the cuda-source rows (aggregated), sass rows have an address
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        res.append((cur_file, int(r[0]), r[1].strip()[:80], inst, samples))
    ti, ts = sum(x[3] for x in res) or 1, sum(x[4] for x in res) or 1
    print(f"# {path}: {ti} warp instructions, {ts} stall samples (source-line aggregates)")
    print("## by stall samples")
    for f, ln, src, inst, s in sorted(res, key=lambda x: -x[4])[:top]:
        print(f"{100.0 * s / ts:5.1f}%  inst {100.0 * inst / ti:5.1f}%  {f}:{ln}  {src}")
    print("## by instructions")
    for f, ln, src, inst, s in sorted(res, key=lambda x: -x[3])[:top // 2]:
        print(f"inst {100.0 * inst / ti:5.1f}%  {100.0 * s / ts:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
