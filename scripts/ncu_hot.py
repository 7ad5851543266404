"""Hot SASS instructions of an ncu --set full report (stall samples), with source lines.

    python scripts/ncu_hot.py gpurun_out/prof_x.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    iSrc, iA = hdr.index("Source"), hdr.index("Address")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[iS]), int(r[iE]), r[iA][-5:], r[iSrc].strip()))
        except (ValueError, IndexError):
            pass
    ts, te = sum(d[0] for d in data), sum(d[1] for d in data)
    print(f"# {path}: {ts} stall samples, {te} warp instructions")
    for d in sorted(data, key=lambda x: -x[0])[:top]:
        print(f"{d[0]:6d} {100.0 * d[0] / ts:5.1f}% exec={d[1]:8d} {d[2]} {d[3]}")
    # cumulative samples by 256-byte address window
    win = {}
    for d in data:
        k = int(d[2], 16) // 0x200
        win[k] = win.get(k, 0) + d[0]
    print("# hottest 512-B windows (address // 0x200: samples)")
    for k, v in sorted(win.items(), key=lambda x: -x[1])[:12]:
        print(f"  {k * 0x200:05x}: {v} ({100.0 * v / ts:.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
