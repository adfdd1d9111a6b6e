"""Per-source-line instruction and stall shares of one kernel in an ncu report.
Usage: python tools/ncu_lines.py <report.ncu-rep> [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, kern="", top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, fn, agg = None, "", {}
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No" or kern not in fn or not r[0]:
            continue
        agg[(cur_file, int(r[0]))] = (num(r[7]), num(r[4]), r[1].strip()[:100])
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"warp instructions {tot}, stall samples {ts}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"inst {v[0] / tot:6.3f} stall {v[1] / ts:6.3f}  {k[0]}:{k[1]}  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 40)
