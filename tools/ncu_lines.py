"""Per-source-line hot spots of an ncu --set full --import-source capture:
warp-stall samples, instructions executed and the dominant stall reasons per
CUDA line (from `ncu -i rep --page source --print-source cuda,sass --csv`).

usage: python tools/ncu_lines.py <capture.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    col = {name: i for i, name in enumerate(h) if name not in col_seen(h, i)} if False else None
    idx = {}
    for i, name in enumerate(h):
        idx.setdefault(name, i)
    stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    lines = []
    total = 0
    for r in rows[hi + 1:]:
        if not r or not r[0] or r[0] == "Line No":
            continue
        try:
            samp = int(r[idx["Warp Stall Sampling (All Samples)"]])
            inst = int(r[idx["Instructions Executed"]])
        except (ValueError, KeyError, IndexError):
            continue
        stalls = sorted(((int(r[i]) if r[i].isdigit() else 0, n[6:]) for i, n in stall_cols), reverse=True)[:3]
        lines.append((samp, inst, r[0], r[1].strip()[:90], stalls))
        total += samp
    lines.sort(reverse=True)
    print(f"total stall samples {total}")
    for samp, inst, ln, src, st in lines[:top]:
        s = " ".join(f"{n}:{v}" for v, n in st if v)
        print(f"{samp:7d} {100.0 * samp / max(1, total):5.1f}% inst {inst:10d} L{ln:>4} {src}  [{s}]")


def col_seen(h, i):
    return set()


if __name__ == "__main__":
    main()
