"""SASS hot spots of an ncu --set full capture: per instruction the warp-stall
samples, executions and dominant stall reasons, plus a per-region rollup
(regions split at BAR/branch targets are not inferred: pass address ranges).

usage: ncu -i rep --page source --csv --print-source sass > sass.csv
       python tools/ncu_sass_hot.py sass.csv [top]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    ia, isrc = h.index("Address"), h.index("Source")
    isamp, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    st = [(i, n[6:]) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(float(r[isamp] or 0) for r in data)
    totex = sum(float(r[iex] or 0) for r in data)
    print(f"total samples {tot:.0f}, instructions executed {totex:.0f}")
    order = sorted(range(len(data)), key=lambda k: -float(data[k][isamp] or 0))
    for k in order[:top]:
        r = data[k]
        s = float(r[isamp] or 0)
        reasons = sorted(((float(r[i] or 0), n) for i, n in st), reverse=True)[:3]
        rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
        print(f"{k:5d} {s / tot * 100:5.1f}% ex={float(r[iex] or 0):9.0f}  {r[isrc].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
