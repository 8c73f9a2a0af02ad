"""Per-source-line aggregation of an ncu source page (development aid):
    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
    python tools/ncu_lines.py X.csv [top]
Sums warp-stall samples, their top stall reasons and shared-memory wavefronts per CUDA line."""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    agg = defaultdict(lambda: defaultdict(float))
    text = {}
    fname, hdr, cur = None, None, None
    with open(path) as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                fname = row[1].split("/")[-1]
                continue
            if row[0] == "Line No":
                hdr = row
                continue
            if hdr is None or len(row) != len(hdr):
                continue
            if row[0]:
                cur = (fname, int(row[0]))
                text[cur] = row[1].strip()[:90]
                continue
            d = dict(zip(hdr[2:], row[2:]))
            a = agg[cur]
            for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
                      "L1 Wavefronts Shared Excessive"):
                try:
                    a[k] += float(d.get(k, 0) or 0)
                except ValueError:
                    pass
            for k, v in d.items():
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        a[k] += float(v or 0)
                    except ValueError:
                        pass
    tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]
    print(f"total samples {tot:.0f}")
    for (fn, ln), a in rows:
        s = a["Warp Stall Sampling (All Samples)"]
        st = sorted(((v, k[6:]) for k, v in a.items() if k.startswith("stall_")), reverse=True)[:3]
        print(f"{100 * s / tot:5.1f}% {fn}:{ln:<5} inst {a['Instructions Executed']:9.0f} smem {a['L1 Wavefronts Shared']:8.0f}"
              f" (+{a['L1 Wavefronts Shared Excessive']:.0f})  " + " ".join(f"{k}:{v:.0f}" for v, k in st) + f" | {text.get((fn, ln), '')}")


if __name__ == "__main__":
    main()
