"""Hot SASS lines of an `ncu --page source --csv --print-source sass` export.

python tools/ncu_src_hot.py report_src.csv [kernel-substring] [top-n]
Prints, per kernel section, total stall samples by reason and the top-n lines.
"""
import csv
import sys
from collections import Counter


def sections(path):
    cur, rows, header = None, [], None
    with open(path, newline="") as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "Kernel Name":
                if cur:
                    yield cur, header, rows
                cur, rows, header = rec[1], [], None
            elif rec[0] == "Address":
                header = rec
            elif header:
                rows.append(dict(zip(header, rec)))
    if cur:
        yield cur, header, rows


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    seen = set()
    for name, header, rows in sections(path):
        if want not in name or name in seen:
            continue
        seen.add(name)
        reasons = [h for h in header if h.startswith("stall_") and "Not Issued" not in h]
        tot = Counter()
        for r in rows:
            for h in reasons:
                tot[h] += int(r.get(h, "0") or 0)
        samples = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
        inst = sum(int(r["Instructions Executed"] or 0) for r in rows)
        print(f"== {name[:110]}\n   samples={samples} warp-inst={inst}")
        print("   " + " ".join(f"{k[6:]}={v}" for k, v in tot.most_common(10) if v))
        idx = {i: r for i, r in enumerate(rows)}
        hot = sorted(idx, key=lambda i: -int(idx[i]["Warp Stall Sampling (All Samples)"] or 0))[:top]
        for i in sorted(hot):
            r = idx[i]
            st = Counter({h[6:]: int(r.get(h, "0") or 0) for h in reasons})
            print(f"   {i:5d} {r['Warp Stall Sampling (All Samples)']:>6s} ex={r['Instructions Executed']:>8s} "
                  f"{r['Source'].strip()[:60]:60s} {' '.join(f'{k}={v}' for k, v in st.most_common(3) if v)}")


if __name__ == "__main__":
    main()
