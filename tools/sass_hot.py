"""Hot SASS instructions from an `ncu --page source --csv --print-source sass` export.

    python tools/sass_hot.py <file.csv[.gz]> [top] [lo_addr hi_addr]

Prints the stall-reason totals and the `top` instructions by warp-stall samples
(address, samples, top reasons, SASS), so a kernel's critical loop can be read
without the GUI.
"""
import csv
import gzip
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        rows = list(csv.reader(f))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    return hdr, [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr, rows = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {s: 0 for s in stalls}
    samples = []
    for k, r in enumerate(rows):
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        for s in stalls:
            tot[s] += int(r[ix[s]] or 0)
        samples.append((n, k))
    all_n = sum(n for n, _ in samples)
    print(f"instructions {len(rows)}  samples {all_n}")
    for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {s:28s} {v:8d} {100.0 * v / max(1, all_n):5.1f}%")
    print()
    for n, k in sorted(samples, reverse=True)[:top]:
        r = rows[k]
        rs = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
        why = " ".join(f"{s}:{v}" for v, s in rs if v)
        print(f"{k:5d} {n:6d} {100.0 * n / all_n:5.2f}%  {r[ix['Source']].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main()
