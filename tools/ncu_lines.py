"""Per-source-line hot spots from an ncu mixed source page export
(ncu -i rep --page source --csv --print-source cuda,sass -k regex:K --launch-count 1).
Usage: python tools/ncu_lines.py export.csv [top]"""
import csv
import sys


def main(path, top=40):
    rows = []
    fname = "?"
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            samp = int(r[4]); inst = int(r[7])
        except ValueError:
            continue
        rows.append((samp, inst, fname, r[0], r[1].strip()[:90]))
    ts = sum(x[0] for x in rows) or 1
    ti = sum(x[1] for x in rows) or 1
    print(f"total samples {ts}  total warp-inst {ti:.3e}")
    for samp, inst, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*samp/ts:5.1f}% samp {100*inst/ti:5.1f}% inst  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
