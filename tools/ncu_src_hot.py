"""Source-line hot-spot table from an ncu report (``--page source --print-source
cuda,sass --csv``): per CUDA source line, warp-stall samples and executed warp
instructions (aggregated over the SASS it maps to), sorted by samples.

usage: python tools/ncu_src_hot.py report.ncu-rep KERNEL_REGEX [top] [--json out.json]"""
import csv
import io
import json
import subprocess
import sys


def hot(rep, kregex, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", "regex:" + kregex, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows, path, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[2] != "-":
            continue
        d = dict(zip(hdr[2:], r[2:]))
        rows.append({"file": path.split("/")[-1], "line": int(r[0]), "src": r[1].strip()[:90],
                     "samples": int(d.get("Warp Stall Sampling (All Samples)", 0) or 0),
                     "inst": int(d.get("Instructions Executed", 0) or 0)})
    tot_s = sum(x["samples"] for x in rows) or 1
    tot_i = sum(x["inst"] for x in rows) or 1
    rows.sort(key=lambda x: -x["samples"])
    for x in rows:
        x["samples_frac"] = round(x["samples"] / tot_s, 4)
        x["inst_frac"] = round(x["inst"] / tot_i, 4)
    return {"kernel": kregex, "total_samples": tot_s, "total_warp_inst": tot_i, "lines": rows[:top]}


if __name__ == "__main__":
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    res = hot(a[0], a[1], int(a[2]) if len(a) > 2 else 40)
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    print(f"total samples {res['total_samples']}  warp inst {res['total_warp_inst']:.3e}")
    for x in res["lines"]:
        print(f"{x['samples_frac']*100:5.1f}% {x['inst_frac']*100:5.1f}%  {x['file']}:{x['line']:<5d} {x['src']}")
