"""Summarise an ncu dram-bytes capture of the hot kernels into
profiles/ncu_summary.json (read by bench.py for roofline.traffic).

Capture (one GPU, full bench size; three metrics = one pass, no replay):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv -k regex:"k_expand|k_nd_pass|k_materialize|k_patch" -s 6 -c 6 \
      --log-file gpurun_out/dram_full.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu
Usage: python tools/ncu_summary.py gpurun_out/dram_full.csv [profiles/ncu_summary.json] [config]
"""
import csv
import json
import sys
from collections import defaultdict

PHASE = {"k_expand": "expand", "k_nd_pass": "expand", "k_materialize": "materialize", "k_patch": "materialize",
         "k_overflow_fix": "materialize"}


def main(src, dst="profiles/ncu_summary.json", config=4):
    rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0].isdigit()]
    per_launch = defaultdict(dict)  # launch id -> {kernel, metrics}
    for r in rows:
        d = per_launch[int(r[0])]
        d["kernel"] = r[4]
        d[r[12]] = float(r[14])
    # the last launch of each kernel name (steady state)
    last = {}
    for lid in sorted(per_launch):
        name = per_launch[lid]["kernel"]
        key = next((k for k in PHASE if k in name), None)
        if key:
            last[key] = per_launch[lid]
    phases = {}
    for key, d in last.items():
        ph = phases.setdefault(PHASE[key], {"kernels": [], "dram_read": 0.0, "dram_write": 0.0, "duration_ms": 0.0})
        ph["kernels"].append(d["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", ""))
        ph["dram_read"] += d.get("dram__bytes_read.sum", 0.0)
        ph["dram_write"] += d.get("dram__bytes_write.sum", 0.0)
        ph["duration_ms"] += d.get("gpu__time_duration.sum", 0.0) / 1e6
    for ph in phases.values():
        ph["dram_bytes_per_launch"] = ph["dram_read"] + ph["dram_write"]
    out = {"note": "dram bytes per launch (read + write) of each hot phase's kernels at the bench's "
                   "full size, one ncu pass with three metrics (no replay); cold-cache serialised launches",
           "source": src, "config": int(config), "kernels": phases}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
