"""Summarise an `ncu --set full` report of the hot kernels (one launch each)
into a small JSON under profiles/: time, DRAM bytes, instructions, issue and
occupancy, LSU load, tensor-pipe activity and the stall-reason mix.
Usage: python tools/ncu_full_summary.py gpurun_out/<tag>/prof.ncu-rep profiles/r01/<name>.json "<capture cmd>" """
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, out, capture):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"capture": capture, "kernels": {}}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("snp::<unnamed>::", "").replace("<unnamed>::", "")
        k = {key: [d.get(key), u.get(key)] for key in KEYS if key in d}
        st = [(key.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for key, v in d.items()
              if key.startswith("smsp__pcsamp_warps_issue_stalled_") and v and not key.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        k["stall_reasons_pct"] = {a: round(100 * v / tot, 1) for a, v in sorted(st, key=lambda x: -x[1])[:8]}
        res["kernels"].setdefault(name, k)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main(*sys.argv[1:4])
