"""Summarise an ncu --set full report: per kernel, the metrics the roofline needs plus the
top warp-stall reasons.

usage: python scripts/ncu_summary.py report.ncu-rep [summary.json]

The JSON maps the kernel base name (k_local_sort, k_segment_sort, ...) of the FIRST
captured instance (the top-level, keys) to dram bytes per launch, duration, pipe
utilisation and stalls; bench.py reads `dram_bytes_per_launch` as roofline.traffic."""
import csv
import io
import json
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    out = {"report": rep, "kernels": {}, "all": []}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        base = re.sub(r"^void ", "", name).split("<")[0].split("(")[0].replace("gbs::", "")
        d = {"kernel": name}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)]
                try:
                    d[w] = float(v.replace(",", "")) * SCALE.get(units[hdr.index(w)], 1)
                except ValueError:
                    d[w] = v
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i].replace(",", "")), hdr[i]))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        d["top_stalls"] = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                            round(v, 3)) for v, h in stalls[:6]]
        d["dram_bytes_per_launch"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        d["duration_us"] = d.get("gpu__time_duration.sum")
        prev = out["all"][-1]["kernel"] if out["all"] else None
        out["all"].append(d)
        first = out["kernels"].get(base)
        if first is None:
            out["kernels"][base] = dict(d, launches=1, parts=[name])
        elif prev is not None and prev.split("<")[0] == name.split("<")[0] \
                and prev.split(",")[0] == name.split(",")[0] and first["parts"][-1] == prev:
            # a step issued as back-to-back launches of one kernel and item kind (Step 9's
            # split by bucket size): the step's traffic and time are their sum
            first["dram_bytes_per_launch"] += d["dram_bytes_per_launch"]
            first["duration_us"] = (first["duration_us"] or 0) + (d["duration_us"] or 0)
            first["launches"] += 1
            first["parts"].append(name)
    js = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(js)
    for d in out["all"]:
        print("==", d["kernel"])
        for w in WANT:
            if w in d:
                print(f"   {w}: {d[w]}")
        print("   stalls:", d["top_stalls"])


if __name__ == "__main__":
    main()
