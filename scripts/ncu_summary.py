"""Summarise an ncu --set full report: per kernel, the metrics the roofline needs plus
the top warp-stall reasons.  usage: python scripts/ncu_summary.py report.ncu-rep [json_out]"""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {"report": rep, "kernels": {}}
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  and h.endswith(".ratio")] or \
                 [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        d = {}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)]
                try:
                    d[w] = float(v.replace(",", ""))
                except ValueError:
                    d[w] = v
                d[w + ".unit"] = units[hdr.index(w)]
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i].replace(",", "")), hdr[i]))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        d["top_stalls"] = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), round(v, 3))
                           for v, h in stalls[:6]]
        out["kernels"].setdefault(name, []).append(d)
    js = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(js)
    for k, lst in out["kernels"].items():
        for d in lst:
            print("==", k)
            for w in WANT:
                if w in d:
                    print(f"   {w}: {d[w]} {d[w + '.unit']}")
            print("   stalls:", d["top_stalls"])


if __name__ == "__main__":
    main()
