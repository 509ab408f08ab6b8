"""Summarise `ncu --set full` captures of the first sort of a bench run into
profiles/ncu_full_summary.json: per (workload, step kernel, level) the DRAM bytes of that
launch (a step issued as several launches -- Step 9's size tiers, Step 8's two forms --
summed), its duration and what bounds it (issue slots, ALU pipe, shared-memory
wavefronts, bank conflicts, top warp stalls).  bench.py reads `roofline.traffic` and
`roofline.limiter` from it.

usage: python scripts/ncu_summary.py summary.json LABEL=report.ncu-rep [LABEL=report ...]

Kernel base names are normalised (k_sample_index_tma -> k_sample_index, k_relocate_grouped
-> k_relocate, k_segment_sort_rare -> k_segment_sort); the item kind is the first template
argument (0 keys, 1 pairs, 2 u64 sample levels = Step 4).  A launch belongs to level k when
k local sorts of its kind precede it (every level starts with its Step 2).  The report must
hold exactly one sort (bench.py --ncu-one)."""
import csv
import io
import json
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
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
NORM = {"k_sample_index_tma": "k_sample_index", "k_relocate_grouped": "k_relocate",
        "k_segment_sort_rare": "k_segment_sort"}
SUM = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")


def launches(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
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
        yield d


def base_kind(name):
    n = re.sub(r"^void ", "", name).replace("gbs::", "")
    base = n.split("<")[0].split("(")[0]
    m = re.match(r"[^<]*<\(?(?:gbs::)?(?:Kind\))?(\d+)", n)
    kind = int(m.group(1)) if m else -1
    return NORM.get(base, base), kind


def main():
    out_path = sys.argv[1]
    try:
        summary = json.load(open(out_path))
    except (OSError, ValueError):
        summary = {"kernels": {}}
    for spec in sys.argv[2:]:
        label, rep = spec.split("=", 1)
        recs = list(launches(rep))
        cur = {}
        for d in recs:
            base, kind = base_kind(d["kernel"])
            if base == "k_local_sort" and kind in (0, 1):
                cur[kind] = cur.get(kind, 0) + 1          # a local sort starts every level
            if kind == 2:
                key = f"{label}:{base}:step4"
            elif base in ("k_local_sort", "k_sample_index", "k_relocate", "k_scan", "k_segment_sort",
                          "k_local_sort_pair", "k_bucket_tiers"):
                key = f"{label}:{base}:level{max(1, cur.get(kind, 1))}"
            else:
                key = f"{label}:{base}"
            e = summary["kernels"].get(key)
            if e is None or e.get("_rep") != rep:
                e = dict(d, launches=1, parts=[d["kernel"]], _rep=rep, _longest=d.get("gpu__time_duration.sum", 0))
                summary["kernels"][key] = e
            else:
                # a step issued as several launches of one step kernel: sum traffic and time;
                # the utilisation and stall figures are those of its longest launch
                longest = d.get("gpu__time_duration.sum", 0) > e.get("_longest", 0)
                for w in SUM:
                    if isinstance(d.get(w), float):
                        e[w] = e.get(w, 0.0) + d[w]
                if longest:
                    for w, v in d.items():
                        if w not in SUM and w != "kernel":
                            e[w] = v
                    e["_longest"] = d.get("gpu__time_duration.sum", 0)
                e["launches"] += 1
                e["parts"].append(d["kernel"])
            e["dram_bytes_one_launch"] = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
            e["duration_us"] = e.get("gpu__time_duration.sum")
            e["capture"] = f"ncu --set full, {label}, first sort of the bench command"
    for e in summary["kernels"].values():
        e.pop("_rep", None)
        e.pop("_longest", None)
    open(out_path, "w").write(json.dumps(summary, indent=1))
    for k, e in summary["kernels"].items():
        print(f"{k:40s} {e.get('duration_us', 0):10.1f} us  DRAM {e['dram_bytes_one_launch'] / 1e6:9.1f} MB  "
              f"issue {e.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
              f"alu {e.get('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
              f"smem {e.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 0):5.1f}%  "
              f"stalls {e['top_stalls'][:3]}")


if __name__ == "__main__":
    main()
