#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of ONE step of a multi-kernel bench
mode (backward, multi-resolution, temporal) into profiles/.

    python scripts/summarize_ncu_step.py REP TAG "WORKLOAD" ALGO_BYTES

REP holds the kernels of one step (ncu -k/-s/-c chosen so), TAG names the
output profiles/ncu_TAG.md, WORKLOAD is the bench line's config.workload
string and ALGO_BYTES the algorithmic bytes of one step.  The DRAM bytes of
the step (summed over its kernels) go to profiles/traffic.json under WORKLOAD
with the libkmd source hash; bench.py reports them as roofline.traffic.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

from summarize_ncu import raw, to_bytes  # noqa: E402

COLS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def main():
    rep, tag, workload, algo = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    recs, units = raw(rep)
    lines = [f"# ncu summary `{tag}` — one step of: {workload}", "",
             f"Source: `{os.path.basename(rep)}` (`ncu --set full --clock-control none`, the "
             f"{len(recs)} kernels of one bench step; cold cache, serialised).", "",
             "| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM read MB | DRAM write MB |",
             "|---|" + "---|" * (len(COLS) + 2)]
    tot_rd = tot_wr = tot_t = 0.0
    for d in recs:
        rd = to_bytes(d["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
        tot_rd += rd
        tot_wr += wr
        vals = []
        for k, _, scale in COLS:
            v = d.get(k, "")
            try:
                v = float(str(v).replace(",", ""))
                if k == "gpu__time_duration.sum":
                    unit = units.get(k, "nsecond")
                    v = v * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
                    tot_t += v
                vals.append(f"{v * scale:,.1f}")
            except ValueError:
                vals.append(str(v))
        name = d.get("Kernel Name", "?").split("(")[0][:70]
        lines.append(f"| `{name}` | " + " | ".join(vals) + f" | {rd / 1e6:,.1f} | {wr / 1e6:,.1f} |")
    lines += ["", f"Step total: {tot_t / 1e3:,.1f} us (cold), DRAM {(tot_rd + tot_wr) / 1e6:,.1f} MB "
                  f"= {(tot_rd + tot_wr) / algo:.2f}x the algorithmic {algo / 1e6:,.1f} MB."]
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    import bench  # noqa: E402  (source hash)
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t[workload] = {"dram_bytes_per_launch": tot_rd + tot_wr, "dram_read": tot_rd, "dram_write": tot_wr,
                   "per": "step", "lib_sha": bench.lib_sources_hash(), "capture": os.path.basename(rep), "tag": tag}
    json.dump(t, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
