#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of the fused kernel into profiles/.

    python scripts/summarize_ncu.py gpurun_out/prof_TAG.ncu-rep TAG [launches.csv]

Writes profiles/ncu_TAG.md (key counters, stall breakdown) and records the
per-launch DRAM traffic in profiles/traffic.json keyed by the bench workload
and the libkmd source hash, which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = [
    ("gpu__time_duration.sum", "duration (cold cache, serialised)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic shared memory / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    recs, units = raw(rep)
    d = recs[0]
    lines = [f"# ncu summary `{tag}` — `{d.get('Kernel Name', '?')[:90]}`", "",
             f"Source: `{os.path.basename(rep)}` (`ncu --set full --clock-control none`, one launch "
             "of `python bench.py --steps 16 --warmup 8 --no-cpu-baseline --e2e-steps 0` "
             "= 1920x1080, sizes {3,5,7,9,11,13}).", "",
             "| counter | value | unit |", "|---|---|---|"]
    for k, name in KEYS:
        if k in d:
            lines.append(f"| {name} (`{k}`) | {d[k]} | {units.get(k, '')} |")
    stalls = sorted(((k, float(v)) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
                     and v not in ("", None)), key=lambda x: -x[1])
    lines += ["", "Warp stall reasons (cycles per issued instruction):", "",
              "| reason | ratio |", "|---|---|"]
    for k, v in stalls[:10]:
        if v > 0.02:
            lines.append(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {v:.3f} |")
    rd = to_bytes(d["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
    wr = to_bytes(d["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
    algo = 72 * 1920 * 1080
    lines += ["", f"DRAM traffic per launch: {rd + wr:,.0f} B vs algorithmic {algo:,} B "
                  f"({(rd + wr) / algo:.3f}x). Halo re-reads are served from L2/shared memory, not DRAM."]
    if launches and os.path.exists(launches):
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10 and r[0].isdigit()]
        tot = {}
        for r in rows:
            name = r[4].split("(")[0][:60]
            tot.setdefault(name, []).append(float(r[-1]))
        lines += ["", f"Launch list (`{os.path.basename(launches)}`, gpu__time_duration.sum per launch, ns):", "",
                  "| kernel | launches | mean ns | total share |", "|---|---|---|---|"]
        allt = sum(sum(v) for v in tot.values())
        for name, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{name}` | {len(v)} | {sum(v) / len(v):,.0f} | {sum(v) / allt:.1%} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    # traffic record for bench.py
    import bench  # noqa: E402  (for the workload string + source hash)
    workload = "1920x1080 frame, sizes [3, 5, 7, 9, 11, 13], fusion (BASELINE.json configs[2])"
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t[workload] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "lib_sha": bench.lib_sources_hash(), "capture": os.path.basename(rep), "tag": tag}
    json.dump(t, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
