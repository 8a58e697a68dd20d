"""Summarise an ncu report (or an ncu launch-list CSV) into profiles/.

    python tools/ncu_summary.py report.ncu-rep  profiles/ncu_fused_fwd_r01   [--bytes-per-launch N]
    python tools/ncu_summary.py launches.csv    profiles/launches_r01

For a full-set report writes <out>.txt (key throughput / pipe / stall metrics
per kernel) and <out>.json (dram bytes per launch etc.; bench.py reads
profiles/ncu_fused_fwd.json for the roofline "traffic").  For a launch list
writes per-kernel launch counts, mean/total device time and share of the step.
"""

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "sm cycles"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe %"),
    ("l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 TEX data-pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared ld bank conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:] if len(r) == len(hdr)]


def summarise_report(rep, out, bytes_per_launch=None):
    lines, js = [], OrderedDict()
    for i, (d, u) in enumerate(raw_rows(rep)):
        name = d.get("Kernel Name", f"kernel{i}")
        lines.append(f"== launch {i}: {name}")
        rec = OrderedDict()
        for key, label in KEYS:
            if key in d:
                lines.append(f"  {label:28s} {d[key]:>16s} {u.get(key, '')}")
                rec[key] = d[key]
        stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v))
                  for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and v not in ("", "0")]
        tot = sum(v for _, v in stalls) or 1.0
        stalls.sort(key=lambda kv: -kv[1])
        lines.append("  top stall reasons (pc sampling): " +
                     ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in stalls[:6]))
        rd = float(d.get("dram__bytes_read.sum", "nan") or "nan")
        wr = float(d.get("dram__bytes_write.sum", "nan") or "nan")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= mult.get(u.get("dram__bytes_read.sum", "byte"), 1)
        wr *= mult.get(u.get("dram__bytes_write.sum", "byte"), 1)
        rec["dram_bytes_per_launch"] = rd + wr
        if bytes_per_launch:
            rec["algorithmic_bytes_per_launch"] = bytes_per_launch
            lines.append(f"  dram bytes / algorithmic bytes = {(rd + wr) / bytes_per_launch:.3f}")
        js[f"{i}:{name}"] = rec
    open(out + ".txt", "w").write("\n".join(lines) + "\n")
    first = next(iter(js.values()))
    summary = {"source": rep, "kernels": js, "dram_bytes_per_launch": first["dram_bytes_per_launch"]}
    json.dump(summary, open(out + ".json", "w"), indent=1)
    print("\n".join(lines))


def summarise_launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            recs.append(dict(zip(hdr, r)))
    agg = defaultdict(list)
    for r in recs:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"]].append(float(r["Metric Value"]))
    total = sum(sum(v) for v in agg.values()) or 1.0
    lines = [f"{'kernel':70s} {'launches':>8s} {'mean_ns':>12s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:70]:70s} {len(v):8d} {sum(v) / len(v):12.1f} {100 * sum(v) / total:6.1f}%")
    open(out + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    bpl = None
    if "--bytes-per-launch" in sys.argv:
        bpl = float(sys.argv[sys.argv.index("--bytes-per-launch") + 1])
    if src.endswith(".csv"):
        summarise_launches(src, dst)
    else:
        summarise_report(src, dst, bpl)
