"""Summarize an ncu launch list (CSV) and full captures (.ncu-rep) into markdown for profiles/."""
import csv
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_writes_op_utcmma.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    agg = defaultdict(lambda: defaultdict(float))
    ids = defaultdict(set)
    for r in data:
        if len(r) < len(h):
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ddcca::", "")
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "second": 1e3, "s": 1e3}.get(r[ui], 1.0)
        elif r[ui] in ("Kbyte", "KB"):
            v *= 1e3
        elif r[ui] in ("Mbyte", "MB"):
            v *= 1e6
        elif r[ui] in ("Gbyte", "GB"):
            v *= 1e9
        agg[name][r[mi]] += v
        ids[name].add(r[idi])
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = ["| kernel | launches | ms (serialized, cold) | share | DRAM GB |", "|---|---:|---:|---:|---:|"]
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        out.append(f"| `{n}` | {len(ids[n])} | {t:.2f} | {100 * t / tot:.1f} % | "
                   f"{(a['dram__bytes_read.sum'] + a['dram__bytes_write.sum']) / 1e9:.2f} |")
    out.append(f"| total | | {tot:.2f} | | |")
    return "\n".join(out)


def full(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    units = dict(zip(h, rows[1])) if len(rows) > 1 else {}  # second row: the metric units
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        out.append(f"**{d.get('Kernel Name', '?')}** (grid {d.get('launch__grid_size')}, block "
                   f"{d.get('launch__block_size')}, {d.get('launch__registers_per_thread')} regs)\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS[:1] + KEYS[1:]:
            if k in d and k not in ("launch__grid_size", "launch__block_size", "launch__registers_per_thread"):
                out.append(f"| `{k}` | {d[k]} | {units.get(k, '')} |")
        stalls = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        out.append("\nTop stall reasons (pc sampling): " +
                   ", ".join(f"{n} {100 * v / tot:.0f} %" for v, n in sorted(stalls, reverse=True)[:6]) + "\n")
    return "\n".join(out)


if __name__ == "__main__":
    d = Path(sys.argv[1])
    parts = ["## Launch list\n", launches(d / "launches.csv"), ""]
    for rep in sorted(d.glob("*.ncu-rep")):
        parts += [f"## Full capture: {rep.name}\n", full(rep), ""]
    print("\n".join(parts))
