#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked evidence).

    python tools/ncu_summarize.py --rep gpurun_out/a.ncu-rep gpurun_out/b.ncu-rep \
        --launches gpurun_out/launches.csv --config c2 --out profiles/r01_ncu_c2

Writes <out>.md (human-readable) and merges per-phase DRAM bytes per launch
into profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

PHASE_OF = {  # kernel name fragment (mangled or demangled) -> bench phase name
    "coldot_pipe_kernelILi1": "adjoint",
    "coldot_pipe_kernel<1": "adjoint",
    "herm_gapply_persist_kernel": "gapply",
    "fwd_kernel<0, 256": "forward",
    "fwd_kernel<0, 512": "forward",
    "fwd_kernel<0, 1024": "forward",
    "coldot_kernelI6float2Li1": "adjoint",
    "fwd_kernelILi0": "forward",
    "coldot_kernelI7double2Li0": "gapply",
    "coldot_kernelI7double2Li2": "primal",
    "fusion_kernel": "fusion",
    "fused_sweep2_kernel": "sweep",
    "herm_gapply_tma_kernel": "gapply",
    "herm_gapply_kernel": "gapply",
    "herm_reduce_kernel": "gapply_reduce",
    "gram_dmma_kernel": "gram",
    "frame_batch2_kernelILi0": "frames_forward",
    "frame_batch2_kernelILi2": "frames_adjoint",
    "coldot_kernel<float2, 1": "adjoint",
    "fwd_kernel<0>": "forward",
    "coldot_kernel<double2, 0": "gapply",
    "coldot_kernel<double2, 2": "primal",
}
METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[2:]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = r[h.index("Kernel Name")].split("(")[0]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[h.index("Metric Value")].replace(",", ""))
    return agg


def capture_rows(rep):
    h, rows = raw(rep)
    out = []
    for r in rows:
        d = {m: r[h.index(m)] for m in METRICS if m in h}
        d["name"] = r[h.index("Kernel Name")]
        d["rep"] = os.path.basename(rep)
        st = {}
        for i, col in enumerate(h):
            if col.startswith("smsp__pcsamp_warps_issue_stalled_") and not col.endswith("not_issued"):
                try:
                    st[col.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        d["stalls"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:4]}
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    md = [f"# ncu summary {os.path.basename(a.out)} ({a.config})", "", a.note, ""]
    summary_path = os.path.join(os.path.dirname(a.out), "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## launch list (gpu__time_duration.sum, cold-cache serialised; compare shares)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{n}` | {c} | {v / 1e6:.3f} | {100 * v / tot:.1f}% |")
        md.append("")
    if a.rep:
        md += ["## full-set captures", ""]
        per = collections.defaultdict(list)
        for rep in a.rep:
            for d in capture_rows(rep):
                try:  # a launch cut off by -c has no metric values
                    if float(d.get("dram__bytes_read.sum", "").replace(",", "")) != \
                            float(d.get("dram__bytes_read.sum", "").replace(",", "")):
                        continue  # nan
                except ValueError:
                    continue
                for frag, phase in PHASE_OF.items():
                    if frag in d["name"]:
                        per[phase].append(d)
                        break
        for phase, ds in per.items():
            rd = [float(x["dram__bytes_read.sum"]) for x in ds]
            wr = [float(x["dram__bytes_write.sum"]) for x in ds]
            dur = [float(x["gpu__time_duration.sum"]) for x in ds]
            traffic = (sum(rd) + sum(wr)) / len(ds)
            summary.setdefault(a.config, {})[phase] = {
                "dram_bytes_per_launch": traffic, "duration_ns": sum(dur) / len(dur), "captures": len(ds),
                "source": ds[0]["rep"]}
            md += [f"### {phase} (`{ds[0]['name'][:90]}`)", "",
                   f"- launches captured: {len(ds)}; mean duration {sum(dur) / len(dur) / 1e3:.1f} us "
                   f"(ncu, clocks uncontrolled)",
                   f"- DRAM read {sum(rd) / len(ds) / 1e9:.4f} GB + write {sum(wr) / len(ds) / 1e9:.4f} GB per launch",
                   f"- DRAM throughput {ds[0].get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}% of "
                   f"peak; warps active {ds[0].get('sm__warps_active.avg.pct_of_peak_sustained_active')}%; "
                   f"regs {ds[0].get('launch__registers_per_thread')}; grid {ds[0].get('launch__grid_size')} x "
                   f"{ds[0].get('launch__block_size')}",
                   f"- fp64 pipe {ds[0].get('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active')}%; "
                   f"tensor pipe {ds[0].get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')}%; "
                   f"smem ld bank conflicts {ds[0].get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum')};"
                   f" L2 hit {ds[0].get('lts__t_sector_hit_rate.pct')}%",
                   f"- top stalls: {ds[0]['stalls']}", ""]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
