"""Summarise ncu artefacts into small, committable text files under profiles/.

    python tools/ncu_summary.py report <file.ncu-rep> <kernel-regex> <out.md>
    python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe active % (of elapsed)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "FP64 tensor (DMMA) sub-pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("smsp__warps_active.avg.per_cycle_active", "warps active / SMSP"),
    ("smsp__warps_eligible.avg.per_cycle_active", "warps eligible / SMSP"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep, regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{regex}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(units, r))) for r in rows[2:]]


def report(rep, regex, out):
    recs = raw(rep, regex)
    lines = [f"# ncu --set full summary: `{regex}`", "", f"source: `{rep}` "
             "(ncu --set full --clock-control none --import-source on; cold-cache replay)", ""]
    summary = {}
    for i, d in enumerate(recs):
        name = d.get("Kernel Name", ("", "?"))[1]
        lines += [f"## launch {i}: `{name[:90]}`", "", "| metric | value | unit |", "|---|---|---|"]
        for k, label in KEYS:
            if k in d:
                u, v = d[k]
                lines.append(f"| {label} (`{k}`) | {v} | {u} |")
                summary.setdefault(name, {})[k] = [v, u]
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(v[1])) for h, v in d.items()
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("ratio")
              and v[1] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        lines += ["", "top stall reasons (warps stalled per issued instruction):", ""]
        lines += [f"- {n}: {v:.3f}" for n, v in st[:8]]
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    open(out.replace(".md", ".json"), "w").write(json.dumps(summary, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        agg[r[iK]].append(float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# launch list: `{path}`", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
             "compare shares, not absolutes)", "",
             "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        short = re.sub(r"\(.*", "", k)[:70]
        lines.append(f"| `{short}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot * 100:.1f}% |")
    # the timed Schur step only: the kernels one SM-partitioned cfg3 step
    # launches (setup, GMRES, SVD, peaks and torch's L2-flush fills excluded),
    # each kernel's total time divided by the number of steps (= K1s launches)
    step_re = re.compile(r"bloch_weight_1|ct_gemv|sum_parts|pinv_gemv|pinv_uh|pinv_v|b_gemv|"
                         r"m2l_sym_kernel|m2l_sym_stage_kernel|k1s_reduce")
    nsteps = sum(len(v) for k, v in agg.items() if "m2l_sym_kernel" in k or "m2l_sym_stage_kernel" in k) or 1
    step = {k: v for k, v in agg.items() if step_re.search(k)}
    ts = sum(sum(v) for v in step.values()) / nsteps
    lines += ["", f"per Schur step ({nsteps} steps = K1s launches; every step kernel's total time / "
              "steps; shares of their sum):", "",
              "| kernel | launches per step | us per step | share of step |", "|---|---|---|---|"]
    for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
        short = re.sub(r"\(.*", "", k)[:70]
        m = sum(v) / nsteps
        lines.append(f"| `{short}` | {len(v) / nsteps:g} | {m:.1f} | {m / ts * 100:.1f}% |")
    lines.append(f"| total | | {ts:.1f} | |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
