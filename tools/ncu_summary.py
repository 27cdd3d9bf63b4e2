"""Summarise an ncu --set full report of the fused kernel into profiles/ (markdown + JSON).

usage: python tools/ncu_summary.py <report.ncu-rep> <tag> [config] [texels]
Writes profiles/<tag>_fused_ncu.md, profiles/<tag>_fused_ncu.json and refreshes
profiles/latest_fused_traffic.json (read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def main(rep, tag, config=3, texels=4096 * 4096):
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    out = {"report": os.path.basename(rep), "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for k in KEYS:
        if k in m:
            out[k] = m[k]
    stalls = {h.split("issue_stalled_")[1].split("_per")[0]: float(v) for h, v in zip(hdr, vals)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio") and v}
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    ops = collections.Counter()
    for r in src[2:]:
        if len(r) <= iE:
            continue
        mm = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
        try:
            n = int(r[iE])
        except ValueError:
            continue
        if mm:
            ops[mm.group(2)] += n
    total = sum(ops.values())
    out["warp_instructions"] = total
    out["thread_instructions_per_texel"] = total * 32 / texels
    out["op_mix_per_texel"] = {k: round(v * 32 / texels, 1) for k, v in ops.most_common(25)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(m["dram__bytes_read.sum"][0]) * scale[m["dram__bytes_read.sum"][1]]
    wr = float(m["dram__bytes_write.sum"][0]) * scale[m["dram__bytes_write.sum"][1]]
    out["dram_bytes_per_launch"] = rd + wr
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_fused_ncu.json"), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "profiles", "latest_fused_traffic.json"), "w") as f:
        def pct(k):
            return float(m[k][0]) / 100.0 if k in m else None
        json.dump({"config": config, "dram_bytes_per_launch": rd + wr, "source": f"{tag}_fused_ncu.json",
                   "issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                   "fma_pipe": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                   "tensor_pipe": pct("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                   "thread_instructions_per_texel": out.get("thread_instructions_per_texel")}, f)
    lines = [f"# ncu --set full summary: {out['kernel'][:90]}", "", f"report: `{rep}` (tag {tag})", "",
             "| metric | value |", "|---|---|"]
    for k in KEYS:
        if k in out:
            lines.append(f"| {k} | {out[k][0]} {out[k][1]} |")
    lines += ["", f"thread instructions per texel: {out['thread_instructions_per_texel']:.0f}", "",
              "| op | thread-instr per texel |", "|---|---|"]
    lines += [f"| {k} | {v} |" for k, v in out["op_mix_per_texel"].items()]
    lines += ["", "| stall reason | warps per issue |", "|---|---|"]
    lines += [f"| {k} | {v:.3f} |" for k, v in out["stalls_per_issue"].items()]
    with open(os.path.join(ROOT, "profiles", f"{tag}_fused_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(int(x) for x in sys.argv[3:]))
