"""profiles/config_sweep_<tag>.md from a tools/experiments/config_sweep.py run
(gpurun_out/config_sweep.jsonl, and config_sweep_ttm5_before.jsonl = the same
ttm sweep with TL_TTM_FEW=0, i.e. without the few-row box kernel).

    python tools/summarize_sweep.py r05
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def load(name):
    path = os.path.join(OUT, name)
    if not os.path.exists(path):
        return []
    return [json.loads(l) for l in open(path) if l.startswith("{") and '"op"' in l]


def key_of(r):
    if r["op"] == "ttm":
        return "frac_fp64" if r["cfg"] == "cfg3" else "frac_hbm"
    return "frac"


def main(tag):
    rows = load("config_sweep.jsonl")
    before = {(tuple(r["layout"]), r["mode"]): r for r in load("config_sweep_ttm5_before.jsonl")}
    md = [f"# Config shapes under every layout and mode ({tag})", "",
          "`tools/experiments/config_sweep.py`: each config's shape in EVERY permutation layout (cfg2: 24, cfg3/cfg4: 6) or in",
          "seeded random layouts (cfg5's order-7 / order-6 shapes), every mode, timed by CUDA-graph replays; fraction of the",
          "pod's measured HBM copy peak for the algorithmic bytes (ttv, small-J ttm, inner, norm) or of the 37.05 TF/s FP64",
          "peak (cfg3 ttm). Every ttv / ttm result is compared with the first-order layout's result of the same logical",
          "tensor (`bit_identical` / `max_abs_diff_vs_first` = 0: each output is the same k-ordered chain in every layout).", "",
          "| op | shape | cases | min | p10 | median | max | >= 0.8 | < 0.5 | all bit-identical |", "|---|---|---|---|---|---|---|---|---|---|"]
    names = {"cfg2": "128^4 f32", "cfg3": "512^3 f64 x 384x512", "cfg4": "400^3 f64", "cfg5": "3x33x5x17(x9)x2x640 f64"}
    for op, cfg in sorted({(r["op"], r["cfg"]) for r in rows}):
        rs = [r for r in rows if r["op"] == op and r["cfg"] == cfg]
        fr = sorted(r[key_of(r)] for r in rs)
        if op == "ttv":
            same = all(r.get("bit_identical", True) for r in rs)
        elif op == "ttm":
            same = all(r.get("max_abs_diff_vs_first", 0.0) == 0.0 for r in rs)
        else:
            same = "-"
        unit = " (of FP64 peak)" if (op, cfg) == ("ttm", "cfg3") else ""
        md.append(f"| {op}{unit} | {names.get(cfg, cfg)} | {len(fr)} | {fr[0]:.3f} | {fr[len(fr) // 10]:.3f} | "
                  f"{statistics.median(fr):.3f} | {fr[-1]:.3f} | {sum(f >= 0.8 for f in fr)} | {sum(f < 0.5 for f in fr)} | {same} |")
    md.append("")
    t5 = [r for r in rows if r["op"] == "ttm" and r["cfg"] == "cfg5"]
    if t5:
        md += ["## Few-row ttm (J = 16) on the config-5 operand shape: before / after the box kernel (`csrc/ttm_few.cu`)", "",
               "`before` = the same build with `TL_TTM_FEW=0` (staged / GETT / one-thread-per-output paths).", "",
               "| layout | mode | K | before us | before frac | before path | after us | after frac | after path |",
               "|---|---|---|---|---|---|---|---|---|"]
        shape = (3, 33, 5, 17, 2, 640)
        for r in t5:
            b = before.get((tuple(r["layout"]), r["mode"]))
            md.append(f"| {tuple(r['layout'])} | {r['mode']} | {shape[r['mode'] - 1]} | "
                      + (f"{b['us']} | {b['frac_hbm']} | {b['kernel']} | " if b else "- | - | - | ")
                      + f"{r['us']} | {r['frac_hbm']} | {r['kernel']} |")
        if before:
            fb = sorted(b["frac_hbm"] for b in before.values())
            fa = sorted(r["frac_hbm"] for r in t5)
            md += ["", f"Median {statistics.median(fb):.3f} -> {statistics.median(fa):.3f}, min {fb[0]:.3f} -> {fa[0]:.3f}; "
                   f"largest single gain {max(before[(tuple(r['layout']), r['mode'])]['us'] / r['us'] for r in t5 if (tuple(r['layout']), r['mode']) in before):.1f}x."]
        md.append("")
    v5 = [r for r in rows if r["op"] == "ttv" and r["cfg"] == "cfg5"]
    if v5:
        md += ["## ttv on the config-5 shape, by kernel", "", "| kernel | cases | min | median | max |", "|---|---|---|---|---|"]
        for k in sorted({r["kernel"] for r in v5}):
            fr = sorted(r["frac"] for r in v5 if r["kernel"] == k)
            md.append(f"| {k} | {len(fr)} | {fr[0]:.3f} | {statistics.median(fr):.3f} | {fr[-1]:.3f} |")
        md.append("")
    open(os.path.join(ROOT, "profiles", f"config_sweep_{tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r05")


def layout_sweep_md(tag, seeds=(7, 11)):
    """profiles/layout_sweep_<tag>.md from gpurun_out/layout_sweep_<tag>_<seed>.jsonl (tools/experiments/layout_sweep.py)."""
    import re
    md = [f"# Random-layout ttv sweep ({tag})", "",
          "`tools/experiments/layout_sweep.py 24 SEED`: random order 2-7, extents 2..10^6 with ~512 MB per tensor (float32 /",
          "float64 alternating), random permutation layout, every mode; ttv timed by graph replays; fraction of the pod's",
          "measured HBM copy peak for algorithmic bytes. Same seeds and cases as `layout_sweep_r04.md` (whose 'after' rows are",
          "the start of this comparison).", "",
          "| run | ttvs | p10 | p25 | median | p75 | >= 0.8 | < 0.5 |", "|---|---|---|---|---|---|---|---|"]
    allrows = []
    for sd in seeds:
        path = os.path.join(OUT, f"layout_sweep_{tag}_{sd}.jsonl")
        rows = [json.loads(l) for l in open(path) if '"case"' in l]
        allrows += rows
        fr = sorted(r["frac"] for r in rows)
        q = lambda p: fr[int(p * (len(fr) - 1))]
        md.append(f"| seed {sd} | {len(fr)} | {q(0.1):.3f} | {q(0.25):.3f} | {statistics.median(fr):.3f} | {q(0.75):.3f} | "
                  f"{sum(f >= 0.8 for f in fr)} | {sum(f < 0.5 for f in fr)} |")
    md += ["", "Both seeds, by kernel:", "", "| kernel | ttvs | min | median | max |", "|---|---|---|---|---|"]
    by = {}
    for r in allrows:
        by.setdefault(r["kernel"].split(" ")[0], []).append(r["frac"])
    for k, v in sorted(by.items(), key=lambda kv: -statistics.median(kv[1])):
        v.sort()
        md.append(f"| {k} | {len(v)} | {v[0]:.3f} | {statistics.median(v):.3f} | {v[-1]:.3f} |")
    md.append("")
    open(os.path.join(ROOT, "profiles", f"layout_sweep_{tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))
