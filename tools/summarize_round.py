"""Turn a tools/profile_round.sh session (gpurun_out/) into the committed
evidence under profiles/:

  profiles/bench_<tag>.json          the bench line
  profiles/launches_<tag>.md         ncu launch list: per-kernel count, mean time, share
  profiles/ncu_<tag>.md              --set full summary per captured kernel
  profiles/ncu_summary.json          numbers bench.py reads (traffic per ttv launch)

    python tools/summarize_round.py r01
"""

import csv
import gzip
import json
import os
import re
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name):
    name = re.sub(r"\(tl::\w+\)$", "", name)
    return name.replace("void tl::", "").replace("(bool)", "").replace("(int)", "")


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 12 and r[0] != "ID"]
    agg = OrderedDict()
    for r in rows:
        k = short(r[4])
        t = float(r[14])
        agg.setdefault(k, []).append(t)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list ({tag})", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv "
             "python bench.py --steps 2 --warmup 3 --no-components --no-cpu --no-e2e` "
             "(cold-cache, serialised per launch: compare shares, not absolutes).", "",
             "| kernel | launches | mean us | share of device time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / total:.1f}% |")
    lines.append("")
    ours = sum(len(v) for k, v in agg.items() if "at::" not in k)
    other = sum(len(v) for k, v in agg.items() if "at::" in k)
    lines.append(f"Total launches: {ours + other}; {ours} are this repo's kernels"
                 + (f", {other} one-time torch fill (zero-initialised reduce workspace)." if other else "."))
    open(os.path.join(PROF, f"launches_{tag}.md"), "w").write("\n".join(lines) + "\n")
    return agg


def details(name):
    path = os.path.join(OUT, f"{name}_details.csv")
    if not os.path.exists(path):
        return {}
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    out = OrderedDict()
    for r in rows[1:]:
        kid = (r[idx["ID"]], short(r[idx["Kernel Name"]]))
        out.setdefault(kid, OrderedDict())[r[idx["Metric Name"]]] = (r[idx["Metric Value"]], r[idx["Metric Unit"]])
    return out


def raw(name):
    path = os.path.join(OUT, f"{name}_raw.csv.gz")
    if not os.path.exists(path):
        return []
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[0]
    units = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[idx["Kernel Name"]])}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
                    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"):
            col = idx.get(key)
            if col is None:  # some sections prefix the metric name (e.g. "TPC.TriageCompute.")
                col = next((i for h, i in idx.items() if h.endswith("." + key)), None)
            if col is not None:
                v, u = r[col], units[col]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    continue
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1e-6, "ms": 1e-3,
                         "ns": 1e-9, "s": 1.0}.get(u, 1.0)
                d[key] = v * scale if u in ("Gbyte", "Mbyte", "Kbyte", "byte", "us", "ms", "ns", "s") else v
        res.append(d)
    return res


def stall_summary(name, top=6):
    path = os.path.join(OUT, f"{name}_source.csv.gz")
    if not os.path.exists(path):
        return {}
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import io

    from ncu_summarize import blocks

    out = OrderedDict()
    for kname, lines in blocks(path):
        k = short(kname)
        if k in out:
            continue
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        idx = {h: i for i, h in enumerate(hdr)}
        cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = defaultdict(float)
        sass = defaultdict(int)
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            for c in cols:
                try:
                    tot[c] += float(r[idx[c]] or 0)
                except ValueError:
                    pass
            op = r[idx["Source"]].strip().split(" ")
            op = [o for o in op if o and not o.startswith("@")]
            if op:
                m = op[0].split(".")[0]
                if m in ("DMMA", "UBLKCP", "LDGSTS", "SYNCS", "DADD", "DFMA", "DMUL", "LDS", "LDG", "UTMALDG"):
                    sass[m] += 1
        s = sum(tot.values()) or 1.0
        out[k] = {"stalls": {c: round(100 * v / s, 1) for c, v in sorted(tot.items(), key=lambda x: -x[1])[:top]},
                  "sass_mnemonics": dict(sass)}
    return out


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    line = open(os.path.join(OUT, "bench_line.json")).read().strip()
    json.loads(line)
    open(os.path.join(PROF, f"bench_{tag}.json"), "w").write(line + "\n")
    agg = launches(tag)
    md = [f"# ncu --set full summary ({tag})", ""]
    summary = {"tag": tag}
    ttv_dram = []
    names = sorted(f[:-len("_details.csv")] for f in os.listdir(OUT) if f.startswith("prof_") and
                   f.endswith("_details.csv"))
    for name in names:
        det = details(name)
        rw = raw(name)
        st = stall_summary(name)
        md.append(f"## {name}")
        md.append("")
        md.append("| id | kernel | duration | DRAM thru | SM thru | IPC | regs | dram read | dram write |")
        md.append("|---|---|---|---|---|---|---|---|---|")
        for n, ((kid, k), m) in enumerate(det.items()):
            g = lambda key: " ".join(m.get(key, ("-", ""))).strip()
            r = rw[n] if n < len(rw) else {}
            rd = r.get("dram__bytes_read.sum")
            wr = r.get("dram__bytes_write.sum")
            md.append(f"| {kid} | `{k}` | {g('Duration')} | {g('DRAM Throughput')} | {g('Compute (SM) Throughput')} | "
                      f"{g('Executed Ipc Active')} | {g('Registers Per Thread')} | "
                      f"{rd / 1e6 if rd else float('nan'):.1f} MB | {wr / 1e6 if wr else float('nan'):.1f} MB |")
            if name == "prof_ttv" and rd is not None and wr is not None:
                ttv_dram.append(rd + wr)
        for n, ((kid, k), m) in enumerate(det.items()):
            r = rw[n] if n < len(rw) else {}
            dm = r.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
            tp = r.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
            if dm:
                extra = ""
                t = r.get("gpu__time_duration.sum")
                if name == "prof_ttm" and t:  # config-3 GETT: 2 * 512^3 * 384 flops per launch
                    extra = f", {2 * 512 ** 3 * 384 / t / 1e12:.2f} FP64 TFLOP/s (cold, serialised)"
                md.append(f"- id {kid} DMMA pipe: {dm:.1f}% of peak DMMA issue, tensor pipe active "
                          f"{tp if tp is not None else float('nan'):.1f}% of elapsed{extra}")
        md.append("")
        for k, v in st.items():
            md.append(f"- `{k}` stalls: " + ", ".join(f"{c[6:]} {p}%" for c, p in v["stalls"].items()))
            md.append(f"  SASS evidence: {v['sass_mnemonics']}")
        md.append("")
    if ttv_dram:
        summary["ttv_dram_bytes_per_launch"] = sum(ttv_dram) / len(ttv_dram)
        summary["ttv_launches_captured"] = len(ttv_dram)
    open(os.path.join(PROF, f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    json.dump(summary, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print(open(os.path.join(PROF, f"ncu_{tag}.md")).read())
    print(open(os.path.join(PROF, f"launches_{tag}.md")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
