#!/bin/bash
# Cold (ncu flushes caches before each kernel) per-kernel durations of a
# command, summarised per kernel name: tools/ncu_times.sh TAG REGEX CMD...
# -> gpurun_out/TAG_times.csv + a one-line-per-kernel summary on stdout.
set -u
tag=$1; regex=$2; shift 2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none ${NCU_EXTRA:-} \
    -k "regex:${regex}" --csv --log-file gpurun_out/${tag}_times.csv "$@" > gpurun_out/${tag}_cmd.log 2>&1
python - "$tag" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/{tag}_times.csv") if l.startswith('"')))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
acc = collections.OrderedDict()
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    key = (r[idx["ID"]], r[idx["Kernel Name"]][:90])
    acc.setdefault(key, {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
for (i, name), m in acc.items():
    t = m.get("gpu__time_duration.sum", 0)
    rd = m.get("dram__bytes_read.sum", 0)
    print(f"{tag} {i:>4} {t/1e3:9.2f} us  rd {rd/1e6:9.2f} MB  {name}")
PY
