#!/bin/bash
# Per-source-line executed instructions of one BFS launch, for two policies (never / scheduler),
# to find where the scheduler-armed kernel executes more (a -lineinfo build).
#   bash tools/ncu_src_lines.sh TAG
set -u
T=${1:-src}
mkdir -p /tmp/ncu gpurun_out
for pol in never scheduler; do
  ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 2 -c 1 -o /tmp/ncu/${T}_$pol \
      python tools/prof_bfs.py --policy $pol --src 0 --warm 2 --n 1 > gpurun_out/${T}_${pol}_run.log 2>&1
  ncu -i /tmp/ncu/${T}_$pol.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu/${T}_${pol}_cs.csv 2>/dev/null
  python - "$T" "$pol" <<'PY'
import csv, sys, collections
T, pol = sys.argv[1], sys.argv[2]
agg = collections.Counter()
fname, hdr = "?", None
for r in csv.reader(open(f"/tmp/ncu/{T}_{pol}_cs.csv")):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or not r[0]:
        continue
    try:
        agg[f"{fname}:{r[0]}"] += int(float(r[ie] or 0))
    except (ValueError, IndexError):
        pass
with open(f"gpurun_out/{T}_{pol}_lines.csv", "w") as f:
    for k, v in agg.most_common():
        if v:
            f.write(f"{k},{v}\n")
PY
  head -c 3000 /tmp/ncu/${T}_${pol}_cs.csv > gpurun_out/${T}_${pol}_head.csv
done
