#!/bin/bash
# ncu source-level capture of one BFS launch (SASS with line info), to find spills (LDL/STL)
#   COOP_LIB=<variant.so> bash tools/ncu_src_locals.sh NAME [prof_bfs args]
set -u
name=$1; shift
mkdir -p /tmp/ncu gpurun_out
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 2 -c 1 -o /tmp/ncu/$name python tools/prof_bfs.py "$@" > gpurun_out/${name}_run.log 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/${name}_src.csv 2>/dev/null
python - "$name" <<'PY'
import csv, sys
name = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/ncu/{name}_src.csv")))
hdr = rows[0]
out = open(f"gpurun_out/{name}_locals.csv", "w")
w = csv.writer(out)
w.writerow(hdr)
for r in rows[1:]:
    if any(("LDL" in c or "STL" in c) for c in r[:4]):
        w.writerow(r)
out.close()
open(f"gpurun_out/{name}_hdr.txt", "w").write("\n".join(hdr))
PY
