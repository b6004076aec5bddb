#!/bin/bash
# ncu --set full capture of one cooperative kernel launch on the GPU box, exported to
# small CSV pages (raw metrics, details, source hot spots) so gpurun_out stays small.
#   tools/ncu_capture.sh NAME ARGS...   (ARGS: the profiled command, e.g. python tools/prof_bfs.py --flags 2)
set -u
name=$1; shift
mkdir -p /tmp/ncu gpurun_out
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 2 -c 1 -o /tmp/ncu/$name "$@" > gpurun_out/${name}_run.log 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/${name}_src.csv 2>/dev/null
head -c 4000000 /tmp/ncu/${name}_src.csv > gpurun_out/${name}_source_head.csv
