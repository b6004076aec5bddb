set -u
mkdir -p gpurun_out
for pol in never scheduler; do
  COOP_LIB=${COOP_LIB:-paper_1707_01989_b200/libcoop.so} ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 2 -c 1 -o /tmp/cmp_$pol python tools/prof_bfs.py --policy $pol --src 0 --warm 2 --n 1 > gpurun_out/s11_ncu_$pol.log 2>&1
  ncu -i /tmp/cmp_$pol.ncu-rep --page raw --csv > gpurun_out/s11_${pol}_raw.csv 2>/dev/null
  ncu -i /tmp/cmp_$pol.ncu-rep --page details --csv > gpurun_out/s11_${pol}_details.csv 2>/dev/null
done
