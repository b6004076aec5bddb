#!/bin/bash
# End-of-session evidence on the GPU box: GPU tests, the bench line, ncu captures of the dominant
# kernel (direction-optimising and top-down), the launch list of a quick bench, the C4 barrier sweep,
# the paper-preset multitask grid and Table 3.  Everything lands in gpurun_out/${TAG}_*.
#   bash tools/round_artifacts.sh TAG
set -u
T=${1:-r02g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gputests.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 bash tools/ncu_capture.sh ${T}_ncu_bfs_diropt python tools/prof_bfs.py --flags 2
timeout 600 bash tools/ncu_capture.sh ${T}_ncu_bfs_topdown python tools/prof_bfs.py --flags 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"coop_kernel|ctl_init" -c 400 --csv \
    --log-file gpurun_out/${T}_launches_bench_quick.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu \
    > gpurun_out/${T}_launches_run.log 2>&1
timeout 900 python tools/sweep.py c4 > gpurun_out/${T}_c4_barrier_sweep.log 2>&1
timeout 900 python tools/multitask_paper.py --cells all > gpurun_out/${T}_multitask_paper_grid.jsonl 2> gpurun_out/${T}_multitask.err
timeout 600 python tools/preemption_compare.py > gpurun_out/${T}_preemption_table3.jsonl 2> gpurun_out/${T}_preemption.err
echo done > gpurun_out/${T}_done.txt
