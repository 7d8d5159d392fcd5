#!/bin/bash
# One GPU-box pass of the round's measurements (run from the repo root under
# gpurun; every output lands in gpurun_out/, summarised into profiles/ here):
#   1. bench.py default line (C3) and the other workloads' lines
#   2. the launch list of the default bench command (ncu, cold, serialised)
#   3. ncu --set full with source of one C3 step-kernel launch
#   4. ncu counters (DRAM bytes, fp64 / all instruction counts) of one launch of
#      the C3 and C5 step kernels and of the C3 reset_kernel
# Every number printed under ncu is a profiler number, never a bench value.
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi -q -d CLOCK > $O/${TAG}_clocks_before.txt 2>&1
timeout 600 python bench.py > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference_arm.json 2> $O/${TAG}_bench_reference_arm.err
for c in c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > $O/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
  -o $O/${TAG}_c3_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-episode \
  > $O/${TAG}_ncu_full.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_fp64.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:step_kernel -s 3 -c 1 --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-episode > $O/${TAG}_counts_c3.csv 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:step_kernel -s 3 -c 1 --csv \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-episode > $O/${TAG}_counts_c5.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:reset_kernel -c 1 --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-episode > $O/${TAG}_counts_reset.csv 2>&1
nvidia-smi -q -d CLOCK > $O/${TAG}_clocks_after.txt 2>&1
ls -la $O
