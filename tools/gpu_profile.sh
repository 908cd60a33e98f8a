#!/bin/bash
# Standard GPU evidence pass (run under gpurun): the full bench line, the launch list of the bench command
# and one full ncu capture of the SpMV kernel.
#   bash tools/gpu_profile.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/launches_${TAG}.log 2>&1
echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 5 -c 1 \
  -o gpurun_out/prof_spmv_${TAG} python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
