#!/bin/bash
# One GPU call: build check, gpu tests, bench, launch list, ncu full of K1 and the Bloom kernels.
# Usage (from the repo root on the GPU box): bash tools/gpu_round.sh TAG [tests|notests]
TAG=${1:-run}; MODE=${2:-tests}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "$MODE" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $O/status
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/status
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "ncu launches exit $?" >> $O/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_minhash -s 8 -c 1 \
  -o $O/k1_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_k1.log 2>&1
echo "ncu k1 exit $?" >> $O/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k[3-6]_" -s 40 -c 4 \
  -o $O/bloom_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_bloom.log 2>&1
echo "ncu bloom exit $?" >> $O/status
