#!/bin/bash
# One GPU call: gpu tests, smoke, bench (both arms), launch list, ncu full of K1 (C3 screened
# kernel) and of the window sweep's K8 (C5 geometry).
# Usage (from the repo root on the GPU box): bash tools/gpu_round.sh TAG [tests|notests]
TAG=${1:-run}; MODE=${2:-tests}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "$MODE" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $O/status
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/status
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/status
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo "bench reference exit $?" >> $O/status
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-hbm --no-secondary \
  > $O/ncu_launch.log 2>&1
echo "ncu launches exit $?" >> $O/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_minhash_scr4 -c 1 \
  -o $O/k1_full python tools/k1_mode_probe.py C3 60000 1 > $O/ncu_k1.log 2>&1
echo "ncu k1 exit $?" >> $O/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k8_sweep -c 1 \
  -o $O/k8_full python tools/sweep_probe.py 4000000 1 > $O/ncu_k8.log 2>&1
echo "ncu k8 exit $?" >> $O/status
