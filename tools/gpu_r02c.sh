# Round 2, GPU call 3: triplet accurate by default (with the split last
# round), full GPU suite, sanitizers, small-n launch lists, bench.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_gpu_sanitizer.py > gpurun_out/pytest_all.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all.log
for c in 1 2 4; do
  alg=pairwise; [ $c = 2 ] && alg=triplet
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg${c}.csv python tools/run_once.py --config $c --alg $alg --iters 3 > gpurun_out/ncu_cfg$c.log 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -m gpu > gpurun_out/pytest_sanitizer.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_sanitizer.log
echo done
