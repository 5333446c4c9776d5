# Round 2, GPU call 2: accurate mode (256-term blocks), analyze pins, full
# reference parity, sharded transports, then a bench line (anchor, shim_e2e).
set -x
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 1200 python -m pytest tests/test_gpu_accurate.py tests/test_gpu_analyze.py tests/test_gpu_multi.py tests/test_gpu_sharded.py -q -m gpu > gpurun_out/pytest_b1.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_b1.log
timeout 1500 python -m pytest tests/test_gpu_reference.py -q -m gpu -s > gpurun_out/pytest_ref.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ref.log
timeout 600 python -m pytest tests/test_gpu_bench.py -q -m gpu > gpurun_out/pytest_bench.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_bench.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
