# Round 2, GPU call 1: new parity / accurate / multi-device tests, the full
# GPU suite, smoke, and one bench line (regression check of the stage
# release change).
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_accurate.py tests/test_gpu_multi.py tests/test_gpu_reference.py -x -q -m gpu -s > gpurun_out/pytest_new.log 2>&1
echo "new_rc=$?" >> gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_reference.py > gpurun_out/pytest_gpu.log 2>&1
echo "all_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
