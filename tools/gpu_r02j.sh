# Round 2: the whole GPU suite + smoke + bench on the final build.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_gpu_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/smoke_r02.txt
( time timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err ) 2> gpurun_out/bench_r02.time
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err ) 2> gpurun_out/bench_ref_r02.time
tail -4 gpurun_out/pytest_gpu_r02.txt; cat gpurun_out/smoke_r02.txt gpurun_out/bench_r02.time gpurun_out/bench_ref_r02.time
