# Round 2, GPU call 5 (after the container was re-created): the whole GPU
# suite, smoke, the bench line, its launch list, traffic and --set full.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 3000 python -m pytest tests -q -m gpu --deselect tests/test_gpu_sanitizer.py --durations=15 > gpurun_out/pytest_gpu_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/smoke_r02.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
echo "rc=$?" >> gpurun_out/bench_r02.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_traffic_cfg5_n32768_r02.csv -k regex:"pald_sym|pald_tile|row_rank|rank_layout" python tools/run_once.py --config 5 --iters 1 > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pald_sym|pald_tile_kernel" -c 3 -o gpurun_out/ncu_cfg3_r02 python tools/run_once.py --config 3 --iters 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pald_sym|pald_tile_kernel" -c 4 -o gpurun_out/ncu_cfg2_r02 python tools/run_once.py --config 2 --alg triplet --iters 1 > gpurun_out/ncu_full2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py -q -m gpu -rs > gpurun_out/pytest_sanitizer_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_sanitizer_r02.txt
ls -la gpurun_out
