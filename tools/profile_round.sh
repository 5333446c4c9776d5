set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_traffic_cfg5.csv -k regex:"pald_sym|pald_tile|row_rank|rank_layout" python tools/run_once.py --config 5 --iters 1 > gpurun_out/ncu_traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"pald_tile_kernel|row_rank_bins|rank_layout" -c 3 -o gpurun_out/ncu_cfg3_rank python tools/run_once.py --config 3 --iters 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
