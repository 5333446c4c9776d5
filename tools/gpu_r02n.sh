# Round 2, final build: launch list of the bench command, traffic at n = 32768, --set full at configs 3 and 2
# (summaries extracted on the box: the reports together exceed the 64 MiB that comes back).
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_traffic_cfg5_n32768_r02.csv -k regex:"pald_sym|pald_tile|row_rank|rank_layout" python tools/run_once.py --config 5 --iters 1 > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pald_sym|pald_tile_kernel" -c 3 -o /tmp/ncu_cfg3_r02 python tools/run_once.py --config 3 --iters 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_extract.py /tmp/ncu_cfg3_r02.ncu-rep > gpurun_out/ncu_cfg3_n8192_r02.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pald_sym|pald_tile_kernel" -c 5 -o /tmp/ncu_cfg2_r02 python tools/run_once.py --config 2 --alg triplet --iters 1 > gpurun_out/ncu_full2.log 2>&1
python tools/ncu_extract.py /tmp/ncu_cfg2_r02.ncu-rep > gpurun_out/ncu_cfg2_triplet_n4096_r02.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pald_sym" -c 1 -o /tmp/ncu_cfg3_acc_r02 python tools/run_once.py --config 3 --iters 1 --accurate > gpurun_out/ncu_full3.log 2>&1
python tools/ncu_extract.py /tmp/ncu_cfg3_acc_r02.ncu-rep > gpurun_out/ncu_cfg3_accurate_r02.json
cp /tmp/ncu_cfg3_r02.ncu-rep gpurun_out/
for l in base u4 u2b u4b; do echo == $l; L=$PWD/paper_2307_16652_b200/lib/libpald_gpu.so; [ $l != base ] && L=$PWD/tools/ab/libpald_$l.so; PALD_GPU_LIB=$L python tools/time_kernels.py --configs 5:pairwise,3:pairwise --iters 3 --check; done > gpurun_out/rank_loop_variants_r02.txt 2>&1
cat gpurun_out/rank_loop_variants_r02.txt | grep -E "==|cfg|check"
