# accurate-mode block length at n = 32768: error (72 rows vs fp64) and step time
mkdir -p gpurun_out; rm -f gpurun_out/acc_block_cfg5_r02.txt
for b in 1024 2048 4096 8192; do
  echo "== PALD_GPU_ACC_BLOCK=$b" >> gpurun_out/acc_block_cfg5_r02.txt
  PALD_GPU_ACC_BLOCK=$b timeout 900 python -m pytest tests/test_gpu_reference.py -q -m gpu -s -k cfg5_rows 2>&1 | grep -E "cfg5 rows|passed|failed" >> gpurun_out/acc_block_cfg5_r02.txt
  PALD_GPU_ACC_BLOCK=$b timeout 600 python tools/small_n.py --config 5 --iters 2 --accurate 2>&1 | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:round(v,2) for k,v in j.items() if k.endswith('_ms')})" >> gpurun_out/acc_block_cfg5_r02.txt
done
cat gpurun_out/acc_block_cfg5_r02.txt
