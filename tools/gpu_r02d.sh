# Round 2, GPU call 4: accurate-mode block sweep, ncu of the accurate pair
# kernel, small-n / triplet knob A/B.
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_accurate.py -q -m gpu -k "tie_marks" > gpurun_out/pytest_marks.log 2>&1
for b in 256 1024 4096; do
  PALD_GPU_ACC_BLOCK=$b timeout 600 python tools/acc_sweep.py >> gpurun_out/acc_sweep.jsonl 2>> gpurun_out/acc_sweep.err
done
for env in "" "PALD_GPU_RANK=2" "PALD_GPU_COHESION_TILE=32" "PALD_GPU_RANK=2 PALD_GPU_COHESION_TILE=32"; do
  env $env timeout 300 python tools/small_n.py --config 1 >> gpurun_out/small_n.jsonl 2>> gpurun_out/small_n.err
done
for env in "" "PALD_GPU_RANK=2"; do
  env $env timeout 300 python tools/small_n.py --config 4 >> gpurun_out/small_n.jsonl 2>> gpurun_out/small_n.err
done
for env in "" "PALD_GPU_TRI_MARKS=0" "PALD_GPU_TRIPLET_FP32=1" "PALD_GPU_TRIPLET_FP32=1 PALD_GPU_TRI_MARKS=0" "PALD_GPU_ACC_BLOCK=1024"; do
  env $env timeout 300 python tools/small_n.py --config 2 --alg triplet >> gpurun_out/small_n.jsonl 2>> gpurun_out/small_n.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pald_sym -c 1 -o gpurun_out/ncu_acc_cfg3 python tools/run_once.py --config 3 --iters 1 --accurate > gpurun_out/ncu_acc.log 2>&1
echo done
