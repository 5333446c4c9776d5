# Round 2: accurate-mode block sweep + config-5 parity test output (printed errors).
mkdir -p gpurun_out; rm -f gpurun_out/acc_sweep_r02.jsonl
for b in 256 1024 4096; do
  PALD_GPU_ACC_BLOCK=$b timeout 600 python tools/acc_sweep.py >> gpurun_out/acc_sweep_r02.jsonl 2>> gpurun_out/acc_sweep.err
done
timeout 900 python -m pytest tests/test_gpu_reference.py -q -m gpu -s > gpurun_out/pytest_reference_r02.txt 2>&1
tail -5 gpurun_out/pytest_reference_r02.txt; cat gpurun_out/acc_sweep_r02.jsonl | cut -c1-300
