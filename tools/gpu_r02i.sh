# Round 2: pipelined f64io (shim) checks: shim tests, acceptance corpus, multi-device shim, then shim_bench at n = 32768.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_shim.py tests/test_gpu_multi.py tests/test_abi.py "tests/test_gpu_reference.py::test_reference_acceptance_corpus_through_shim" -q -m gpu -x 2>&1 | tail -4
python - <<'PY'
import json, sys
sys.path.insert(0, '.')
import bench
from paper_2307_16652_b200 import datagen
cfg = datagen.config(5)
print(json.dumps(bench.shim_e2e(cfg, 20230731, 2, 1)))
cfg3 = datagen.config(1)
print(json.dumps(bench.shim_e2e(cfg3, 20230731, 3, 1)))
PY
