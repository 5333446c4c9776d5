# Round 2, GPU call: small-n / triplet knob A/B (device-resident phase times).
mkdir -p gpurun_out; rm -f gpurun_out/small_n_r02.jsonl
for env in "" "PALD_GPU_TRI_MARKS=0" "PALD_GPU_TRIPLET_FP32=1" "PALD_GPU_ACC_BLOCK=4096" "PALD_GPU_ACC_BLOCK=512" "PALD_GPU_SPLIT=0"; do
  env $env timeout 300 python tools/small_n.py --config 2 --alg triplet >> gpurun_out/small_n_r02.jsonl 2>> gpurun_out/small_n.err
done
for env in "" "PALD_GPU_RANK=2" "PALD_GPU_COHESION_TILE=32" "PALD_GPU_RANK=2 PALD_GPU_COHESION_TILE=32"; do
  env $env timeout 300 python tools/small_n.py --config 1 >> gpurun_out/small_n_r02.jsonl 2>> gpurun_out/small_n.err
  env $env timeout 300 python tools/small_n.py --config 1 --oneshot >> gpurun_out/small_n_r02.jsonl 2>> gpurun_out/small_n.err
done
for env in "" "PALD_GPU_RANK=2" "PALD_GPU_COHESION_TILE=64"; do
  env $env timeout 300 python tools/small_n.py --config 4 >> gpurun_out/small_n_r02.jsonl 2>> gpurun_out/small_n.err
done
timeout 300 python tools/small_n.py --config 4 --alg triplet >> gpurun_out/small_n_r02.jsonl 2>> gpurun_out/small_n.err
python - <<'PY'
import json
for l in open('gpurun_out/small_n_r02.jsonl'):
    j=json.loads(l)
    print(j.get('config'),j.get('alg'),j.get('env'),{k:round(v,4) for k,v in j.items() if k.endswith('_ms')},(j.get('info') or {}).get('cohesion_kernel'))
PY
tail -3 gpurun_out/small_n.err
