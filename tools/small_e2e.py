import sys, json
sys.path.insert(0, '.')
import torch, bench
for cfg in (1, 4, 2):
    D, c = bench.make_input(cfg, "cuda", 20230731)
    v, t, _ = bench.e2e_host(c.n, D, 20, 3)
    print(json.dumps({"config": cfg, "n": c.n, "host_call_ms": t * 1e3}))
