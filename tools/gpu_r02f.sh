# Round 2, GPU call 6: operand-reuse experiments. (1) microbench5 as compiled,
# with every reuse flag cleared, and with extra flags; (2) the pair kernel's
# inner loop with its reuse flags rewritten by tools/sass_reuse.py policies.
set -x
mkdir -p gpurun_out
for b in microbench5 microbench5_noflags microbench5_allflags; do
  echo "== $b" >> gpurun_out/microbench5_r02.txt
  timeout 120 tools/ab/$b >> gpurun_out/microbench5_r02.txt 2>&1
done
for p in base none next pipe hold hold2; do
  echo "== $p" >> gpurun_out/reuse_policies_r02.txt
  PALD_GPU_LIB=$PWD/tools/ab/libpald_$p.so timeout 300 python tools/time_kernels.py --configs 3:pairwise --iters 5 --check >> gpurun_out/reuse_policies_r02.txt 2>&1
done
echo done
