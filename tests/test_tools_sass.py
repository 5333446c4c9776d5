"""tools/sass_patch.py / tools/sass_reuse.py (the SASS-level operand-reuse
study): the control-word fields are edited in place,
instruction bytes and order stay, and only the selected loop's reuse flags
change. Runs on CPU (nvcc cross-compiles a tiny sm_100a kernel)."""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

SRC = r"""
__global__ void axpy8(float* out, const float* in, int iters) {
  float acc[8], x[8];
  for (int i = 0; i < 8; ++i) { acc[i] = in[i * 32 + threadIdx.x]; x[i] = in[(8 + i) * 32 + threadIdx.x]; }
  const float s = in[16 * 32 + threadIdx.x];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(x[i], s, acc[i]);
  float r = 0.f;
  for (int i = 0; i < 8; ++i) r += acc[i];
  out[threadIdx.x] = r;
}
int main() { return 0; }
"""


@pytest.mark.skipif(shutil.which("nvcc") is None or shutil.which("cuobjdump") is None, reason="CUDA toolkit not present")
def test_reuse_flags_are_rewritten_in_place(tmp_path):
    import sass_patch as sp

    cu = tmp_path / "k.cu"
    cu.write_text(SRC)
    exe = tmp_path / "k"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--no-compress", "-o", str(exe), str(cu)],
                   check=True, capture_output=True)
    funcs = sp.disassemble(str(exe))
    name = next(n for n in funcs if "axpy8" in n)
    ins = funcs[name]
    ffma = [x for x in ins if x.op == "FFMA"]
    assert len(ffma) >= 8
    flagged = sum(1 for x in ffma if x.reuse)
    assert flagged > 0  # ptxas flags the shared multiplier
    # decoded operands: three register sources, one destination
    assert all(len(x.sources()) == 3 and x.dest() is not None for x in ffma)
    for x in ins:
        x.set_reuse(0)
    out = tmp_path / "k_noflags"
    changed = sp.apply(str(exe), str(out), {name: ins})
    assert changed == sum(1 for x in ins if x.hi != x.new_hi) and changed >= flagged
    again = sp.disassemble(str(out))[name]
    assert len(again) == len(ins)
    assert all(a.lo == b.lo and a.op == b.op for a, b in zip(again, ins))  # same instructions, same order
    assert all(a.reuse == 0 for a in again)
    # every other control field untouched
    keep = ~(0xF << 58)
    assert all((a.hi & keep) == (b.hi & keep) for a, b in zip(again, ins))
