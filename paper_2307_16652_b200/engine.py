"""Device-resident engine: a staged plan over the C ABI, with torch as the
memory/stream plumbing.

``Engine`` wraps ``pald_gpu_plan`` (include/pald_gpu.h). Its buffers are
exposed to torch as zero-copy views through ``__cuda_array_interface__`` so
that torch.distributed (NCCL) can reduce/gather them in the multi-GPU
driver (paper_2307_16652_b200.distributed).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .api import _raise_for


class _DeviceView:
    """Minimal __cuda_array_interface__ exporter over plan-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str, strides, owner):
        self._owner = owner  # keeps the plan alive while a view exists
        self.__cuda_array_interface__ = {
            "shape": tuple(shape),
            "typestr": typestr,
            "data": (int(ptr), False),
            "strides": tuple(strides),
            "version": 3,
        }


class Engine:
    """One PaLD problem of size n on one GPU.

    Steps (each asynchronous on ``stream`` unless noted):
      load(D)                 validate + range check (one small sync) + layout
      focus()                 pass 1: U and W = 1/U
        = focus_counts(part, parts) + focus_finish()   (multi-GPU split)
      cohesion(r0, r1)        pass 2 over C rows [r0, r1)
      cohesion_share(p, q)    pass 2, share p of q into a zeroed C (multi-GPU:
                              the SUM of the q buffers is the full C)
    Views: ``U``, ``W``, ``C`` (n x n, strided by ld).
    """

    def __init__(self, n: int, algorithm: str = "pairwise", device: int | None = None,
                 force_exact: bool = False, skip_validation: bool = False, policy: str = "strict",
                 accurate: bool = False):
        self.lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.n = int(n)
        self.algorithm = algorithm
        alg = {"pairwise": _lib.PAIRWISE, "triplet": _lib.TRIPLET}[algorithm]
        flags = (_lib.FLAG_FORCE_EXACT if force_exact else 0) | (
            _lib.FLAG_SKIP_VALIDATION if skip_validation else 0) | (_lib.FLAG_ACCURATE if accurate else 0)
        pol = {"strict": _lib.STRICT, "split": _lib.INCLUSIVE_SPLIT}[policy]
        opts = _lib.make_opts(algorithm=alg, policy=pol, device=self.device, flags=flags)
        self._plan = C.c_void_p()
        _raise_for(self.lib.pald_gpu_plan_create(self.n, C.byref(opts), C.byref(self._plan)))
        b = _lib.Buffers()
        _raise_for(self.lib.pald_gpu_plan_buffers(self._plan, C.byref(b)))
        self.ld = int(b.ld)
        self.tile = int(b.tile)
        self.tiles_per_dim = int(b.tiles_per_dim)
        self._ptrs = (b.U, b.W, b.C)

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            self.lib.pald_gpu_plan_destroy(plan)
            self._plan = None

    # -- views ---------------------------------------------------------
    def _view(self, ptr: int, typestr: str, dtype) -> torch.Tensor:
        n, ld = self.n, self.ld
        v = _DeviceView(ptr, (n, n), typestr, (ld * 4, 4), self)
        return torch.as_tensor(v, device=f"cuda:{self.device}")

    @property
    def U(self) -> torch.Tensor:
        return self._view(self._ptrs[0], "<i4", torch.int32)

    @property
    def W(self) -> torch.Tensor:
        return self._view(self._ptrs[1], "<f4", torch.float32)

    @property
    def C(self) -> torch.Tensor:
        return self._view(self._ptrs[2], "<f4", torch.float32)

    @property
    def C64(self) -> torch.Tensor:
        """Accurate mode's double sums (n x n), after an accurate cohesion call."""
        b = _lib.Buffers()
        _raise_for(self.lib.pald_gpu_plan_buffers(self._plan, C.byref(b)))
        if not b.C64:
            raise RuntimeError("no accurate-mode cohesion has run on this engine")
        n, ld = self.n, self.ld
        v = _DeviceView(b.C64, (n, n), "<f8", (ld * 8, 8), self)
        return torch.as_tensor(v, device=f"cuda:{self.device}")

    def full_U(self) -> torch.Tensor:
        """The whole ld-strided U buffer as a flat tensor (for collectives)."""
        v = _DeviceView(self._ptrs[0], (self.n * self.ld,), "<i4", (4,), self)
        return torch.as_tensor(v, device=f"cuda:{self.device}")

    def full_W(self) -> torch.Tensor:
        v = _DeviceView(self._ptrs[1], (self.n * self.ld,), "<f4", (4,), self)
        return torch.as_tensor(v, device=f"cuda:{self.device}")

    def row_block_C(self, r0: int, r1: int) -> torch.Tensor:
        v = _DeviceView(self._ptrs[2] + r0 * self.ld * 4, ((r1 - r0) * self.ld,), "<f4", (4,), self)
        return torch.as_tensor(v, device=f"cuda:{self.device}")

    # -- steps -----------------------------------------------------------
    def _stream(self, stream) -> int:
        """The raw handle of `stream`, or of the current stream OF THIS
        ENGINE'S DEVICE (the C ABI switches to the plan's device)."""
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        elif stream.device.index is not None and stream.device.index != self.device:
            raise ValueError(f"stream of {stream.device} used with an engine on cuda:{self.device}")
        return stream.cuda_stream

    def load(self, D: torch.Tensor, stream=None) -> None:
        if D.dtype != torch.float32 or not D.is_cuda or D.dim() != 2:
            raise TypeError("D must be a 2-D float32 CUDA tensor")
        if D.shape[0] != self.n or D.shape[1] != self.n or D.stride(1) != 1:
            raise ValueError("D must be n x n with unit column stride")
        _raise_for(self.lib.pald_gpu_plan_load(self._plan, D.data_ptr(), D.stride(0),
                                               self._stream(stream)))

    def load_host(self, D, stream=None) -> None:
        """D: C-contiguous float32 host array/tensor (pinned for full speed)."""
        ptr = D.data_ptr() if isinstance(D, torch.Tensor) else D.ctypes.data
        _raise_for(self.lib.pald_gpu_plan_load_host(self._plan, ptr, self._stream(stream)))

    def focus(self, stream=None) -> None:
        """Pass 1 over all pairs: U and W = 1/U."""
        _raise_for(self.lib.pald_gpu_plan_focus(self._plan, self._stream(stream)))

    def focus_counts(self, part: int = 0, parts: int = 1, stream=None) -> None:
        """Pass 1, share `part` of `parts` equal shares: counts into W."""
        _raise_for(self.lib.pald_gpu_plan_focus_counts(self._plan, part, parts, self._stream(stream)))

    def focus_finish(self, stream=None) -> None:
        """Counts (W buffer, summed over ranks) -> U and W = 1/U."""
        _raise_for(self.lib.pald_gpu_plan_focus_finish(self._plan, self._stream(stream)))

    @property
    def focus_units(self) -> int:
        return int(self.lib.pald_gpu_focus_units(self._plan))

    def cohesion(self, row_begin: int = 0, row_end: int | None = None, stream=None) -> None:
        if row_end is None:
            row_end = self.n
        _raise_for(self.lib.pald_gpu_plan_cohesion(self._plan, row_begin, row_end,
                                                   self._stream(stream)))

    def cohesion_share(self, part: int = 0, parts: int = 1, stream=None) -> None:
        """Pass 2, share `part` of `parts` (tile pairs or row bands) into a
        zeroed C: every entry is computed by exactly one share."""
        _raise_for(self.lib.pald_gpu_plan_cohesion_share(self._plan, part, parts,
                                                         self._stream(stream)))

    # -- fused multi-GPU exchange over peer memory (include/pald_gpu.h) --
    def export_buffers(self) -> tuple[bytes, bytes]:
        """CUDA IPC handles of this plan's W and C (64 bytes each)."""
        w, c = _lib.IpcHandle(), _lib.IpcHandle()
        _raise_for(self.lib.pald_gpu_plan_export_buffers(self._plan, C.byref(w), C.byref(c)))
        return bytes(w.bytes), bytes(c.bytes)

    def attach_peers(self, rank: int, w_handles: list[bytes], c_handles: list[bytes]) -> None:
        world = len(w_handles)
        arr_t = _lib.IpcHandle * world
        wa, ca = arr_t(), arr_t()
        for q in range(world):
            C.memmove(wa[q].bytes, w_handles[q], 64)
            C.memmove(ca[q].bytes, c_handles[q], 64)
        _raise_for(self.lib.pald_gpu_plan_attach_peers(self._plan, world, rank, wa, ca))

    def export_u(self) -> bytes:
        """CUDA IPC handle of this plan's U (peer-pull finish, ABI v4)."""
        u = _lib.IpcHandle()
        _raise_for(self.lib.pald_gpu_plan_export_u(self._plan, C.byref(u)))
        return bytes(u.bytes)

    def attach_peers_u(self, u_handles: list[bytes]) -> None:
        arr = (_lib.IpcHandle * len(u_handles))()
        for q, h in enumerate(u_handles):
            C.memmove(arr[q].bytes, h, 64)
        _raise_for(self.lib.pald_gpu_plan_attach_peers_u(self._plan, arr))

    def focus_finish_peers(self, part: int, parts: int, u_mode: int = 1, stream=None) -> None:
        """Peer-pull exchange of pass 1: finish share `part` of `parts` of the
        tiles from every rank's counts, storing W everywhere and U per u_mode
        (0 own, 1 every rank, 2 the rank owning the row's tile band)."""
        _raise_for(self.lib.pald_gpu_plan_focus_finish_peers(self._plan, part, parts, int(u_mode),
                                                             self._stream(stream)))

    def pair_kernel_preferred(self) -> bool:
        """Whether a full-range cohesion of the loaded D would run the pair kernel."""
        return bool(self._info().pair_kernel_preferred)

    def detach_peers(self) -> None:
        _raise_for(self.lib.pald_gpu_plan_detach_peers(self._plan))

    def focus_counts_peers(self, part: int, parts: int, stream=None) -> None:
        """Pass 1 share with its counts added into every attached rank's W."""
        _raise_for(self.lib.pald_gpu_plan_focus_counts_peers(self._plan, part, parts,
                                                             self._stream(stream)))

    def cohesion_share_peers(self, part: int, parts: int, stream=None) -> bool:
        """Pass 2 share stored into every attached rank's C; False when the
        pair kernel does not run for this D (caller falls back)."""
        rc = self.lib.pald_gpu_plan_cohesion_share_peers(self._plan, part, parts, self._stream(stream))
        if rc == _lib.ERR_UNSUPPORTED:
            return False
        _raise_for(rc)
        return True

    def _info(self):
        i = _lib.PlanInfo()
        i.struct_size = C.sizeof(_lib.PlanInfo)
        _raise_for(self.lib.pald_gpu_plan_get_info(self._plan, C.byref(i)))
        return i

    def info(self) -> dict:
        """Pass-2 kernel of the last cohesion call and the tie statistics."""
        i = self._info()
        return {"cohesion_kernel": _lib.KERNEL_NAMES.get(i.cohesion_kernel, str(i.cohesion_kernel)),
                "exact_path": bool(i.exact_path), "pair_kernel_ready": bool(i.pair_kernel_ready),
                "exact_step_share": i.exact_step_share, "launches": int(i.launches),
                "rank_codes": bool(i.rank_codes), "pair_kernel_preferred": bool(i.pair_kernel_preferred)}

    def run(self, D: torch.Tensor, stream=None) -> None:
        self.load(D, stream)
        self.focus(stream=stream)
        self.cohesion(stream=stream)

    # -- epilogue: fill_diagonal, depths, strong ties -----
    def fill_diagonal(self, stream=None) -> torch.Tensor:
        """reference.hpp:213-220 on the device: c_xx = sum_{y!=x} 1/u_xy (double)."""
        out = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}")
        _raise_for(self.lib.pald_gpu_fill_diagonal(self._ptrs[0], self.ld, self.n, out.data_ptr(),
                                                   self._stream(stream)))
        return out

    def local_depths(self, diag: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Row sums of the normalized C (reference.hpp:223-241), double."""
        out = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}")
        _raise_for(self.lib.pald_gpu_local_depths(self._ptrs[2], self.ld, self.n,
                                                  diag.data_ptr() if diag is not None else None,
                                                  out.data_ptr(), self._stream(stream)))
        return out

    def strong_ties(self, diag: torch.Tensor | None = None, threshold: float | None = None,
                    stream=None):
        """Strong-tie graph of the normalized C (analyze.hpp:34-53):
        returns (threshold, xs, ys, strength) with edges in row-major order."""
        dev = f"cuda:{self.device}"
        thr_out = torch.empty(1, dtype=torch.float64, device=dev)
        thr_in = (torch.tensor([threshold], dtype=torch.float64, device=dev)
                  if threshold is not None else None)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        st = self._stream(stream)
        dptr = diag.data_ptr() if diag is not None else None
        tptr = thr_in.data_ptr() if thr_in is not None else None
        _raise_for(self.lib.pald_gpu_strong_ties(self._ptrs[2], self.ld, self.n, dptr, tptr,
                                                 thr_out.data_ptr(), 0, None, None, None,
                                                 cnt.data_ptr(), st))
        m = int(cnt.item())
        xs = torch.empty(m, dtype=torch.int32, device=dev)
        ys = torch.empty(m, dtype=torch.int32, device=dev)
        sv = torch.empty(m, dtype=torch.float64, device=dev)
        if m:
            _raise_for(self.lib.pald_gpu_strong_ties(self._ptrs[2], self.ld, self.n, dptr, tptr,
                                                     thr_out.data_ptr(), m, xs.data_ptr(),
                                                     ys.data_ptr(), sv.data_ptr(), cnt.data_ptr(), st))
        return float(thr_out.item()), xs, ys, sv

    def normalized_cohesion(self, diag: torch.Tensor | None = None) -> torch.Tensor:
        """normalize (reference.hpp:223-228) on the device: double(C) * (1/(n-1)),
        the reference's double arithmetic, with an optional fill_diagonal."""
        c = self.C.double()
        if diag is not None:
            c.diagonal().copy_(diag)
        return c * (1.0 / float(self.n - 1))

    def nearest_neighbors(self, focus: int, k: int, diag: torch.Tensor | None = None, stream=None):
        """analyze.hpp:60-75 on the device (pald_gpu_nearest_neighbors): top-k
        points by min(c'_fz, c'_zf), strongest first, ties toward the smaller
        index (stable sort). Returns (z int32, strength float64) tensors."""
        dev = f"cuda:{self.device}"
        kk = max(int(k), 0)
        zs = torch.empty(max(kk, 1), dtype=torch.int32, device=dev)
        sv = torch.empty(max(kk, 1), dtype=torch.float64, device=dev)
        _raise_for(self.lib.pald_gpu_nearest_neighbors(
            self._ptrs[2], self.ld, self.n, diag.data_ptr() if diag is not None else None, int(focus), int(k),
            zs.data_ptr(), sv.data_ptr(), self._stream(stream)))
        return zs[:kk], sv[:kk]

    @property
    def exact_path(self) -> bool:
        b = _lib.Buffers()
        _raise_for(self.lib.pald_gpu_plan_buffers(self._plan, C.byref(b)))
        return bool(b.exact_path)

    @property
    def launches(self) -> int:
        return int(self.lib.pald_gpu_plan_launches(self._plan))


def points_to_distances(points: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Euclidean D of a float64 CUDA point cloud (ingest.hpp:303-322) on the GPU."""
    lib = _lib.load()
    if points.dtype != torch.float64 or not points.is_cuda:
        raise TypeError("points must be a float64 CUDA tensor")
    points = points.contiguous()
    n, dim = points.shape
    if out is None:
        out = torch.empty((n, n), dtype=torch.float32, device=points.device)
    s = (stream or torch.cuda.current_stream(points.device)).cuda_stream
    _raise_for(lib.pald_gpu_points_to_distances(points.data_ptr(), n, dim, out.data_ptr(),
                                                out.stride(0), s))
    return out

