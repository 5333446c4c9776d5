"""ctypes binding of the C ABI (include/pald_gpu.h).

This is the only way the Python mirror reaches the GPU: there is no CPU
fallback. If the sm_100a library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from ._build import LIB_PATH

PAIRWISE, TRIPLET = 0, 1
STRICT, INCLUSIVE_SPLIT = 0, 1
FLAG_SKIP_VALIDATION = 1
FLAG_FORCE_EXACT = 2
FLAG_ACCURATE = 4
MAX_DEVICES = 8
EXCHANGE_AUTO, EXCHANGE_PEER, EXCHANGE_NCCL, EXCHANGE_RED = 0, 1, 2, 3
OPTS_V3_SIZE = 48

OK, ERR_VALIDATION, ERR_UNSUPPORTED, ERR_IO, ERR_CUDA, ERR_COMM = 0, 2, 3, 4, 5, 6

# Every symbol include/pald_gpu.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "pald_gpu_opts_init",
    "pald_gpu_last_error",
    "pald_gpu_abi_version",
    "pald_gpu_visible_devices",
    "pald_gpu_cohesion_f32",
    "pald_gpu_cohesion_f32_device",
    "pald_gpu_plan_create",
    "pald_gpu_plan_destroy",
    "pald_gpu_plan_load",
    "pald_gpu_plan_load_host",
    "pald_gpu_plan_focus",
    "pald_gpu_plan_focus_counts",
    "pald_gpu_plan_focus_finish",
    "pald_gpu_plan_cohesion",
    "pald_gpu_plan_cohesion_share",
    "pald_gpu_plan_buffers",
    "pald_gpu_plan_launches",
    "pald_gpu_plan_get_info",
    "pald_gpu_plan_export_buffers",
    "pald_gpu_plan_attach_peers",
    "pald_gpu_plan_detach_peers",
    "pald_gpu_plan_focus_counts_peers",
    "pald_gpu_plan_cohesion_share_peers",
    "pald_gpu_cohesion_f64io_begin",
    "pald_gpu_cohesion_f64io_outputs",
    "pald_gpu_cohesion_f64io_end",
    "pald_gpu_host_prefault",
    "pald_gpu_cohesion_f64io",
    "pald_gpu_release_host_staging",
    "pald_gpu_plan_export_u",
    "pald_gpu_plan_attach_peers_u",
    "pald_gpu_plan_focus_finish_peers",
    "pald_gpu_focus_units",
    "pald_gpu_fill_diagonal",
    "pald_gpu_points_to_distances",
    "pald_gpu_local_depths",
    "pald_gpu_strong_ties",
    "pald_gpu_nearest_neighbors",
    "pald_gpu_normalize_f64",
    "pald_gpu_row_sums_f64",
    "pald_gpu_read_binary_header",
    "pald_gpu_read_distance_binary",
)


class Opts(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("algorithm", C.c_int32),
        ("policy", C.c_int32),
        ("device", C.c_int32),
        ("block", C.c_uint64),
        ("block_focus", C.c_uint64),
        ("block_cohesion", C.c_uint64),
        ("flags", C.c_uint32),
        ("reserved", C.c_uint32),
        ("num_devices", C.c_int32),
        ("devices", C.c_int32 * 8),
        ("exchange_focus", C.c_int32),
        ("exchange_cohesion", C.c_int32),
    ]


class PhaseTimes(C.Structure):
    _fields_ = [
        ("focus_seconds", C.c_double),
        ("cohesion_seconds", C.c_double),
        ("overhead_seconds", C.c_double),
        ("total_seconds", C.c_double),
    ]


class Buffers(C.Structure):
    _fields_ = [
        ("U", C.c_void_p),
        ("W", C.c_void_p),
        ("C", C.c_void_p),
        ("ld", C.c_uint64),
        ("n", C.c_uint64),
        ("tile", C.c_uint64),
        ("tiles_per_dim", C.c_uint64),
        ("exact_path", C.c_int32),
        ("reserved", C.c_int32),
        ("C64", C.c_void_p),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("cohesion_kernel", C.c_int32),
        ("exact_path", C.c_int32),
        ("pair_kernel_ready", C.c_int32),
        ("exact_step_share", C.c_double),
        ("launches", C.c_uint64),
        ("rank_codes", C.c_int32),
        ("pair_kernel_preferred", C.c_int32),
    ]


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


KERNEL_NAMES = {0: "none", 1: "pald_tile_kernel<cohesion,128>", 2: "pald_tile_kernel<cohesion,64>",
                3: "pald_sym_cohesion_kernel"}

_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load libpald_gpu.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    import os

    env = os.environ.get("PALD_GPU_LIB")  # A/B experiments: load another build
    p = Path(path) if path else (Path(env) if env else LIB_PATH)
    if not p.exists():
        try:
            from ._build import build

            build()
        except Exception as e:  # no nvcc on this host
            raise RuntimeError(
                f"{p} is missing and could not be built ({e}); the PaLD engine has no CPU fallback"
            ) from e
    lib = C.CDLL(str(p))
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
    sig = {
        "pald_gpu_opts_init": (None, [C.POINTER(Opts)]),
        "pald_gpu_last_error": (C.c_char_p, []),
        "pald_gpu_abi_version": (i32, []),
        "pald_gpu_visible_devices": (i32, []),
        "pald_gpu_cohesion_f32": (i32, [vp, u64, C.POINTER(Opts), vp, vp, C.POINTER(PhaseTimes)]),
        "pald_gpu_cohesion_f32_device": (i32, [vp, u64, u64, C.POINTER(Opts), vp, u64, vp, u64, vp]),
        "pald_gpu_plan_create": (i32, [u64, C.POINTER(Opts), C.POINTER(vp)]),
        "pald_gpu_plan_destroy": (i32, [vp]),
        "pald_gpu_plan_load": (i32, [vp, vp, u64, vp]),
        "pald_gpu_plan_load_host": (i32, [vp, vp, vp]),
        "pald_gpu_plan_focus": (i32, [vp, vp]),
        "pald_gpu_plan_focus_counts": (i32, [vp, u64, u64, vp]),
        "pald_gpu_plan_focus_finish": (i32, [vp, vp]),
        "pald_gpu_plan_cohesion": (i32, [vp, u64, u64, vp]),
        "pald_gpu_plan_cohesion_share": (i32, [vp, u64, u64, vp]),
        "pald_gpu_plan_get_info": (i32, [vp, C.POINTER(PlanInfo)]),
        "pald_gpu_plan_export_buffers": (i32, [vp, C.POINTER(IpcHandle), C.POINTER(IpcHandle)]),
        "pald_gpu_plan_attach_peers": (i32, [vp, i32, i32, C.POINTER(IpcHandle), C.POINTER(IpcHandle)]),
        "pald_gpu_plan_detach_peers": (i32, [vp]),
        "pald_gpu_plan_focus_counts_peers": (i32, [vp, u64, u64, vp]),
        "pald_gpu_plan_cohesion_share_peers": (i32, [vp, u64, u64, vp]),
        "pald_gpu_cohesion_f64io_begin": (i32, [vp, u64, C.POINTER(Opts), C.POINTER(vp)]),
        "pald_gpu_cohesion_f64io_outputs": (i32, [vp, vp, vp]),
        "pald_gpu_cohesion_f64io_end": (i32, [vp, vp, vp, C.POINTER(PhaseTimes)]),
        "pald_gpu_host_prefault": (i32, [vp, u64]),
        "pald_gpu_cohesion_f64io": (i32, [vp, u64, C.POINTER(Opts), vp, vp, C.POINTER(PhaseTimes)]),
        "pald_gpu_release_host_staging": (i32, []),
        "pald_gpu_plan_export_u": (i32, [vp, C.POINTER(IpcHandle)]),
        "pald_gpu_plan_attach_peers_u": (i32, [vp, C.POINTER(IpcHandle)]),
        "pald_gpu_plan_focus_finish_peers": (i32, [vp, u64, u64, i32, vp]),
        "pald_gpu_plan_buffers": (i32, [vp, C.POINTER(Buffers)]),
        "pald_gpu_plan_launches": (u64, [vp]),
        "pald_gpu_focus_units": (u64, [vp]),
        "pald_gpu_fill_diagonal": (i32, [vp, u64, u64, vp, vp]),
        "pald_gpu_points_to_distances": (i32, [vp, u64, u64, vp, u64, vp]),
        "pald_gpu_local_depths": (i32, [vp, u64, u64, vp, vp, vp]),
        "pald_gpu_strong_ties": (i32, [vp, u64, u64, vp, vp, vp, u64, vp, vp, vp, vp, vp]),
        "pald_gpu_nearest_neighbors": (i32, [vp, u64, u64, vp, u64, u64, vp, vp, vp]),
        "pald_gpu_normalize_f64": (i32, [vp, u64, u64, vp]),
        "pald_gpu_row_sums_f64": (i32, [vp, u64, u64, vp, vp]),
        "pald_gpu_read_binary_header": (i32, [C.c_char_p, C.POINTER(u64), C.POINTER(C.c_int32)]),
        "pald_gpu_read_distance_binary": (i32, [C.c_char_p, vp, u64, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name, None)
        if f is None:  # only possible for an older build loaded via PALD_GPU_LIB
            continue
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().pald_gpu_last_error()
    return msg.decode() if msg else ""


def make_opts(algorithm: int = PAIRWISE, policy: int = STRICT, device: int = -1, block: int = 128,
              block_focus: int = 128, block_cohesion: int = 128, flags: int = 0,
              devices=None, exchange_focus: int = EXCHANGE_AUTO,
              exchange_cohesion: int = EXCHANGE_AUTO) -> Opts:
    """pald_gpu_opts; ``devices`` (a list of ordinals, repeats allowed) runs
    one call across several GPUs (include/pald_gpu.h, ABI v4)."""
    o = Opts()
    load().pald_gpu_opts_init(C.byref(o))
    o.algorithm, o.policy, o.device = algorithm, policy, device
    o.block, o.block_focus, o.block_cohesion, o.flags = block, block_focus, block_cohesion, flags
    if devices is not None:
        devices = list(devices)
        if len(devices) > MAX_DEVICES:
            raise ValueError(f"at most {MAX_DEVICES} devices")
        o.num_devices = len(devices)
        for i, d in enumerate(devices):
            o.devices[i] = int(d)
    o.exchange_focus, o.exchange_cohesion = exchange_focus, exchange_cohesion
    return o
