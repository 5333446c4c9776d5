"""The reference's binary distance-matrix format on the GPU
(ingest.hpp:214-283; C ABI pald_gpu_read_distance_binary).

``read_distance_binary(path)`` returns the validated, symmetrized fp32 D as
a CUDA tensor (the reference's read_distance_binary followed by
to_real<float>). ``write_matrix_binary`` writes the same layout from host
values (test and tooling helper, mirrors ingest.hpp:218-238).
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np
import torch

from . import _lib
from .api import _raise_for

MAGIC = b"PALD"
VERSION = 1


def write_matrix_binary(path: str, values: np.ndarray, width: int = 8) -> None:
    if width not in (4, 8):
        from .api import ValidationError

        raise ValidationError(f"unsupported binary element width {width}")
    v = np.ascontiguousarray(values, np.float64)
    n = v.shape[0]
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<BBQ", VERSION, width, n))
        f.write((v if width == 8 else v.astype(np.float32)).astype("<f8" if width == 8 else "<f4").tobytes())


def read_binary_header(path: str) -> tuple[int, int]:
    n = C.c_uint64()
    w = C.c_int32()
    _raise_for(_lib.load().pald_gpu_read_binary_header(str(path).encode(), C.byref(n), C.byref(w)))
    return int(n.value), int(w.value)


def read_distance_binary(path: str, device=None, stream=None) -> torch.Tensor:
    n, _ = read_binary_header(path)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((n, n), dtype=torch.float32, device=dev)
    s = (stream or torch.cuda.current_stream(dev)).cuda_stream
    _raise_for(_lib.load().pald_gpu_read_distance_binary(str(path).encode(), out.data_ptr(), n, s))
    return out
