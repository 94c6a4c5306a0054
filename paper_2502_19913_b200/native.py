"""ctypes binding of libspx.so (the C-ABI declared in include/spx.h).

This is the only way the host reaches the GPU compute path.  There is no fallback: if the
library is missing or a call fails, a :class:`NativeError` is raised.  Arguments cross the
boundary as plain device pointers (``tensor.data_ptr()``), int64 shapes and a raw
``cudaStream_t`` — no torch types in the ABI.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libspx.so"

# (name, argtypes) for every symbol declared in include/spx.h; tests check the export list.
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F = ctypes.c_float

SIGNATURES: dict[str, list] = {
    "spx_abi_version": [],
    "spx_last_error": [],
    "spx_device_sm_count": [],
    "spx_enable_peer_access": [_I32, _I32],
    "spx_hop": [_I32, _P, _I32, _P, _I64, _P],
    "spx_gemm_bf16": [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _F, _P],
}

EPI_BF16, EPI_BF16_RESID, EPI_F32, EPI_SWIGLU = 0, 1, 2, 3


class NativeError(RuntimeError):
    """A libspx call failed (or the library could not be loaded)."""


_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load libspx.so once; raise NativeError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise NativeError(
            f"{_LIB_PATH} is not built; run `make` (or __graft_entry__.build()). "
            "There is no CPU fallback for the executor."
        )
    lib = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_char_p if name == "spx_last_error" else ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().spx_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (rc={rc}): {msg}")


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream) -> int:
    if stream is None:
        import torch

        return int(torch.cuda.current_stream().cuda_stream)
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def gemm(A, B, C, *, M, N, K, lda, ldb, ldc, a_mn=False, b_mn=False, epilogue=EPI_BF16, R=None, C2=None,
         ldc2=0, beta=0.0, stream=None) -> None:
    """D = A·Bᵀ with the layouts/epilogues documented at spx_gemm_bf16 in include/spx.h."""
    rc = load().spx_gemm_bf16(_ptr(A), _ptr(B), _ptr(C), _ptr(R), _ptr(C2), M, N, K, lda, ldb, ldc, ldc2,
                              int(a_mn), int(b_mn), epilogue, float(beta), _stream(stream))
    _check(rc, "spx_gemm_bf16")


def hop(dst, dst_dev: int, src, src_dev: int, nbytes: int, stream=None) -> None:
    _check(load().spx_hop(dst_dev, _ptr(dst), src_dev, _ptr(src), nbytes, _stream(stream)), "spx_hop")


def enable_peer_access(dev: int, peer: int) -> None:
    _check(load().spx_enable_peer_access(dev, peer), "spx_enable_peer_access")
