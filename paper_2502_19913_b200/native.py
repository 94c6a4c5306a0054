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
    "spx_launch_count": [],
    "spx_enable_peer_access": [_I32, _I32],
    "spx_hop": [_I32, _P, _I32, _P, _I64, _P],
    "spx_ipc_export": [_P, _P, _P],
    "spx_ipc_open": [_P, _P],
    "spx_ipc_close": [_P],
    "spx_hop_push": [_P, _P, _I64, _P, _I32, _P],
    "spx_hop_push_ce": [_P, _P, _I64, _P, _P],
    "spx_hop_wait": [_P, ctypes.c_uint32, _P],
    "spx_hop_set_timeout": [ctypes.c_double],
    "spx_comm_unique_id": [_P],
    "spx_comm_init": [_P, _I32, _I32, _P],
    "spx_allreduce": [_P, _P, _I64, _I32, _P],
    "spx_comm_destroy": [_P],
    "spx_gemm_bf16": [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _F, _P],
    "spx_attn_fwd": [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F, _P],
    "spx_attn_bwd_ws_floats": [_I64, _I64, _I64, _I64],
    "spx_attn_bwd_ws_floats_ex": [_I64, _I64, _I64, _I64, _I64],
    "spx_attn_bwd": [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F, _P, _P],
    "spx_gemm_set_workspace": [_P, _I64],
    "spx_gemm_f32_group": [_I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P],
    "spx_gemm_bf16_rope": [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P],
    "spx_gemm_bf16_attn_delta": [_P, _P, _P, _P, _I64, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                                 _P],
    "spx_attn_bwd_ex": [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F, _P, _I32, _P],
    "spx_rmsnorm_fwd": [_P, _P, _P, _P, _I64, _I64, _F, _P],
    "spx_rmsnorm_bwd": [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _P],
    "spx_rmsnorm_ws_floats": [_I64, _I64],
    "spx_rope": [_P, _P, _I64, _I64, _I64, _I64, _I64, _I32, _P],
    "spx_swiglu_bwd": [_P, _P, _P, _I64, _I64, _P],
    "spx_embed_fwd": [_P, _P, _P, _I64, _I64, _P],
    "spx_embed_bwd": [_P, _P, _P, _P, _I64, _P, _P, _I64, _P],
    "spx_token_prep": [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P],
    "spx_xent_fwd_bwd": [_P, _P, _P, _I64, _I64, _I64, _F, _P],
    "spx_xent_from_parts": [_P, _P, _I64, _P, _P, _I64, _I64, _I64, _F, _P],
    "spx_sum_f32": [_P, _I64, _P, _F, _I32, _P],
    "spx_add_f32": [_P, _P, _I64, _P],
    "spx_add_f32_clear": [_P, _P, _I64, _P],
    "spx_sumsq_ws_floats": [],
    "spx_sumsq": [_P, _I64, _P, _P, _P],
    "spx_clip_scale": [_P, _I32, _F, _P, _P, _P],
    "spx_adamw": [_P, _P, _P, _P, _P, _I64, _I64, _F, _F, _F, _F, _F, _I64, _P, _P],
    "spx_adamw_clear": [_P, _P, _P, _P, _P, _I64, _I64, _F, _F, _F, _F, _F, _I64, _P, _P],
}
_RESTYPE = {"spx_last_error": ctypes.c_char_p, "spx_rmsnorm_ws_floats": ctypes.c_int64, "spx_launch_count": ctypes.c_int64,
            "spx_attn_bwd_ws_floats": ctypes.c_int64,
            "spx_attn_bwd_ws_floats_ex": ctypes.c_int64,
            "spx_sumsq_ws_floats": ctypes.c_int64}

EPI_BF16, EPI_BF16_RESID, EPI_F32, EPI_SWIGLU = 0, 1, 2, 3
EPI_SWIGLU_BWD = 6
EPI_XENT = 7


# kernel-launch accounting (bench.py "gpu_launches") and GEMM call recording (roofline timing)
_STATS = {"record": False, "gemms": {}, "gemm_log": []}


def launches() -> int:
    """Kernels libspx has launched (or recorded under graph capture) in this process."""
    return int(load().spx_launch_count())


def record_gemms(on: bool) -> None:
    _STATS["record"] = bool(on)


def take_gemm_log() -> list:
    """GEMM keys recorded since the last call (the executor tags them per captured graph)."""
    log = _STATS["gemm_log"]
    _STATS["gemm_log"] = []
    return log


def recorded_gemms() -> dict:
    """(M, N, K, a_mn, b_mn, epilogue) -> (calls recorded, closure re-issuing one such call)."""
    return _STATS["gemms"]


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
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
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
    if _STATS["record"]:
        key = (M, N, K, bool(a_mn), bool(b_mn), int(epilogue))
        cnt = _STATS["gemms"].get(key, (0, None))[0]
        args = (A, B, C)
        kw = dict(M=M, N=N, K=K, lda=lda, ldb=ldb, ldc=ldc, a_mn=a_mn, b_mn=b_mn, epilogue=epilogue, R=R, C2=C2,
                  ldc2=ldc2, beta=beta)

        def again(args=args, kw=kw):
            rec = _STATS["record"]
            _STATS["record"] = False
            try:
                gemm(*args, **kw)
            finally:
                _STATS["record"] = rec

        _STATS["gemms"][key] = (cnt + 1, again)
        _STATS["gemm_log"].append(key)


def gemm_f32_group(problems, *, a_mn=True, b_mn=True, stream=None) -> None:
    """Grouped fp32-accumulating GEMMs in one launch (spx_gemm_f32_group).  problems: list of dicts
    with A, B, C (tensors) and M, N, K, lda, ldb, ldc, beta."""
    k = len(problems)
    P64 = ctypes.c_void_p * k
    I64 = ctypes.c_int64 * k
    arr = lambda key: I64(*[int(p[key]) for p in problems])  # noqa: E731
    rc = load().spx_gemm_f32_group(k, P64(*[_ptr(p["A"]) for p in problems]), P64(*[_ptr(p["B"]) for p in problems]),
                                   P64(*[_ptr(p["C"]) for p in problems]), arr("M"), arr("N"), arr("K"), arr("lda"),
                                   arr("ldb"), arr("ldc"), (ctypes.c_float * k)(*[float(p["beta"]) for p in problems]),
                                   int(a_mn), int(b_mn), _stream(stream))
    _check(rc, "spx_gemm_f32_group")
    if _STATS["record"]:
        key = ("group", tuple((int(p["M"]), int(p["N"]), int(p["K"])) for p in problems), bool(a_mn), bool(b_mn))
        cnt = _STATS["gemms"].get(key, (0, None))[0]

        def again(pr=list(problems), kw=dict(a_mn=a_mn, b_mn=b_mn)):
            rec = _STATS["record"]
            _STATS["record"] = False
            try:
                gemm_f32_group(pr, **kw)
            finally:
                _STATS["record"] = rec

        _STATS["gemms"][key] = (cnt + 1, again)
        _STATS["gemm_log"].append(key)


def gemm_rope(A, B, C, *, M, N, K, lda, ldb, ldc, cos_sin, rope_cols, T, head_dim, stream=None) -> None:
    """QKV projection with RoPE fused into the epilogue (spx_gemm_bf16_rope)."""
    _check(load().spx_gemm_bf16_rope(_ptr(A), _ptr(B), _ptr(C), M, N, K, lda, ldb, ldc, _ptr(cos_sin), rope_cols, T,
                                     head_dim, _stream(stream)), "spx_gemm_bf16_rope")
    if _STATS["record"]:
        key = (M, N, K, False, False, 4)
        cnt = _STATS["gemms"].get(key, (0, None))[0]

        def again(a=(A, B, C), kw=dict(M=M, N=N, K=K, lda=lda, ldb=ldb, ldc=ldc, cos_sin=cos_sin,
                                        rope_cols=rope_cols, T=T, head_dim=head_dim)):
            rec = _STATS["record"]
            _STATS["record"] = False
            try:
                gemm_rope(*a, **kw)
            finally:
                _STATS["record"] = rec

        _STATS["gemms"][key] = (cnt + 1, again)
        _STATS["gemm_log"].append(key)


def gemm_set_workspace(partials) -> None:
    """Register the split-K partials buffer (fp32 device tensor) for the current device; None disables split-K."""
    _check(load().spx_gemm_set_workspace(_ptr(partials), 0 if partials is None else partials.numel()),
           "spx_gemm_set_workspace")


def hop(dst, dst_dev: int, src, src_dev: int, nbytes: int, stream=None) -> None:
    _check(load().spx_hop(dst_dev, _ptr(dst), src_dev, _ptr(src), nbytes, _stream(stream)), "spx_hop")


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding tensor ``t``, byte offset of ``t`` in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _check(load().spx_ipc_export(_ptr(t), h, ctypes.byref(off)), "spx_ipc_export")
    return h.raw, int(off.value)


def ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation; returns its base address in this process."""
    base = ctypes.c_void_p(0)
    _check(load().spx_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(base)), "spx_ipc_open")
    return int(base.value)


def ipc_close(base: int) -> None:
    _check(load().spx_ipc_close(ctypes.c_void_p(base)), "spx_ipc_close")


def hop_push(dst_addr: int, src, nbytes: int, flag_addr: int, ctas: int, stream=None) -> None:
    _check(load().spx_hop_push(ctypes.c_void_p(dst_addr), _ptr(src), nbytes, ctypes.c_void_p(flag_addr), ctas,
                               _stream(stream)), "spx_hop_push")


def hop_push_ce(dst_addr: int, src, nbytes: int, flag_addr: int, stream=None) -> None:
    """Copy-engine hop into a peer-mapped buffer, then +1 on the peer-mapped flag (0: no flag)."""
    _check(load().spx_hop_push_ce(ctypes.c_void_p(dst_addr), _ptr(src), nbytes, ctypes.c_void_p(flag_addr),
                                  _stream(stream)), "spx_hop_push_ce")


DTYPE_F32, DTYPE_BF16 = 0, 1


def comm_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (one rank creates it and broadcasts it to its group)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().spx_comm_unique_id(buf), "spx_comm_unique_id")
    return buf.raw


def comm_init(uid: bytes, nranks: int, rank: int) -> int:
    """Join an NCCL group (libspx-owned communicator); returns the communicator handle."""
    if len(uid) != 128:
        raise NativeError("comm_init: the unique id must be 128 bytes")
    out = ctypes.c_void_p()
    _check(load().spx_comm_init(ctypes.create_string_buffer(uid, 128), nranks, rank, ctypes.byref(out)),
           "spx_comm_init")
    return out.value


def allreduce(comm: int, buf, count: int | None = None, stream=None) -> None:
    """In-place sum of a flat fp32 / bf16 device tensor over the communicator's group."""
    import torch

    dt = {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16}.get(buf.dtype)
    if dt is None:
        raise NativeError(f"allreduce: unsupported dtype {buf.dtype}")
    n = buf.numel() if count is None else count
    _check(load().spx_allreduce(ctypes.c_void_p(comm), _ptr(buf), n, dt, _stream(stream)), "spx_allreduce")


def comm_destroy(comm: int) -> None:
    _check(load().spx_comm_destroy(ctypes.c_void_p(comm)), "spx_comm_destroy")


def hop_set_timeout(seconds: float) -> None:
    """Process-wide spx_hop_wait timeout (a lost hop traps after it)."""
    _check(load().spx_hop_set_timeout(float(seconds)), "spx_hop_set_timeout")


def hop_wait(flag, target: int, stream=None) -> None:
    """``flag``: a device address (int) or tensor element pointer."""
    addr = flag if isinstance(flag, int) else flag.data_ptr()
    _check(load().spx_hop_wait(ctypes.c_void_p(addr), target & 0xFFFFFFFF, _stream(stream)), "spx_hop_wait")


def enable_peer_access(dev: int, peer: int) -> None:
    _check(load().spx_enable_peer_access(dev, peer), "spx_enable_peer_access")


def attn_fwd(qkv, o, lse, *, B, T, H, Hkv, hd, ld_qkv, ld_o, scale, stream=None) -> None:
    _check(load().spx_attn_fwd(_ptr(qkv), _ptr(o), _ptr(lse), B, T, H, Hkv, hd, ld_qkv, ld_o, float(scale),
                               _stream(stream)), "spx_attn_fwd")


def attn_bwd_ws_floats(B: int, H: int, T: int, hd: int, Hkv: int | None = None) -> int:
    """Workspace of spx_attn_bwd in floats (spx_attn_bwd_ws_floats); with Hkv, the size that also
    allows the GQA-split dK/dV pass (spx_attn_bwd_ws_floats_ex)."""
    if Hkv is not None:
        return int(load().spx_attn_bwd_ws_floats_ex(B, H, Hkv, T, hd))
    return int(load().spx_attn_bwd_ws_floats(B, H, T, hd))


ATTN_DELTA_READY = 1
ATTN_WS_EX = 2


def attn_bwd(qkv, o, dout, lse, delta_ws, dqkv, *, B, T, H, Hkv, hd, ld_qkv, ld_o, scale, rope_cs=None,
             delta_ready=False, stream=None) -> None:
    """delta_ws: fp32 workspace of at least attn_bwd_ws_floats(B, H, T) elements; delta_ready: its D and
    lse*log2e prefix was written by gemm_attn_delta (spx_attn_bwd_ex with SPX_ATTN_DELTA_READY)."""
    need = attn_bwd_ws_floats(B, H, T, hd)
    if delta_ws.numel() < need:
        raise ValueError(f"attn_bwd: workspace needs {need} floats, got {delta_ws.numel()}")
    flags = ATTN_DELTA_READY if delta_ready else 0
    if delta_ws.numel() >= attn_bwd_ws_floats(B, H, T, hd, Hkv):
        flags |= ATTN_WS_EX  # room for the GQA-split dK/dV partials
    _check(load().spx_attn_bwd_ex(_ptr(qkv), _ptr(o), _ptr(dout), _ptr(lse), _ptr(delta_ws), _ptr(dqkv), B, T, H,
                                  Hkv, hd, ld_qkv, ld_o, float(scale), _ptr(rope_cs), flags, _stream(stream)),
           "spx_attn_bwd_ex")


def gemm_attn_delta(A, B, dO, O, lse, delta_ws, *, M, N, K, lda, ldb, ldc, ld_o, batch, T, head_dim,
                    stream=None) -> None:
    """dO = A . B (B MN-major) with the attention backward's D = rowsum(dO*O) per head and lse*log2e
    written into delta_ws's prefix (spx_gemm_bf16_attn_delta); then attn_bwd(..., delta_ready=True)."""
    if delta_ws.numel() < 2 * M * (N // head_dim):
        raise ValueError("gemm_attn_delta: workspace too small")
    _check(load().spx_gemm_bf16_attn_delta(_ptr(A), _ptr(B), _ptr(dO), _ptr(O), ld_o, _ptr(lse), _ptr(delta_ws), M, N,
                                           K, lda, ldb, ldc, batch, T, head_dim, _stream(stream)),
           "spx_gemm_bf16_attn_delta")


def rmsnorm_fwd(x, g, y, rstd, *, rows, d, eps, stream=None) -> None:
    _check(load().spx_rmsnorm_fwd(_ptr(x), _ptr(g), _ptr(y), _ptr(rstd), rows, d, float(eps), _stream(stream)),
           "spx_rmsnorm_fwd")


def rmsnorm_bwd(x, g, rstd, dy, dres, dx, dg, ws, *, rows, d, stream=None) -> None:
    _check(load().spx_rmsnorm_bwd(_ptr(x), _ptr(g), _ptr(rstd), _ptr(dy), _ptr(dres), _ptr(dx), _ptr(dg), _ptr(ws),
                                  rows, d, _stream(stream)), "spx_rmsnorm_bwd")


def rmsnorm_ws_floats(rows: int, d: int) -> int:
    return int(load().spx_rmsnorm_ws_floats(rows, d))


def rope(qkv, cos_sin, *, rows, T, n_heads, hd, ld, inverse=False, stream=None) -> None:
    _check(load().spx_rope(_ptr(qkv), _ptr(cos_sin), rows, T, n_heads, hd, ld, int(inverse), _stream(stream)),
           "spx_rope")


def swiglu_bwd(gu, dh, dgu, *, rows, F, stream=None) -> None:
    _check(load().spx_swiglu_bwd(_ptr(gu), _ptr(dh), _ptr(dgu), rows, F, _stream(stream)), "spx_swiglu_bwd")


def embed_fwd(ids, table, out, *, n, d, stream=None) -> None:
    _check(load().spx_embed_fwd(_ptr(ids), _ptr(table), _ptr(out), n, d, _stream(stream)), "spx_embed_fwd")


def embed_bwd(perm, seg_start, seg_id, n_segments, max_segments, dout, dtable, *, d, stream=None) -> None:
    """n_segments: int32 device tensor holding the segment count (graph-capturable)."""
    _check(load().spx_embed_bwd(_ptr(perm), _ptr(seg_start), _ptr(seg_id), _ptr(n_segments), int(max_segments),
                                _ptr(dout), _ptr(dtable), d, _stream(stream)), "spx_embed_bwd")


def token_prep(tokens, ids, targets, perm, seg_start, seg_id, n_segments, *, b, T, ld=None, stream=None) -> None:
    """Device-side split of a [b, T+1] int64 token block into ids / targets and the embedding-
    backward grouping (same values as ``embed_segments`` on the host)."""
    _check(load().spx_token_prep(_ptr(tokens), b, T, T + 1 if ld is None else ld, _ptr(ids), _ptr(targets), _ptr(perm),
                                 _ptr(seg_start), _ptr(seg_id), _ptr(n_segments), _stream(stream)), "spx_token_prep")


def embed_segments(ids) -> tuple:
    """Host-side grouping of token positions by id for the deterministic embedding backward:
    (perm, seg_start, seg_id, n_segments) as int32 CPU tensors padded to len(ids).  The executor
    computes the same grouping on the device (``token_prep``); this is the tests' reference."""
    import torch

    ids = ids.reshape(-1).to(torch.int64).cpu()
    n = ids.numel()
    perm = torch.argsort(ids * n + torch.arange(n))
    sid = ids[perm]
    uniq, counts = torch.unique_consecutive(sid, return_counts=True)
    seg_start = torch.zeros(n + 1, dtype=torch.int32)
    seg_start[1:len(uniq) + 1] = counts.cumsum(0).to(torch.int32)
    seg_id = torch.zeros(n, dtype=torch.int32)
    seg_id[:len(uniq)] = uniq.to(torch.int32)
    return perm.to(torch.int32), seg_start, seg_id, torch.tensor([len(uniq)], dtype=torch.int32)


def xent_from_parts(logits, parts, targets, row_loss, *, nb, n, V, ld, scale, stream=None) -> None:
    """Cross-entropy from the EPI_XENT head GEMM's (max, sum) partials; dlogits in place if scale."""
    _check(load().spx_xent_from_parts(_ptr(logits), _ptr(parts), nb, _ptr(targets), _ptr(row_loss), n, V, ld,
                                      float(scale), _stream(stream)), "spx_xent_from_parts")


def xent_fwd_bwd(logits, targets, row_loss, *, n, V, ld, scale, stream=None) -> None:
    _check(load().spx_xent_fwd_bwd(_ptr(logits), _ptr(targets), _ptr(row_loss), n, V, ld, float(scale),
                                   _stream(stream)), "spx_xent_fwd_bwd")


def add_f32(dst, src, n, *, clear=False, stream=None) -> None:
    """dst[:n] += src[:n] (fp32); clear=True also zeroes src[:n]."""
    if clear:
        _check(load().spx_add_f32_clear(_ptr(dst), _ptr(src), n, _stream(stream)), "spx_add_f32_clear")
    else:
        _check(load().spx_add_f32(_ptr(dst), _ptr(src), n, _stream(stream)), "spx_add_f32")


def sum_f32(x, n, out, *, scale=1.0, accumulate=False, stream=None) -> None:
    _check(load().spx_sum_f32(_ptr(x), n, _ptr(out), float(scale), int(accumulate), _stream(stream)), "spx_sum_f32")


def sumsq_ws_floats() -> int:
    return int(load().spx_sumsq_ws_floats())


def sumsq(x, n, ws, out, *, stream=None) -> None:
    _check(load().spx_sumsq(_ptr(x), n, _ptr(ws), _ptr(out), _stream(stream)), "spx_sumsq")


def clip_scale(sumsq_vec, count, max_norm, scale_out, norm_out=None, *, stream=None) -> None:
    _check(load().spx_clip_scale(_ptr(sumsq_vec), count, float(max_norm), _ptr(scale_out), _ptr(norm_out),
                                 _stream(stream)), "spx_clip_scale")


def adamw(p, g, m, v, p_bf16, *, n, n_decay, lr, beta1, beta2, eps, weight_decay, step, grad_scale=None,
          clear_grad=False, stream=None) -> None:
    """torch.optim.AdamW step over a flat fp32 set; clear_grad=True zeroes g after reading it."""
    fn = load().spx_adamw_clear if clear_grad else load().spx_adamw
    _check(fn(_ptr(p), _ptr(g), _ptr(m), _ptr(v), _ptr(p_bf16), n, n_decay, float(lr), float(beta1),
              float(beta2), float(eps), float(weight_decay), int(step), _ptr(grad_scale),
              _stream(stream)), "spx_adamw_clear" if clear_grad else "spx_adamw")
