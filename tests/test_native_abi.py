"""The C-ABI boundary: libspx.so loads on a CPU-only box and exports every symbol declared in
include/spx.h; the ctypes binding covers exactly that set; no torch types cross the ABI; the
product package never imports the oracle; the executor refuses to run without CUDA."""

import ast
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spx.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(spx_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_19913_b200 import native

    if not native.lib_path().exists():
        subprocess.run(["make", "-C", ROOT], check=True)
    return native.load()


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_matches_header():
    from paper_2502_19913_b200 import native

    assert sorted(native.SIGNATURES) == declared_symbols()


def test_abi_version_and_error_channel(lib):
    assert lib.spx_abi_version() == 1
    # argument validation happens before any CUDA call, so it works without a GPU
    rc = lib.spx_gemm_bf16(None, None, None, None, None, 0, 32, 32, 32, 32, 32, 0, 0, 0, 0, ctypes.c_float(0), None)
    assert rc == -1
    assert b"non-positive" in lib.spx_last_error()
    rc = lib.spx_attn_fwd(None, None, None, 1, 100, 4, 4, 64, 768, 256, ctypes.c_float(0.1), None)
    assert rc == -1 and b"multiple of 64" in lib.spx_last_error()


def test_no_torch_types_in_header():
    txt = open(HEADER).read()
    assert "torch" not in txt.split("*/", 1)[1].lower() or "at::" not in txt
    assert "Tensor" not in txt


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2502_19913_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), fn
                if isinstance(node, ast.ImportFrom) and node.module:
                    assert node.module.split(".")[0] != "oracle", fn


def test_executor_requires_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2502_19913_b200 import native
    from paper_2502_19913_b200.configs import get_config
    from paper_2502_19913_b200.executor import Trainer

    rc = get_config("C1")
    with pytest.raises(native.NativeError):
        Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split)


def test_argument_validation_of_newer_entry_points(lib):
    """Invalid arguments are rejected before any CUDA call (no GPU needed)."""
    from paper_2502_19913_b200 import native

    P64 = ctypes.c_void_p * 1
    I64 = ctypes.c_int64 * 1
    F1 = ctypes.c_float * 1
    ptrs, ones = P64(None), I64(64)
    rc = lib.spx_gemm_f32_group(0, ptrs, ptrs, ptrs, ones, ones, ones, ones, ones, ones, F1(1.0), 1, 1, None)
    assert rc == -1 and b"1..4 problems" in lib.spx_last_error()
    rc = lib.spx_gemm_f32_group(5, ptrs, ptrs, ptrs, ones, ones, ones, ones, ones, ones, F1(1.0), 1, 1, None)
    assert rc == -1 and b"1..4 problems" in lib.spx_last_error()
    rc = lib.spx_gemm_f32_group(1, ptrs, ptrs, ptrs, I64(64), I64(48), I64(64), ones, ones, ones, F1(1.0), 1, 1, None)
    assert rc == -1 and b"N % 32" in lib.spx_last_error()
    rc = lib.spx_add_f32(None, None, ctypes.c_int64(-1), None)
    assert rc == -1 and b"negative" in lib.spx_last_error()
    assert lib.spx_add_f32(None, None, ctypes.c_int64(0), None) == 0
    # attention-backward workspace: D + lse*log2e, plus the causal dS^T tiles on the tcgen05 path
    B, H, T = 2, 4, 512
    nqb = T // 128
    assert native.attn_bwd_ws_floats(B, H, T, 48) == 2 * B * H * T
    assert native.attn_bwd_ws_floats(B, H, T, 64) == 2 * B * H * T + B * H * (nqb * (nqb + 1) // 2) * 128 * 128 // 2
    assert lib.spx_launch_count() >= 0


def test_peer_hop_argument_validation(lib):
    """The NVLink peer-hop entry points reject bad arguments before touching CUDA."""
    P = ctypes.c_void_p
    rc = lib.spx_hop_push(P(16), P(32), ctypes.c_int64(24), P(64), 32, None)   # not a multiple of 16
    assert rc == -1 and b"bad size" in lib.spx_last_error()
    rc = lib.spx_hop_push(P(16), P(32), ctypes.c_int64(32), P(64), 0, None)    # no CTAs
    assert rc == -1 and b"bad size" in lib.spx_last_error()
    rc = lib.spx_hop_push(P(16), P(0), ctypes.c_int64(32), P(64), 8, None)     # null source
    assert rc == -1 and b"null" in lib.spx_last_error()
    rc = lib.spx_hop_push(P(24), P(32), ctypes.c_int64(32), P(64), 8, None)    # misaligned destination
    assert rc == -1 and b"aligned" in lib.spx_last_error()
    assert lib.spx_hop_wait(None, ctypes.c_uint32(1), None) == -1
    off = ctypes.c_int64(0)
    assert lib.spx_ipc_export(None, ctypes.create_string_buffer(64), ctypes.byref(off)) == -1
    assert lib.spx_ipc_open(None, None) == -1
    lib.spx_hop_set_timeout.argtypes = [ctypes.c_double]
    assert lib.spx_hop_set_timeout(0.0) == -1 and b"seconds" in lib.spx_last_error()
    assert lib.spx_hop_set_timeout(-5.0) == -1
    assert lib.spx_hop_set_timeout(120.0) == 0
