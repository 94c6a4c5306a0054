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
        Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T)
