"""The C-ABI library loads (no GPU needed) and exports every symbol that
include/layerswap_b200.h declares."""
import ctypes
import re
from pathlib import Path

from paper_2605_11678_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "layerswap_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.library_path()))
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_channel():
    lib = _native.lib()
    assert lib.ls_version().decode() == "0.1.0"
    rc = lib.ls_interleaved_indices(5, 1, (ctypes.c_int64 * 5)())
    assert rc == _native.LS_ERR_VALUE
    assert "layers >= 2" in lib.ls_last_error().decode()


def test_kernel_args_layout_matches_binding():
    """The ctypes mirrors of csrc/kernels.h's argument blocks have the library's sizes
    (kernels._lib() refuses a stale library the same way)."""
    from paper_2605_11678_b200 import kernels

    lib = kernels._lib()
    for kind, st in enumerate((kernels.GemvArgs, kernels.DecodeAttnArgs, kernels.FlashArgs)):
        assert lib.ls_k_args_size(kind) == ctypes.sizeof(st), st.__name__
    assert lib.ls_k_args_size(7) == -1
