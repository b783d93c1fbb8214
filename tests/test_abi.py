"""C-ABI boundary checks that need no GPU: the in-tree library loads and exports every
function include/moe_b200.h declares, and the ctypes binding covers exactly that set."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2603_07685_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "moe_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|long long)\s+(moe_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2603_07685_b200.build import build_lib

        build_lib()
    return ctypes.CDLL(str(_lib.LIB_PATH))


def test_header_declares_the_path():
    names = declared()
    for must in ("moe_router_topk", "moe_router_bwd", "moe_permute_plan", "moe_permute_gather",
                 "moe_combine", "moe_combine_bwd", "moe_gg_fc1_fwd", "moe_gg_fc2_fwd",
                 "moe_gg_fc2_dgrad", "moe_gg_fc1_dgrad", "moe_gg_wgrad", "moe_ep_regroup_map"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), f"{name} declared in moe_b200.h but not exported"


def test_binding_matches_header():
    assert sorted(_lib.exported_symbols()) == declared()


def test_shim_loads_without_gpu():
    assert _lib.load() is not None
    # pure-host queries work without a device
    assert _lib.query("moe_permute_workspace_ints", 64, 2, 8) == 2 * 2 * 8 + 64 * 2


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "missing.so")
    with pytest.raises(_lib.MoEKernelError, match="no CPU fallback"):
        _lib.load()


def _declared_arity():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:int|long long)\s+(moe_\w+)\s*\(([^)]*)\)\s*;", text,
                         flags=re.M | re.S):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_ctypes_signatures_match_header_arity():
    """Every ctypes argtypes list has as many entries as the header declaration has
    parameters (catches ABI drift between include/moe_b200.h and _lib.py)."""
    arity = _declared_arity()
    assert arity, "no declarations parsed"
    for name, argtypes in _lib.SIGNATURES.items():
        assert name in arity, f"{name} bound in _lib.py but not declared"
        assert len(argtypes) == arity[name], (name, len(argtypes), arity[name])
    for name, (argtypes, _) in _lib.QUERIES.items():
        assert len(argtypes) == arity[name], (name, len(argtypes), arity[name])


@pytest.mark.gpu
def test_hbm_write_probe_zeros_exactly_the_range():
    """moe_hbm_write_probe (bench.py's write bound): every mode zeros [dst, dst + bytes) and
    nothing past it, including a non-multiple of the 32 KB bulk chunk; bad arguments fail."""
    import torch

    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for mode in (0, 1, 2):
        for nbytes in (16, 4096, 3 * 32768 + 48, (1 << 22) + 16 * 7):
            buf = torch.full((nbytes // 2 + 64,), 7, dtype=torch.int16, device="cuda")
            assert lib.moe_hbm_write_probe(buf.data_ptr(), nbytes, mode, st) == 0
            torch.cuda.synchronize()
            assert int(buf[: nbytes // 2].abs().sum()) == 0, (mode, nbytes)
            assert bool((buf[nbytes // 2:] == 7).all()), (mode, nbytes)
    buf = torch.zeros((64,), dtype=torch.int16, device="cuda")
    assert lib.moe_hbm_write_probe(buf.data_ptr(), 24, 0, st) != 0      # not a multiple of 16
    assert lib.moe_hbm_write_probe(buf.data_ptr(), 32, 3, st) != 0      # unknown mode
    assert lib.moe_hbm_write_probe(buf.data_ptr() + 8, 32, 0, st) != 0  # misaligned
