"""CPU-side checks of the C-ABI boundary and host logic (no GPU needed)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "omnisparse.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(omni_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2511_12201_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in omnisparse.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes prototype"
    assert lib.omni_abi_version() == 3


def test_workspace_queries_run_without_gpu():
    from paper_2511_12201_b200 import _lib

    assert _lib.size("omni_kv_probe_workspace", 4, 65536, 128, 256) == 8 * 4 * 256 * 128
    assert _lib.size("omni_probe_mass_workspace", 28, 256) == 8 * 28 * 256 * 258
    assert _lib.size("omni_decode_workspace", 32, 28, 65536, 64, 128, 128) > 0


def test_status_codes_map_to_reference_exceptions():
    from paper_2511_12201_b200 import errors

    pairs = {1: errors.ShapeError, 2: errors.ParameterError, 3: errors.DegenerateRowError,
             4: errors.IntegrityError, 5: errors.LayoutError, 6: errors.DegenerateContextError}
    for code, exc in pairs.items():
        with pytest.raises(exc):
            errors.raise_for_status(code, "omni_x")
    errors.raise_for_status(0, "omni_x")


def test_parameter_validation_without_device():
    """Entry points validate scalars before touching the device (the
    reference's error behaviour: ParameterError / LayoutError)."""
    from paper_2511_12201_b200 import _lib, errors

    with pytest.raises(errors.ParameterError):
        _lib.call("omni_select", None, 4, 4, 2048, 256, 1.5, 0, -1, 0, None, None, None, None, None)
    with pytest.raises(errors.LayoutError):
        _lib.call("omni_kv_probe", None, 0, 4, 2048, 128, 0, 0, 256, None, None, None, None, None)
    with pytest.raises(errors.ParameterError):
        _lib.call("omni_q_score", None, 0, 4, 4, 2048, 128, 1984, 1.0, 1, 256, None, None, None, None, None, None,
                  None, None)
    with pytest.raises(errors.ShapeError):
        _lib.call("omni_sparse_attn_fwd", None, None, None, None, None, None, None, None, 28, 4, 65536, 64, 65536, 0,
                  None, None, None)


def test_sparsity_config_validation():
    from paper_2511_12201_b200.errors import ParameterError
    from paper_2511_12201_b200.pipeline import SparsityConfig

    SparsityConfig()
    for bad in (dict(tau=1.0), dict(tau=-0.1), dict(p=0.0), dict(p=1.01), dict(block_size=0), dict(granularity="x")):
        with pytest.raises(ParameterError):
            SparsityConfig(**bad)


def test_device_ops_refuse_cpu_tensors():
    """No CPU fallback: ops on host tensors raise instead of computing."""
    import torch

    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.errors import ShapeError

    with pytest.raises(ShapeError):
        ops.kv_probe(torch.zeros(4, 256, 128, dtype=torch.bfloat16), 200, 0, 256)
