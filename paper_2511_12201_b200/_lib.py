"""ctypes binding of the C ABI in ``include/omnisparse.h`` (libomnisparse.so).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2511_12201_b200/csrc`` into ``paper_2511_12201_b200/lib``.
There is no fallback: if the library is missing or the device is not a
B200 (sm_100), every op raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CudaError, raise_for_status

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
# the product library; OMNI_LIBRARY=<path> selects another build of the same
# ABI (libomnisparse_variants.so: the measured alternative kernels for A/B
# runs and tests/test_gpu_kernel_variants.py)
LIB_PATH = os.environ.get("OMNI_LIBRARY") or os.path.join(LIB_DIR, "libomnisparse.so")

_c_int, _c_double, _c_size, _p = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/omnisparse.h exactly.
SIGNATURES = {
    "omni_abi_version": (_c_int, []),
    "omni_last_error": (ctypes.c_char_p, []),
    "omni_device_check": (_c_int, []),
    "omni_kv_probe_workspace": (_c_size, [_c_int, _c_int, _c_int, _c_int]),
    "omni_kv_probe": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p]),
    "omni_q_score": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _c_int,
                              _p, _p, _p, _p, _p, _p, _p, _p]),
    "omni_compact_rows": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _p, _p, _p]),
    "omni_probe_mass_workspace": (_c_size, [_c_int, _c_int]),
    "omni_probe_mass": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p]),
    "omni_probe_mass_map": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p]),
    "omni_exact_mass_workspace": (_c_size, [_c_int, _c_int]),
    "omni_exact_mass": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p]),
    "omni_select": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _c_int, _c_int,
                             _p, _p, _p, _p, _p]),
    "omni_select_workspace": (_c_size, [_c_int, _c_int, _c_int]),
    "omni_select_ex": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _c_int, _c_int,
                                _p, _p, _p, _p, _p, _p]),
    "omni_top_blocks_workspace": (_c_size, [_c_int, _c_int, _c_int]),
    "omni_top_blocks": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p]),
    "omni_block_sums": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p]),
    "omni_probe_map": (_c_int, [_p, _c_int, _c_int, _p, _p]),
    "omni_gather_rows": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _p, _c_int, _p, _c_int, _p, _c_int,
                                  _c_int, _p]),
    "omni_scatter_rows": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _p, _c_int, _p, _p, _c_int, _p]),
    "omni_scatter_key_grads": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _c_int, _p, _c_int, _p, _p, _c_int, _c_int, _p]),
    "omni_sparse_attn_fwd": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_int, _c_int, _c_int, _c_int, _c_int,
                                      _c_int, _p, _p, _p]),
    "omni_sparse_attn_fwd_ex": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_int, _c_int, _c_int, _c_int, _c_int,
                                         _c_int, _p, _p, _p, _p]),
    "omni_sparse_attn_bwd_workspace": (_c_size, [_c_int, _c_int]),
    "omni_sparse_attn_bwd": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _c_int, _c_int, _c_int, _c_int,
                                      _c_int, _p, _p, _p, _p, _p, _p]),
    "omni_sparse_attn_bwd_ex": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _c_int, _c_int, _c_int, _c_int,
                                         _c_int, _c_int, _p, _p, _p, _p, _p, _p]),
    "omni_decode_workspace": (_c_size, [_c_int, _c_int, _c_int]),
    "omni_decode": (_c_int, [_p, _p, _p, _c_int, _p, _c_int, _p, _p, _p, _c_int, _p, _p, _c_int, _c_int, _c_int,
                             _c_int, _c_double, _c_int, _p, _p, _p, _p, _p, _p]),
    "omni_append_answer": (_c_int, [_p, _p, _p, _p, _p, _c_int, _p, _p, _p, _c_int, _c_int, _c_int, _p]),
    "omni_page_write": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _c_int, _c_int, _p, _c_int, _c_int, _p, _p]),
    "omni_decode_flags": (_c_int, [_p, _p, _p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _p, _p]),
    "omni_decode_flags_f64": (_c_int, [_p, _p, _p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _p,
                                       _p]),
    "omni_slim_cache": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _c_int, _p, _c_int, _c_int, _c_int, _p, _p, _p]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libomnisparse.so and attach the C prototypes (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CudaError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.omni_abi_version() != 3:
        raise CudaError("libomnisparse ABI version mismatch")
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke an ``omni_*`` entry point and raise the mapped exception on a
    non-zero status."""
    lib = load()
    code = getattr(lib, name)(*args)
    if code:
        raise_for_status(code, name, (lib.omni_last_error() or b"").decode(errors="replace"))


def size(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))
