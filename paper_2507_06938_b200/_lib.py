"""ctypes binding of the stbta C ABI (include/stbta.h).

The shared library is built in-tree (``paper_2507_06938_b200/libstbta.so``)
and is the only compute path: there is no CPU fallback.  Loading fails loudly
when the library is missing or no CUDA device is present.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# STBTA_LIB selects another build of the same ABI (the bounds-checked
# libstbta_check.so of `make check`, for the checking runs)
LIB_PATH = os.environ.get("STBTA_LIB") or os.path.join(_HERE, "libstbta.so")
TOOLS_LIB_PATH = os.path.join(_HERE, "libstbta_tools.so")

_lib = None

# storage tile of stbta_assemble (must equal stbta_assemble_tile_elems())
ASM_TILE = 2048

c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_size = ctypes.c_size_t
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/stbta.h
_SIGNATURES = {
    "stbta_version": (ctypes.c_char_p, []),
    "stbta_storage_elems": (c_ll, [c_int, c_int, c_int]),
    "stbta_pobtaf_workspace_bytes": (c_size, [c_int, c_int, c_int]),
    "stbta_pobtaf": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_size, c_vp]),
    "stbta_pobtaf_ex": (
        c_int,
        [c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_size,
         c_vp],
    ),
    "stbta_pobtas_ex": (
        c_int,
        [c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp, c_size,
         c_vp],
    ),
    "stbta_pobtasi_ex": (
        c_int,
        [c_vp] * 8 + [c_int, c_int, c_int, c_int, c_int, c_vp, c_size, c_vp],
    ),
    "stbta_pobtas_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int]),
    "stbta_pobtas": (
        c_int,
        [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp, c_size, c_vp],
    ),
    "stbta_pobtasi_workspace_bytes": (c_size, [c_int, c_int, c_int]),
    "stbta_pobtasi": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp, c_size, c_vp]),
    "stbta_couple_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int, c_int]),
    "stbta_couple": (
        c_int,
        [c_int, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_ll, c_ll, c_vp, c_ll, c_ll, c_vp, c_ll,
         c_ll, c_int, c_vp, c_size, c_vp],
    ),
    "stbta_stream_memops_supported": (c_int, []),
    "stbta_upload_blocks": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_vp, ctypes.c_uint, c_vp]),
    "stbta_pobtaf_ready": (
        c_int,
        [c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, ctypes.c_uint, c_vp, c_size, c_vp],
    ),
    "stbta_pobtasi_prepare": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_size, c_vp]),
    "stbta_pobtasi_prepared": (
        c_int,
        [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp, c_size, c_vp, c_vp],
    ),
    "stbta_pobtas_w_workspace_bytes": (c_size, [c_int, c_int, c_int]),
    "stbta_pobtas_w": (
        c_int,
        [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp, c_vp, c_size, c_vp],
    ),
    "stbta_pobtasi_stream_out": (
        c_int,
        [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp, c_size, c_vp, c_vp],
    ),
    "stbta_launch_count": (c_ll, []),
    "stbta_debug_set_profile": (None, [c_vp]),
    "stbta_probe_dmma": (c_int, [c_int, c_int, c_vp, c_vp]),
    "stbta_assemble_tile_elems": (c_int, []),
    "stbta_assemble": (c_int, [c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "stbta_quadform": (
        c_int,
        [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_ll, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_vp],
    ),
    "stbta_rhs_combine": (c_int, [c_vp, c_vp, c_vp, c_int, c_ll, c_vp]),
    "stbta_residual": (c_int, [c_vp, c_vp, c_vp, c_ll, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp]),
}

# tools-only library (include/stbta_tools.h): micro-benchmarks, debug probes
_TOOLS_SIGNATURES = {
    "stbta_dgemm": (
        c_int,
        [c_int, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_ll, c_vp, c_ll, c_dbl, c_vp, c_ll, c_vp],
    ),
    "stbta_debug_globaltimer": (c_int, [c_vp, c_vp]),
    "stbta_debug_potrf_bench": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_vp]),
    "stbta_debug_lds_bench": (c_int, [c_int, c_int, c_int, c_vp, c_vp]),
    "stbta_debug_latency": (c_int, [c_int, c_int, c_vp, c_vp, c_vp]),
    "stbta_debug_tile_bench": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp]),
    "stbta_probe_dfma": (c_int, [c_int, c_int, c_vp, c_vp]),
}


class StbtaError(RuntimeError):
    """A C-ABI call returned a non-zero status (launch or argument error)."""


def load(require_cuda=True):
    """Load libstbta.so (once) and declare its signatures."""
    global _lib
    if _lib is not None:
        if require_cuda and not torch.cuda.is_available():
            raise StbtaError("stbta needs a CUDA device (sm_100a); no CPU fallback exists")
        return _lib
    if not os.path.exists(LIB_PATH):
        raise StbtaError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    # torch's libcudart.so.12 must be loaded first so the library binds to it
    torch.cuda.is_available()
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.stbta_assemble_tile_elems() != ASM_TILE:
        raise StbtaError("libstbta.so assemble tile differs from the Python binding")
    _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise StbtaError("stbta needs a CUDA device (sm_100a); no CPU fallback exists")
    return lib


_tools = None


def load_tools():
    """The tools-only library (micro-benchmarks / debug probes for tools/)."""
    global _tools
    if _tools is None:
        load()
        lib = ctypes.CDLL(TOOLS_LIB_PATH)
        for name, (res, args) in _TOOLS_SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _tools = lib
    return _tools


def exported_symbols():
    return list(_SIGNATURES)


def check(status, what):
    if status != 0:
        raise StbtaError(f"{what} failed with status {status}")


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)
