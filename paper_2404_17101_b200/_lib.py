"""ctypes binding of libpasgal_bcc.so (the C-ABI in include/pasgal_bcc.h).

There is no fallback: if the library is missing or fails to load, every entry point
raises.  ``load()`` never compiles on its own; ``build()`` (``__graft_entry__.build``)
does that ahead of time so the .so travels with the repository.
"""

import ctypes
import os

from . import _build

LIB_PATH = os.environ.get("PASGAL_BCC_LIB", _build.LIB)   # override: experiment variants

PASGAL_OK = 0
PASGAL_EINVAL = 1
PASGAL_ENOTSYM = 2
PASGAL_EWORKSPACE = 3
PASGAL_ECUDA = 4
PASGAL_EUNSORTED = 5
PASGAL_ERANGE = 6
PASGAL_BCC_CANONICAL = 1


class PasgalCsr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m_slots", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("targets", ctypes.c_void_p)]


class PasgalBccProf(ctypes.Structure):
    _fields_ = [("events", ctypes.POINTER(ctypes.c_void_p)), ("n_events", ctypes.c_int),
                ("launches", ctypes.c_int)]


STAGES = ["begin", "first_cc", "forest", "listrank", "tour", "tags", "rmq", "last_cc", "artic", "labels",
          "canonical"]
NSTAGES = len(STAGES)


class PasgalBccOut(ctypes.Structure):
    _fields_ = [("edge_label", ctypes.c_void_p), ("artic_bits", ctypes.c_void_p),
                ("bcc_count", ctypes.c_void_p), ("comp", ctypes.c_void_p),
                ("parent", ctypes.c_void_p), ("first", ctypes.c_void_p)]


_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_INT = ctypes.c_int
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); must match include/pasgal_bcc.h exactly
SIGNATURES = {
    "pasgal_bcc_workspace_bytes": (_SZ, [_I64, _I64]),
    "pasgal_csr_validate_workspace_bytes": (_SZ, [_I64, _I64]),
    "pasgal_bcc_two_level_tags": (_INT, [_I64, _I64]),
    "pasgal_bcc": (_INT, [ctypes.POINTER(PasgalCsr), ctypes.POINTER(PasgalBccOut), _VP, _SZ, _U64, _U32, _VP]),
    "pasgal_bcc_ex": (_INT, [ctypes.POINTER(PasgalCsr), ctypes.POINTER(PasgalBccOut), _VP, _SZ, _U64, _U32, _VP,
                             ctypes.POINTER(PasgalBccProf)]),
    "pasgal_bcc_graph_create": (_INT, [ctypes.POINTER(PasgalCsr), ctypes.POINTER(PasgalBccOut), _VP, _SZ, _U64, _U32,
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "pasgal_bcc_graph_launch": (_INT, [_VP, _VP, ctypes.POINTER(ctypes.c_int)]),
    "pasgal_bcc_graph_destroy": (None, [_VP]),
    "pasgal_cc": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _VP, _VP, _SZ, _U64, _VP]),
    "pasgal_canonicalize_temp_bytes": (_SZ, [_I64, _I64, _I64]),
    "pasgal_canonicalize": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _I64, _VP, _VP, _SZ, _VP]),
    "pasgal_csr_first_error": (_INT, [ctypes.POINTER(PasgalCsr), _VP, ctypes.POINTER(ctypes.c_int64), _VP]),
    "pasgal_csr_validate": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _SZ, _VP]),
    "pasgal_csr_validate_begin": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _SZ, _VP]),
    "pasgal_csr_validate_end": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _SZ, _VP]),
    "pasgal_csr_validate_check": (_INT, [ctypes.POINTER(PasgalCsr), _VP, _SZ, _VP, _VP]),
    "pasgal_csr_build_temp_bytes": (_SZ, [_I64, _I64]),
    "pasgal_csr_from_keys": (_INT, [_I64, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "pasgal_gen_grid_temp_bytes": (_SZ, [_I64, _I64]),
    "pasgal_gen_grid": (_INT, [_I64, _I64, _U64, _U64, _INT, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "pasgal_gen_rmat_keys": (_INT, [_INT, _I64, _U64, _U32, _U32, _U32, _VP, _VP, _VP]),
    "pasgal_gen_knn_temp_bytes": (_SZ, [_I64, _INT]),
    "pasgal_gen_knn_keys": (_INT, [_I64, _INT, _U64, _INT, _VP, _VP, _VP, _SZ, _VP]),
    "pasgal_bits_to_bytes": (_INT, [_VP, _I64, _VP, _VP]),
    "pasgal_canonical_checksum": (_INT, [_VP, _I64, _VP, _I64, _VP, _VP]),
    "pasgal_bfs_vgc_workspace_bytes": (_SZ, [_I64]),
    "pasgal_bfs_vgc": (_INT, [ctypes.POINTER(PasgalCsr), _I64, _INT, _VP, ctypes.POINTER(ctypes.c_int64), _VP, _SZ,
                              _VP]),
    "pasgal_bfs_vgc_ex": (_INT, [ctypes.POINTER(PasgalCsr), _I64, _INT, ctypes.c_double, _INT, _VP,
                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), _VP, _SZ, _VP]),
    "pasgal_adj_temp_bytes": (_SZ, [_I64]),
    "pasgal_msbfs_workspace_bytes": (_SZ, [_I64]),
    "pasgal_msbfs": (_INT, [ctypes.POINTER(PasgalCsr), ctypes.POINTER(ctypes.c_int64), _INT, _VP,
                            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), _VP, _SZ, _VP]),
    "pasgal_msbfs_ex": (_INT, [ctypes.POINTER(PasgalCsr), ctypes.POINTER(ctypes.c_int64), _INT, _VP,
                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), _VP, _I64, _VP, _VP,
                               _SZ, _VP]),
    "pasgal_adj_tokenize": (_INT, [_VP, _I64, _VP, _SZ, ctypes.POINTER(ctypes.c_int64), _VP]),
    "pasgal_adj_token_position": (_INT, [_VP, _I64, _VP, _SZ, _I64, ctypes.POINTER(ctypes.c_int64), _VP]),
    "pasgal_adj_parse": (_INT, [_VP, _I64, _VP, _SZ, _I64, _I64, _INT, _VP, _VP, ctypes.POINTER(ctypes.c_int64),
                                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), _VP]),
    "pasgal_strerror": (ctypes.c_char_p, [_INT]),
    "pasgal_version": (ctypes.c_char_p, []),
}

_lib = None


class PasgalError(RuntimeError):
    pass


def load():
    """Load the in-tree shared library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libpasgal_bcc.so not found at {LIB_PATH}: build it first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def strerror(status):
    return load().pasgal_strerror(status).decode()


def check(status, what="pasgal"):
    """Map a status code to the reference's exception types."""
    if status == PASGAL_OK:
        return
    msg = strerror(status)
    if status == PASGAL_ECUDA:
        raise PasgalError(f"{what}: {msg}")
    raise ValueError(msg if status == PASGAL_ENOTSYM else f"{what}: {msg}")
