"""ctypes binding of libhexgram_b200.so (include/hexgram_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a) into ``paper_1711_00984_b200/_lib/``.  There is no fallback: if
the library is missing or no CUDA device is present, every device entry
point raises.
"""

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
# HXG_LIB selects an alternative build of the same library (investigation
# builds with different compile flags, tools/v3p7_check.sh); default: in-tree
LIB_PATH = os.environ.get("HXG_LIB") or os.path.join(LIB_DIR, "libhexgram_b200.so")
CSRC = os.path.join(_HERE, "csrc")

HXG_OK = 0
HXG_ERR_ORDER = -1
HXG_ERR_SPACE = -2
HXG_ERR_KIND = -3
HXG_ERR_WORKSPACE = -4
HXG_ERR_CUDA = -5
HXG_ERR_ARG = -6
HXG_ERR_DEGENERATE = -7
HXG_MAX_ORDER = 12
HXG_MAX_RULE = 16

# device 1D-table block layout (doubles; hxg_plan.h): nodes [LT], weights [LT],
# T[f][k][l] (f 0 chi, 1 chi') [2][KT][LT], F[rs][i][j] [4][KT][KT]
KT = 16
LT = 16
TAB_NODES = 0
TAB_WTS = TAB_NODES + LT
TAB_T = TAB_WTS + LT
TAB_F = TAB_T + 2 * KT * LT
TAB_TOTAL = TAB_F + 4 * KT * KT

SPACE_CODES = {"H1": 0, "Hcurl": 1, "Hdiv": 2, "L2": 3}
PATH_CODES = {"general": 0, "affine": 1, "extrusion": 2}

# every symbol the header declares (checked by the CPU test suite)
EXPORTED = (
    "hxg_version",
    "hxg_fused_order_max",
    "hxg_error_string",
    "hxg_dim",
    "hxg_accumulations",
    "hxg_tables_doubles",
    "hxg_make_tables",
    "hxg_workspace_size",
    "hxg_gram_batched",
    "hxg_metric_batched",
    "hxg_contract_batched",
    "hxg_gram_batched_host",
    "hxg_expand_full",
    "hxg_graph_mixed",
    "hxg_graph_assemble",
    "hxg_condense_workspace_size",
    "hxg_condense_batched",
    "hxg_acoustics_workspace_size",
    "hxg_acoustics_batched",
)

_lib = None

_i = ctypes.c_int
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def build(force: bool = False) -> str:
    """Compile the CUDA library with the in-tree Makefile (nvcc, sm_100a)."""
    cmd = ["make", "-s", f"-j{min(8, os.cpu_count() or 1)}", "-C", CSRC]
    if force:
        cmd.insert(1, "-B")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    """Load the library (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(LIB_PATH)
    L.hxg_version.restype = _i
    L.hxg_fused_order_max.restype = _i
    L.hxg_error_string.argtypes = [_i]
    L.hxg_error_string.restype = ctypes.c_char_p
    L.hxg_dim.argtypes = [_i, _i, _i, _i]
    L.hxg_dim.restype = _i
    L.hxg_accumulations.argtypes = [_i, _i, _i, _i, _i, _i]
    L.hxg_accumulations.restype = ctypes.c_longlong
    L.hxg_tables_doubles.restype = _sz
    L.hxg_make_tables.argtypes = [_i, _vp, _vp, _vp, _vp]
    L.hxg_make_tables.restype = _i
    L.hxg_workspace_size.argtypes = [_i, _i, _i, _i, _i, _i, _i]
    L.hxg_workspace_size.restype = _sz
    L.hxg_gram_batched.argtypes = [_i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp, _sz, _vp]
    L.hxg_gram_batched.restype = _i
    L.hxg_metric_batched.argtypes = [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.hxg_metric_batched.restype = _i
    L.hxg_contract_batched.argtypes = [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp]
    L.hxg_contract_batched.restype = _i
    L.hxg_gram_batched_host.argtypes = [_i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _vp]
    L.hxg_gram_batched_host.restype = _i
    L.hxg_expand_full.argtypes = [_i, _i, _vp, _vp, _vp]
    L.hxg_expand_full.restype = _i
    L.hxg_graph_mixed.argtypes = [_i, ctypes.c_double, _vp, _vp, _vp]
    L.hxg_graph_mixed.restype = _i
    L.hxg_graph_assemble.argtypes = [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp]
    L.hxg_graph_assemble.restype = _i
    L.hxg_condense_workspace_size.argtypes = [_i, _i, _i]
    L.hxg_condense_workspace_size.restype = _sz
    L.hxg_condense_batched.argtypes = [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.hxg_condense_batched.restype = _i
    L.hxg_acoustics_workspace_size.argtypes = [_i, _i, _i, _i]
    L.hxg_acoustics_workspace_size.restype = _sz
    L.hxg_acoustics_batched.argtypes = [_i, _i, ctypes.c_double, _i, _i, _vp, _vp, _vp, _vp, _i,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.hxg_acoustics_batched.restype = _i
    _lib = L
    return L


def error_string(code: int) -> str:
    return lib().hxg_error_string(code).decode()
