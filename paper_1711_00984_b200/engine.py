"""Device engine: owns the per-device 1D tables and workspace and calls the
C ABI of libhexgram_b200.so.

PyTorch is used for device memory, streams and host pinning only; every
floating-point operation of the Gram integration runs in the sm_100a
kernels behind ``hxg_gram_batched``.  There is no CPU fallback: without a
CUDA device or without the built library the engine raises.
"""

import ctypes
import threading

import numpy as np
import torch

from . import _native
from .errors import DegenerateMapError, InvalidOrderError, SimplificationNotApplicableError


def _check(rc: int, what: str) -> None:
    if rc == _native.HXG_OK:
        return
    msg = f"{what}: {_native.error_string(rc)} (code {rc})"
    if rc == _native.HXG_ERR_ORDER:
        raise InvalidOrderError(msg)
    if rc == _native.HXG_ERR_KIND:
        raise SimplificationNotApplicableError(msg)
    if rc == _native.HXG_ERR_DEGENERATE:
        raise DegenerateMapError(float("nan"), ())
    if rc in (_native.HXG_ERR_SPACE, _native.HXG_ERR_ARG):
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class GramEngine:
    """Batched Gram integration on one CUDA device."""

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1711_00984_b200 needs a CUDA device (sm_100a); none found")
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.lib = _native.lib()
        self._tables = {}
        self._ws = {}
        self._lock = threading.Lock()

    # -- 1D tables ---------------------------------------------------------
    def tables(self, L: int, nodes=None, weights=None, stream=None) -> torch.Tensor:
        """Device table block for an L-point rule (Gauss by default, or the
        given nodes/weights of a user Rule1D)."""
        key = (L,) if nodes is None else (L, np.asarray(nodes).tobytes(), np.asarray(weights).tobytes())
        t = self._tables.get(key)
        if t is not None:
            return t
        st = stream or torch.cuda.current_stream(self.device)
        t = torch.empty(self.lib.hxg_tables_doubles(), dtype=torch.float64, device=self.device)
        if nodes is None:
            rc = self.lib.hxg_make_tables(L, None, None, _ptr(t), ctypes.c_void_p(st.cuda_stream))
        else:
            with torch.cuda.stream(st):
                dn = torch.as_tensor(np.ascontiguousarray(nodes, dtype=np.float64)).to(self.device)
                dw = torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float64)).to(self.device)
            rc = self.lib.hxg_make_tables(L, _ptr(dn), _ptr(dw), _ptr(t), ctypes.c_void_p(st.cuda_stream))
        _check(rc, "hxg_make_tables")
        # the cached block is read later from any stream: complete it once here
        st.synchronize()
        self._tables[key] = t
        return t

    def workspace(self, nbytes: int, stream=None) -> torch.Tensor:
        """Scratch buffer of at least `nbytes`, one per stream: calls are stream-ordered,
        so reuse on the same stream is safe and distinct streams never share one."""
        if nbytes == 0:
            return None
        st = stream or torch.cuda.current_stream(self.device)
        ws = self._ws.get(st.cuda_stream)
        if ws is None or ws.numel() < nbytes:
            # allocated on `st`: the caching allocator then recycles the block (and the
            # one it replaces) only in `st` order
            with torch.cuda.stream(st):
                ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._ws[st.cuda_stream] = ws
        return ws

    # -- batched integration -------------------------------------------------
    def integrate(self, space: str, path: str, orders, L: int, kind, params, coef=None,
                  wgrid=None, out=None, status=None, nodes=None, weights=None, stream=None,
                  check_status: bool = True):
        """Integrate E elements.  kind/params/coef/wgrid are device tensors
        (int32 [E], float64 [E, 24], float64 [E], float64 [E, L^3]) or host
        arrays (copied in).  Returns (packed [E, N(N+1)/2] float64 device
        tensor, status [E] int32 device tensor).

        The launch is ordered after the work already queued on the caller's
        current stream (inputs produced there), whichever `stream` it runs on.
        check_status=True waits for the call and raises DegenerateMapError /
        SimplificationNotApplicableError from the device status word;
        check_status=False returns without any host synchronisation (read the
        status later with `raise_for_status(status, path, stream)`)."""
        dev = self.device
        p1, p2, p3 = (int(p) for p in orders)
        sc, pc = _native.SPACE_CODES[space], _native.PATH_CODES[path]
        N = self.lib.hxg_dim(sc, p1, p2, p3)
        _check(N if N < 0 else 0, "hxg_dim")
        cur = torch.cuda.current_stream(dev)
        st = stream or cur
        kind = torch.as_tensor(kind, dtype=torch.int32).to(dev).contiguous()
        E = int(kind.shape[0])
        params = torch.as_tensor(params, dtype=torch.float64).to(dev).reshape(E, 24).contiguous()
        if coef is not None:
            coef = torch.as_tensor(coef, dtype=torch.float64).to(dev).reshape(E).contiguous()
        if wgrid is not None:
            wgrid = torch.as_tensor(wgrid, dtype=torch.float64).to(dev).reshape(E, -1).contiguous()
            if wgrid.shape[1] != L ** 3:
                raise ValueError("wgrid must hold L^3 nodes per element")
        P = N * (N + 1) // 2
        if out is None:
            out = torch.empty((E, P), dtype=torch.float64, device=dev)
        if status is None:
            status = torch.empty(E, dtype=torch.int32, device=dev)
        tab = self.tables(L if path == "general" else max(L, 1), nodes, weights, st)
        if st != cur:
            # inputs (and a caller-provided `out`) were produced on the current stream;
            # tensors allocated here on `cur` are used on `st` until it drains
            st.wait_stream(cur)
            for t in (kind, params, coef, wgrid, out, status):
                if t is not None:
                    t.record_stream(st)
        with self._lock:
            ws_bytes = self.lib.hxg_workspace_size(sc, pc, p1, p2, p3, L, E)
            ws = self.workspace(ws_bytes, st)
            rc = self.lib.hxg_gram_batched(sc, pc, p1, p2, p3, L, E, _ptr(kind), _ptr(params),
                                           _ptr(coef), _ptr(wgrid), _ptr(tab), _ptr(out),
                                           _ptr(status), _ptr(ws), ws_bytes,
                                           ctypes.c_void_p(st.cuda_stream))
        _check(rc, "hxg_gram_batched")
        if check_status:
            self.raise_for_status(status, path, st)
        return out, status

    @staticmethod
    def raise_for_status(status: torch.Tensor, path: str, stream=None) -> None:
        """Raise the reference's exception for the first flagged element.  The
        status word is read on `stream` (the stream the call ran on)."""
        st = stream or torch.cuda.current_stream(status.device)
        with torch.cuda.stream(st):
            s = status.cpu().numpy()
        bad = np.nonzero(s)[0]
        if bad.size == 0:
            return
        e = int(bad[0])
        if s[e] & 2:
            raise SimplificationNotApplicableError(
                f"element {e}: map kind admits no {path} simplification")
        raise DegenerateMapError(float("nan"), (e,))

    def expand(self, packed: torch.Tensor, N: int, stream=None) -> torch.Tensor:
        E = packed.shape[0]
        full = torch.empty((E, N, N), dtype=torch.float64, device=packed.device)
        st = stream or torch.cuda.current_stream(packed.device)
        rc = self.lib.hxg_expand_full(N, E, _ptr(packed), _ptr(full), ctypes.c_void_p(st.cuda_stream))
        _check(rc, "hxg_expand_full")
        return full

    def integrate_host(self, space: str, path: str, orders, L: int, kind: np.ndarray,
                       params: np.ndarray, coef: np.ndarray | None, out: np.ndarray,
                       status: np.ndarray | None = None, nodes=None, weights=None,
                       wgrid: np.ndarray | None = None) -> None:
        """Host buffers in, host buffer out (hxg_gram_batched_host): the
        reference's kernel seam kern(p1, p2, p3, nodes, wts, kind, par, wgrid)
        (gram.py:154-157) batched.  nodes/weights: a user Rule1D (None: Gauss
        rule of L points); wgrid: sampled mass weights [E, L^3] (general path)."""
        p1, p2, p3 = (int(p) for p in orders)
        kind = np.ascontiguousarray(kind, dtype=np.int32)
        params = np.ascontiguousarray(params, dtype=np.float64)
        coef = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        if nodes is not None:
            nodes = np.ascontiguousarray(nodes, dtype=np.float64)
            weights = np.ascontiguousarray(weights, dtype=np.float64)
            if nodes.size != L or weights.size != L:
                raise ValueError("nodes / weights must hold L points")
        E = kind.shape[0]
        if wgrid is not None:
            wgrid = np.ascontiguousarray(wgrid, dtype=np.float64)
            if wgrid.size != E * L ** 3:
                raise ValueError("wgrid must hold L^3 nodes per element")
        rc = self.lib.hxg_gram_batched_host(
            _native.SPACE_CODES[space], _native.PATH_CODES[path], p1, p2, p3, L, E,
            None if nodes is None else nodes.ctypes.data,
            None if weights is None else weights.ctypes.data,
            kind.ctypes.data, params.ctypes.data, None if coef is None else coef.ctypes.data,
            None if wgrid is None else wgrid.ctypes.data,
            out.ctypes.data if isinstance(out, np.ndarray) else out.data_ptr(),
            None if status is None else status.ctypes.data)
        if rc == _native.HXG_ERR_DEGENERATE and status is not None:
            bad = np.nonzero(status & 1)[0]
            raise DegenerateMapError(float("nan"), tuple(int(e) for e in bad[:1]))
        _check(rc, "hxg_gram_batched_host")


_engines = {}


def get_engine(device=None) -> GramEngine:
    key = str(device)
    eng = _engines.get(key)
    if eng is None:
        eng = GramEngine(device)
        _engines[key] = eng
    return eng
