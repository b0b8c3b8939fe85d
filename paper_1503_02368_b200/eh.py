"""Thin Python binding of the C ABI in include/eh.h (argument marshalling only).

Every step of the path runs in libeh.so's CUDA kernels.  There is no CPU
fallback: if the library cannot be loaded or no CUDA device is usable, the
calls raise.  Names follow the C ABI: ``load_edges``, ``count_triangles``,
``count_4cliques``, ``intersect``.

Inputs may be numpy arrays (host), torch CPU tensors (pinned or not) or torch
CUDA tensors (passed with EH_INPUT_ON_DEVICE, no copy).  PyTorch serves only
device memory (optionally as the library's allocator) and streams.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libeh.so")
# EH_LIB=checked loads the checked build (device-side bounds assertions, build.py
# checked=True) -- used by the tests in place of compute-sanitizer
if os.environ.get("EH_LIB") == "checked":
    LIB_PATH = os.path.join(_PKG, "lib", "libeh_checked.so")

EH_OK, EH_EINVAL, EH_ENOMEM, EH_ECUDA, EH_EUNSORTED = 0, -1, -2, -3, -4
EH_COUNT_ERROR = 2**64 - 1
EH_INPUT_ON_DEVICE, EH_SET_DEVICE, EH_ALL_UINT, EH_NO_ALGO, EH_BLOCK_LAYOUT, EH_FORCE_SEARCH = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20

_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class EHConfig(ctypes.Structure):
    _fields_ = [("bitset_tau", ctypes.c_uint32), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("dev_alloc", _ALLOC_FN), ("dev_free", _FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("bin_small_max", ctypes.c_uint32), ("bin_large_min", ctypes.c_uint32),
                ("min_bitset_card", ctypes.c_uint32), ("order", ctypes.c_uint32),
                ("bin_thread_max", ctypes.c_uint32)]

ORDERS = {"degree": 0, "rev_degree": 1, "random": 2, "bfs": 3, "hybrid": 4, "shingle": 5, "id": 6}


class EHStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n_input", "m_undirected", "n_active", "max_out_degree",
                                                "n_bitset_sets", "bitset_words", "device_bytes", "alg_bytes_tri",
                                                "wedge_work")]


class EHError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"eh status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libeh.so (built in-tree by build.py).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1503_02368_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, u32p = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p
        L.eh_load_edges.argtypes = [u32p, u32p, u64]
        L.eh_load_edges.restype = vp
        L.eh_load_edges_ex.argtypes = [u32p, u32p, u64, ctypes.POINTER(EHConfig)]
        L.eh_load_edges_ex.restype = vp
        L.eh_count_triangles.argtypes = [vp]
        L.eh_count_triangles.restype = u64
        L.eh_count_4cliques.argtypes = [vp]
        L.eh_count_4cliques.restype = u64
        for name in ("eh_count_triangles_unpruned", "eh_count_4cliques_unpruned", "eh_alg_bytes_k4"):
            getattr(L, name).argtypes = [vp]
            getattr(L, name).restype = u64
        for name in ("eh_count_triangles_range", "eh_count_4cliques_range"):
            getattr(L, name).argtypes = [vp, u64, u64]
            getattr(L, name).restype = u64
        L.eh_symmetric_stats.argtypes = [vp, ctypes.POINTER(EHStats)]
        L.eh_symmetric_stats.restype = ctypes.c_int
        L.eh_triangles_per_vertex.argtypes = [vp, vp]
        L.eh_triangles_per_vertex.restype = ctypes.c_int
        for name in ("eh_count_lollipop", "eh_count_barbell"):
            getattr(L, name).argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
            getattr(L, name).restype = ctypes.c_int
        L.eh_intersect.argtypes = [u32p, u64, u32p, u64, u32p]
        L.eh_intersect.restype = ctypes.c_int64
        L.eh_graph_stats.argtypes = [vp, ctypes.POINTER(EHStats)]
        L.eh_graph_stats.restype = ctypes.c_int
        L.eh_graph_export.argtypes = [vp, vp, vp, vp, vp]
        L.eh_graph_export.restype = ctypes.c_int
        L.eh_free.argtypes = [vp]
        L.eh_free.restype = None
        L.eh_count_batch.argtypes = [vp, vp, vp, u64, ctypes.c_uint32, ctypes.POINTER(EHConfig), vp]
        L.eh_count_batch.restype = ctypes.c_int
        L.eh_release_cached_memory.argtypes = []
        L.eh_release_cached_memory.restype = None
        L.eh_launch_count.argtypes = []
        L.eh_launch_count.restype = u64
        L.eh_last_status.argtypes = []
        L.eh_last_status.restype = ctypes.c_int
        L.eh_last_error.argtypes = []
        L.eh_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


EXPORTED_SYMBOLS = ("eh_load_edges", "eh_load_edges_ex", "eh_count_triangles", "eh_count_4cliques",
                    "eh_count_triangles_range", "eh_count_4cliques_range", "eh_alg_bytes_k4", "eh_count_batch",
                    "eh_count_triangles_unpruned", "eh_count_4cliques_unpruned", "eh_symmetric_stats",
                    "eh_triangles_per_vertex", "eh_count_lollipop", "eh_count_barbell", "eh_intersect",
                    "eh_graph_stats", "eh_graph_export", "eh_free", "eh_release_cached_memory", "eh_launch_count",
                    "eh_last_status", "eh_last_error")


def _raise():
    L = lib()
    raise EHError(L.eh_last_status(), (L.eh_last_error() or b"").decode())


def _ptr_of(a):
    """(pointer, on_device, keepalive) for a numpy array or torch tensor of uint32/int32."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.dtype not in (torch.int32, torch.uint32):
            raise TypeError(f"expected a 32-bit integer tensor, got {a.dtype}")
        a = a.contiguous()
        return (a.data_ptr() if a.numel() else None), a.is_cuda, a
    arr = np.ascontiguousarray(np.asarray(a), dtype=np.uint32)
    return (arr.ctypes.data if arr.size else None), False, arr


def _numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") and callable(a.numel) else int(np.asarray(a).size)


class _TorchAllocator:
    """Routes the library's device allocations through torch's caching allocator."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device
        self.alloc_cb = _ALLOC_FN(self._alloc)
        self.free_cb = _FREE_FN(self._free)

    def _alloc(self, size, stream, ctx):
        try:
            return self.torch.cuda.caching_allocator_alloc(int(size), self.device, stream or 0)
        except Exception:  # OOM -> NULL -> EH_ENOMEM
            return None

    def _free(self, ptr, stream, ctx):
        self.torch.cuda.caching_allocator_delete(ptr)


@dataclass
class Stats:
    n_input: int
    m_undirected: int
    n_active: int
    max_out_degree: int
    n_bitset_sets: int
    bitset_words: int
    device_bytes: int
    alg_bytes_tri: int
    wedge_work: int


class Graph:
    """A loaded trie (eh_graph*).  ``Graph(src, dst, ...)`` == eh_load_edges_ex."""

    def __init__(self, src, dst, *, tau: int = 0, all_uint: bool = False, no_algo: bool = False, force_search: bool = False,
                 block_layout: bool = False, order: str = "degree", bin_small_max: int = 0,
                 bin_large_min: int = 0, bin_thread_max: int = 0, min_bitset_card: int = 0, stream=None,
                 device: int | None = None,
                 torch_allocator: bool = False):
        L = lib()
        n = _numel(src)
        if _numel(dst) != n:
            raise ValueError("src and dst differ in length")
        ps, sdev, self._ks = _ptr_of(src)
        pd, ddev, self._kd = _ptr_of(dst)
        if sdev != ddev:
            raise ValueError("src and dst must both be host or both be device memory")
        cfg = EHConfig()
        cfg.bitset_tau = tau
        cfg.flags = (EH_INPUT_ON_DEVICE if sdev else 0) | (EH_ALL_UINT if all_uint else 0) | (EH_NO_ALGO if no_algo else 0) \
            | (EH_BLOCK_LAYOUT if block_layout else 0) | (EH_FORCE_SEARCH if force_search else 0)
        if device is not None:
            cfg.flags |= EH_SET_DEVICE
            cfg.device = device
        cfg.bin_small_max = bin_small_max
        cfg.bin_large_min = bin_large_min
        cfg.bin_thread_max = bin_thread_max
        cfg.min_bitset_card = min_bitset_card
        cfg.order = ORDERS[order]
        if stream is not None:
            cfg.stream = getattr(stream, "cuda_stream", stream)
        elif sdev:
            # device-resident inputs are ordered on the stream that produced them: torch's
            # current stream (e.g. the copy .contiguous() may have just launched)
            import torch
            cfg.stream = torch.cuda.current_stream(self._ks.device).cuda_stream
        self._alloc = None
        if torch_allocator:
            import torch
            self._alloc = _TorchAllocator(device if device is not None else torch.cuda.current_device())
            cfg.dev_alloc = self._alloc.alloc_cb
            cfg.dev_free = self._alloc.free_cb
        h = L.eh_load_edges_ex(ps, pd, n, ctypes.byref(cfg))
        self._ks = self._kd = None
        if not h:
            _raise()
        self._h = ctypes.c_void_p(h)

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            lib().eh_free(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def count_triangles(self) -> int:
        r = lib().eh_count_triangles(self._h)
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def count_4cliques(self) -> int:
        r = lib().eh_count_4cliques(self._h)
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def count_triangles_range(self, r0: int, r1: int) -> int:
        """Triangles whose earliest vertex has rank in [r0, r1) (eh_count_triangles_range)."""
        r = lib().eh_count_triangles_range(self._h, int(r0), int(r1))
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def count_4cliques_range(self, r0: int, r1: int) -> int:
        """4-cliques whose earliest vertex has rank in [r0, r1) (eh_count_4cliques_range)."""
        r = lib().eh_count_4cliques_range(self._h, int(r0), int(r1))
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def alg_bytes_k4(self) -> int:
        """B_K4(tau = 32) of SURVEY.md §8(d) (eh_alg_bytes_k4)."""
        r = lib().eh_alg_bytes_k4(self._h)
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def count_triangles_unpruned(self) -> int:
        """NEXT-2: the triangle Generic-Join on the symmetric (unpruned) data = 6T (eh_count_triangles_unpruned)."""
        r = lib().eh_count_triangles_unpruned(self._h)
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def count_4cliques_unpruned(self) -> int:
        """NEXT-2: the 4-clique Generic-Join on the symmetric (unpruned) data = 24 K4 (eh_count_4cliques_unpruned)."""
        r = lib().eh_count_4cliques_unpruned(self._h)
        if r == EH_COUNT_ERROR:
            _raise()
        return int(r)

    def symmetric_stats(self) -> Stats:
        """Statistics of the symmetric trie (eh_symmetric_stats)."""
        st = EHStats()
        if lib().eh_symmetric_stats(self._h, ctypes.byref(st)) != EH_OK:
            _raise()
        return Stats(**{f: int(getattr(st, f)) for f, _ in EHStats._fields_})

    def triangles_per_vertex(self, out=None):
        """t(v) per rank (eh_triangles_per_vertex); rank r is original id export()[2][r].

        ``out``: optional uint64/int64 CUDA tensor of n_active elements (filled on the
        device); otherwise a host numpy uint64 array is returned."""
        n = self.stats().n_active
        if out is None:
            t = np.zeros(max(n, 1), np.uint64)
            ptr = t.ctypes.data
        else:
            import torch
            if not (isinstance(out, torch.Tensor) and out.is_cuda):
                raise TypeError("out must be a CUDA tensor (the host result is returned when out is None)")
            if out.dtype not in (torch.int64, torch.uint64):
                raise TypeError(f"out must be int64 or uint64, got {out.dtype}")
            if not out.is_contiguous():
                raise ValueError("out must be contiguous")
            if out.numel() < n:
                raise ValueError(f"out has {out.numel()} elements, need {n}")
            t, ptr = out, out.data_ptr()
        if lib().eh_triangles_per_vertex(self._h, ptr) != EH_OK:
            _raise()
        return t[:n]

    def _count128(self, fn) -> int:
        out = (ctypes.c_uint64 * 2)()
        if fn(self._h, out) != EH_OK:
            _raise()
        return int(out[0]) | (int(out[1]) << 64)

    def count_lollipop(self) -> int:
        """COUNT(*) of Lollipop L3,1 on the undirected data (eh_count_lollipop), exact (128-bit)."""
        return self._count128(lib().eh_count_lollipop)

    def count_barbell(self) -> int:
        """COUNT(*) of Barbell B3,1 on the undirected data (eh_count_barbell), exact (128-bit)."""
        return self._count128(lib().eh_count_barbell)

    def stats(self) -> Stats:
        st = EHStats()
        if lib().eh_graph_stats(self._h, ctypes.byref(st)) != EH_OK:
            _raise()
        return Stats(**{f: int(getattr(st, f)) for f, _ in EHStats._fields_})

    def export(self):
        """(row_ptr u64[n+1], col u32[m], orig_id u32[n], is_bitset u8[n]) on the host."""
        st = self.stats()
        n, m = st.n_active, st.m_undirected
        row_ptr = np.empty(n + 1, np.uint64)
        col = np.empty(max(m, 1), np.uint32)
        orig = np.empty(max(n, 1), np.uint32)
        isb = np.empty(max(n, 1), np.uint8)
        if lib().eh_graph_export(self._h, row_ptr.ctypes.data, col.ctypes.data, orig.ctypes.data,
                                 isb.ctypes.data) != EH_OK:
            _raise()
        return row_ptr, col[:m], orig[:n], isb[:n]


def launch_count() -> int:
    """Kernels launched by libeh in this process (eh_launch_count)."""
    return int(lib().eh_launch_count())


def count_batch(lists, query: str = "triangles", *, stream=None, tau: int = 0, all_uint: bool = False) -> list:
    """eh_count_batch: load + count + free for each (src, dst) of `lists` (host
    arrays; pinned torch tensors let the upload of list i+1 overlap the work on
    list i).  query: "triangles" or "4cliques".  Returns the counts."""
    L = lib()
    k = len(lists)
    keep = []
    ps = (ctypes.c_void_p * max(k, 1))()
    pd = (ctypes.c_void_p * max(k, 1))()
    ns = (ctypes.c_uint64 * max(k, 1))()
    for i, (src, dst) in enumerate(lists):
        a, adev, ka = _ptr_of(src)
        b, bdev, kb = _ptr_of(dst)
        if adev or bdev:
            raise ValueError("count_batch takes host arrays")
        if _numel(src) != _numel(dst):
            raise ValueError("src and dst differ in length")
        keep += [ka, kb]
        ps[i], pd[i], ns[i] = a, b, _numel(src)
    cfg = EHConfig()
    cfg.bitset_tau = tau
    cfg.flags = EH_ALL_UINT if all_uint else 0
    if stream is not None:
        cfg.stream = getattr(stream, "cuda_stream", stream)
    out = (ctypes.c_uint64 * max(k, 1))()
    q = {"triangles": 0, "4cliques": 1}[query]
    if L.eh_count_batch(ps, pd, ns, k, q, ctypes.byref(cfg), out) != EH_OK:
        _raise()
    return [int(out[i]) for i in range(k)]


def release_cached_memory() -> None:
    """Give the device memory libeh keeps idle back to the driver (eh_release_cached_memory)."""
    lib().eh_release_cached_memory()


def load_edges(src, dst, **kw) -> Graph:
    return Graph(src, dst, **kw)


def count_triangles(g: Graph) -> int:
    return g.count_triangles()


def count_4cliques(g: Graph) -> int:
    return g.count_4cliques()


def intersect(a, b, *, count_only: bool = False):
    """eh_intersect.  Host inputs -> numpy result; CUDA tensors -> CUDA tensor result."""
    L = lib()
    pa, adev, ka = _ptr_of(a)
    pb, bdev, kb = _ptr_of(b)
    na, nb = _numel(a), _numel(b)
    cap = min(na, nb)
    out = None
    pout = None
    if not count_only:
        if adev or bdev:
            import torch
            dev = ka.device if adev else kb.device
            out = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            pout = out.data_ptr()
        else:
            out = np.empty(max(cap, 1), np.uint32)
            pout = out.ctypes.data
    r = L.eh_intersect(pa, na, pb, nb, pout)
    if r < 0:
        raise EHError(int(r), (L.eh_last_error() or b"").decode())
    if count_only:
        return int(r)
    return out[:r]
