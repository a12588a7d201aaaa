"""paper_2505_12065_b200 -- B200-native top-k inner-product retrieval (SearchAgent-X's
retrieval step, arXiv 2505.12065) behind the C ABI in include/sa.h.

This module is a thin ctypes binding: argument marshalling only.  Every step
of the search runs in libsa.so's sm_100a kernels; torch is used for device
memory, streams and process groups.  There is no CPU fallback: importing the
binding without the built library raises.

Function names mirror the C ABI (sa_index_build, sa_search, ...); the `Index`
class is the same calls with RAII.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# SA_LIBRARY=tuning loads libsa_tuning.so (build.py --tuning: the same code, honouring the
# timing-experiment switches); bench.py refuses it.
TUNING = os.environ.get("SA_LIBRARY", "") == "tuning"
_SO = os.path.join(_PKG, "libsa_tuning.so" if TUNING else "libsa.so")

SA_OK, SA_ERR_INVALID_ARG, SA_ERR_STATE, SA_ERR_OOM, SA_ERR_CUDA, SA_ERR_NCCL, SA_ERR_UNSUPPORTED = range(7)
SA_BF16, SA_F32 = 0, 1
SA_GRAPH_FP8 = 1   # sa_search_graph_ex flag (include/sa.h)
KERNEL_KINDS = ("flat_scan", "merge", "stage", "ivf_probe", "ivf_scan", "other", "graph_search")


class SAError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


class _BuildOpts(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int),
        ("kmeans_iters", ctypes.c_int32),
        ("train_per_list", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("row_offset", ctypes.c_int64),
        ("n_total", ctypes.c_int64),
        ("comm", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("centroids", ctypes.c_void_p),
        ("list_shard_world", ctypes.c_int32),
        ("list_shard_rank", ctypes.c_int32),
    ]


class _MaturityOpts(ctypes.Structure):
    _fields_ = [
        ("tau", ctypes.c_double),
        ("window", ctypes.c_int32),
        ("check_every", ctypes.c_int32),
        ("engine_ready", ctypes.c_void_p),
    ]


_lib = None


def _maturity_opts(tau, window, check_every, engine_ready):
    o = _MaturityOpts()
    o.tau = float(tau)
    o.window = int(window)
    o.check_every = int(check_every)
    if engine_ready is not None:
        if engine_ready.dtype != torch.int32 or engine_ready.numel() < 1 or \
                not (engine_ready.is_cuda or engine_ready.is_pinned()):
            raise ValueError("engine_ready must be an int32 CUDA or pinned host tensor")
        o.engine_ready = engine_ready.data_ptr()
    return o


def lib() -> ctypes.CDLL:
    """Load libsa.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: run `python -m paper_2505_12065_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(_SO)
    P, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    st = ctypes.c_int
    sigs = {
        "sa_build_opts_default": (None, [ctypes.POINTER(_BuildOpts)]),
        "sa_index_build": (st, [P, i64, i32, i32, ctypes.POINTER(P)]),
        "sa_index_build_ex": (st, [P, i64, i32, i32, ctypes.POINTER(_BuildOpts), ctypes.POINTER(P)]),
        "sa_search": (st, [P, P, i64, i32, i32, P, P, P]),
        "sa_search_ex": (st, [P, P, ctypes.c_int, i64, i32, i32, P, P, P]),
        "sa_search_host": (st, [P, P, ctypes.c_int, i64, i32, i32, P, P, P]),
        "sa_search_keys": (st, [P, P, ctypes.c_int, i64, i32, i32, P, P]),
        "sa_merge_keys": (st, [P, i32, i64, i32, P, P, P]),
        "sa_index_free": (st, [P]),
        "sa_comm_unique_id": (st, [P]),
        "sa_comm_init": (st, [P, i32, i32, i32, ctypes.POINTER(P)]),
        "sa_comm_free": (st, [P]),
        "sa_comm_group_create": (st, [i32, ctypes.POINTER(P)]),
        "sa_comm_group_free": (st, [P]),
        "sa_comm_init_local": (st, [P, i32, i32, ctypes.POINTER(P)]),
        "sa_comm_set_checks": (st, [P, i32]),
        "sa_comm_set_collectives": (st, [P, i32]),
        "sa_comm_info": (st, [P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "sa_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "sa_last_error": (ctypes.c_char_p, []),
        "sa_index_info": (st, [P, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i32),
                               ctypes.POINTER(i64)]),
        "sa_index_export_centroids": (st, [P, P]),
        "sa_index_export_lists": (st, [P, P, P]),
        "sa_search_probes": (st, [P, P, i64, i32, P, P]),
        "sa_priority_order": (st, [i64, P, P, P, P, P, i32, P, P]),
        "sa_index_build_graph": (st, [P, i32, i32, i32, i32, P]),
        "sa_search_graph": (st, [P, P, ctypes.c_int, i64, i32, i32, i32, i32, i32, P, P, P, P]),
        "sa_index_export_graph": (st, [P, ctypes.POINTER(i32), ctypes.POINTER(i32), P, P]),
        "sa_index_import_graph": (st, [P, i32, P]),
        "sa_search_graph_host": (st, [P, P, ctypes.c_int, i64, i32, i32, i32, i32, i32, P, P, P]),
        "sa_search_graph_ex": (st, [P, P, ctypes.c_int, i64, i32, i32, i32, i32, i32, i32, P, P, P,
                                    P]),
        "sa_index_build_fp8": (st, [P, P]),
        "sa_search_fp8": (st, [P, P, ctypes.c_int, i64, i32, i32, i32, P, P, P]),
        "sa_index_export_fp8": (st, [P, P, ctypes.POINTER(i32)]),
        "sa_search_graph_mature": (st, [P, P, ctypes.c_int, i64, i32, i32, i32, i32, i32,
                                        ctypes.POINTER(_MaturityOpts), P, P, P, P, P, i32, P]),
        "sa_retriever_create": (st, [P, i32, i32, i32, i32, ctypes.POINTER(P)]),
        "sa_retriever_submit": (st, [P, P, i32, i32, i32, i32, ctypes.POINTER(_MaturityOpts),
                                     ctypes.POINTER(i64)]),
        "sa_retriever_submit_graph": (st, [P, P, i32, i32, i32, i32, i32, i32,
                                           ctypes.POINTER(_MaturityOpts), ctypes.POINTER(i64)]),
        "sa_retriever_poll": (st, [P, i64, ctypes.POINTER(i32)]),
        "sa_retriever_result": (st, [P, i64, P, P, P]),
        "sa_retriever_set_engine_ready": (st, [P, i32]),
        "sa_retriever_free": (st, [P]),
        "sa_search_mature": (st, [P, P, ctypes.c_int, i64, i32, i32, ctypes.POINTER(_MaturityOpts),
                                  P, P, P, P, P, P]),
        "sa_debug_scores": (st, [P, P, i64, P, P]),
        "sa_debug_small_phases": (st, [P, P, i64, i32, i32, P, P, P, P, P]),
        "sa_debug_mature_stages": (st, [P, P, i64, i32, i32, ctypes.POINTER(_MaturityOpts), P, P,
                                        P, P, P]),
        "sa_profile_enable": (st, [i32]),
        "sa_profile_read": (st, [i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols():
    import re
    hdr = open(os.path.join(os.path.dirname(_PKG), "include", "sa.h")).read()
    return sorted(set(re.findall(r"\b(sa_[a-z_0-9]+)\s*\(", hdr)))


def status_string(s: int) -> str:
    try:
        return lib().sa_status_string(int(s)).decode()
    except ImportError:
        return str(s)


def last_error() -> str:
    return lib().sa_last_error().decode()


def _check(status: int):
    if status != SA_OK:
        raise SAError(status, last_error())


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return SA_BF16
    if t.dtype == torch.float32:
        return SA_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or f32)")


# ----------------------------------------------------------------- comm
class Comm:
    """Communicator of a row-sharded index: NCCL (one process per GPU; unique id exchanged
    via torch.distributed) or a rank of an in-process group (local_group)."""

    def __init__(self, handle, rank, world, group=None):
        self.handle, self.rank, self.world = handle, rank, world
        self._group = group

    @classmethod
    def local_group(cls, world: int, devices=None):
        """sa_comm_group_create + sa_comm_init_local: `world` in-process ranks (each must be
        driven from its own thread) on `devices` (default: the current device for all)."""
        g = ctypes.c_void_p()
        _check(lib().sa_comm_group_create(world, ctypes.byref(g)))
        grp = _LocalGroup(g, world)
        comms = []
        for r in range(world):
            dev = torch.cuda.current_device() if devices is None else devices[r]
            h = ctypes.c_void_p()
            _check(lib().sa_comm_init_local(g, r, dev, ctypes.byref(h)))
            comms.append(cls(h, r, world, grp))
        return comms

    def set_checks(self, on: bool = True):
        """sa_comm_set_checks: cross-rank argument check before every sharded search."""
        _check(lib().sa_comm_set_checks(self.handle, 1 if on else 0))
        return self

    def set_collectives(self, on: bool = True):
        """sa_comm_set_collectives: the sharded path (broadcasts, all-gather + merge) even at
        world 1 -- one NCCL rank executes the real collective calls."""
        _check(lib().sa_comm_set_collectives(self.handle, 1 if on else 0))
        return self

    @classmethod
    def nccl_single(cls, device: int | None = None):
        """An NCCL communicator of one rank (sa_comm_unique_id + sa_comm_init, world 1)."""
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().sa_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        h = ctypes.c_void_p()
        dev = torch.cuda.current_device() if device is None else device
        _check(lib().sa_comm_init(ctypes.cast(buf, ctypes.c_void_p), 0, 1, dev, ctypes.byref(h)))
        return cls(h, 0, 1)

    def info(self):
        r, w, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().sa_comm_info(self.handle, ctypes.byref(r), ctypes.byref(w), ctypes.byref(n)))
        return dict(rank=r.value, world=w.value, nccl_nranks=n.value)

    @staticmethod
    def exchange_unique_id() -> bytes:
        """Rank 0 creates the 128-byte NCCL unique id (sa_comm_unique_id); torch.distributed
        broadcasts it (works on nccl and gloo process groups)."""
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8)
        if dist.get_rank() == 0:
            buf = (ctypes.c_uint8 * 128)()
            _check(lib().sa_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            uid = uid.cuda()
        dist.broadcast(uid, 0)
        return bytes(uid.cpu().tolist())

    @classmethod
    def from_torch_distributed(cls, device: int | None = None):
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        raw = cls.exchange_unique_id()
        h = ctypes.c_void_p()
        dev = torch.cuda.current_device() if device is None else device
        _check(lib().sa_comm_init(ctypes.c_char_p(raw), rank, world, dev, ctypes.byref(h)))
        return cls(h, rank, world)

    def free(self):
        if self.handle:
            lib().sa_comm_free(self.handle)
            self.handle = None
            if self._group is not None:
                self._group.release()


class _LocalGroup:
    """sa_comm_group handle, freed with its last communicator."""

    def __init__(self, handle, members):
        self.handle, self.members = handle, members

    def release(self):
        self.members -= 1
        if self.members == 0 and self.handle:
            _check(lib().sa_comm_group_free(self.handle))
            self.handle = None


def shard_range(n_total: int, rank: int, world: int):
    """Balanced contiguous split: off_r = r*floor(n/w) + min(r, n mod w)."""
    base, rem = divmod(int(n_total), int(world))
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


# ----------------------------------------------------------------- index
class Index:
    def __init__(self, handle, d):
        self.handle = handle
        self.d = d

    # sa_index_build / sa_index_build_ex
    @classmethod
    def build(cls, corpus: torch.Tensor, nlist: int = 0, *, kmeans_iters: int = 20,
              train_per_list: int = 256, seed: int = 0x5A2505, row_offset: int = 0,
              n_total: int | None = None, comm: Comm | None = None, centroids=None,
              list_shard: tuple[int, int] | None = None, stream=None) -> "Index":
        if not corpus.is_cuda or corpus.dim() != 2 or not corpus.is_contiguous():
            raise ValueError("corpus must be a contiguous 2-D CUDA tensor")
        o = _BuildOpts()
        lib().sa_build_opts_default(ctypes.byref(o))
        o.dtype = _dtype_code(corpus)
        o.kmeans_iters = kmeans_iters
        o.train_per_list = train_per_list
        o.seed = seed
        o.row_offset = row_offset
        o.n_total = n_total if n_total is not None else 0
        o.comm = comm.handle if comm is not None else None
        if list_shard is not None:        # (rank, world): keep lists l % world == rank
            o.list_shard_rank, o.list_shard_world = int(list_shard[0]), int(list_shard[1])
        o.stream = _stream_ptr(stream)
        if centroids is not None:
            if not centroids.is_cuda or centroids.dtype != torch.float32 or \
                    tuple(centroids.shape) != (nlist, corpus.shape[1]):
                raise ValueError("centroids must be a CUDA float32 [nlist, d] tensor")
            centroids = centroids.contiguous()
            o.centroids = centroids.data_ptr()
        h = ctypes.c_void_p()
        _check(lib().sa_index_build_ex(_ptr(corpus), corpus.shape[0], corpus.shape[1], nlist,
                                       ctypes.byref(o), ctypes.byref(h)))
        return cls(h, corpus.shape[1])

    # sa_search / sa_search_ex
    def search(self, queries: torch.Tensor, k: int, nprobe: int = 0, out=None, stream=None):
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        if queries.shape[1] != self.d:
            raise SAError(SA_ERR_INVALID_ARG, f"queries have d={queries.shape[1]}, index d={self.d}")
        nq = queries.shape[0]
        if out is None:
            ids = torch.empty(nq, k, dtype=torch.int64, device=queries.device)
            scores = torch.empty(nq, k, dtype=torch.float32, device=queries.device)
        else:
            ids, scores = out
        _check(lib().sa_search_ex(self.handle, _ptr(queries), _dtype_code(queries), nq, k, nprobe,
                                  _ptr(ids), _ptr(scores), _stream_ptr(stream)))
        return ids, scores

    # sa_search_keys: this shard's sorted packed keys (global ids), int64 view of uint64 [nq, k]
    def search_keys(self, queries: torch.Tensor, k: int, nprobe: int = 0, stream=None):
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        keys = torch.empty(queries.shape[0], k, dtype=torch.int64, device=queries.device)
        _check(lib().sa_search_keys(self.handle, _ptr(queries), _dtype_code(queries),
                                    queries.shape[0], k, nprobe, _ptr(keys), _stream_ptr(stream)))
        return keys

    # sa_search_host: host buffers in and out, copies inside the call
    def search_host(self, queries: torch.Tensor, k: int, nprobe: int = 0, out=None, stream=None):
        if queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D host tensor")
        if queries.shape[1] != self.d:
            raise SAError(SA_ERR_INVALID_ARG, f"queries have d={queries.shape[1]}, index d={self.d}")
        nq = queries.shape[0]
        if out is None:
            ids = torch.empty(nq, k, dtype=torch.int64)
            scores = torch.empty(nq, k, dtype=torch.float32)
        else:
            ids, scores = out
        _check(lib().sa_search_host(self.handle, _ptr(queries), _dtype_code(queries), nq, k, nprobe,
                                    _ptr(ids), _ptr(scores), _stream_ptr(stream)))
        return ids, scores

    # sa_search_mature: IVF search with the non-stall maturity exit (PAPER §3.3)
    def search_mature(self, queries: torch.Tensor, k: int, nprobe_max: int, *, tau: float,
                      window: int, check_every: int = 1, engine_ready: torch.Tensor | None = None,
                      trace: bool = False, stream=None):
        """Returns (ids, scores, lists_scanned[, rq, ema]).  engine_ready: an int32 tensor of
        one element, pinned host (pin_memory()) or CUDA; None = always ready."""
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        if queries.shape[1] != self.d:
            raise SAError(SA_ERR_INVALID_ARG, f"queries have d={queries.shape[1]}, index d={self.d}")
        nq = queries.shape[0]
        dev = queries.device
        ids = torch.empty(nq, k, dtype=torch.int64, device=dev)
        scores = torch.empty(nq, k, dtype=torch.float32, device=dev)
        t = torch.empty(nq, dtype=torch.int32, device=dev)
        rq = ema = None
        if trace:
            rq = torch.empty(nq, nprobe_max, dtype=torch.float64, device=dev)
            ema = torch.empty(nq, nprobe_max, dtype=torch.float64, device=dev)
        o = _maturity_opts(tau, window, check_every, engine_ready)
        _check(lib().sa_search_mature(self.handle, _ptr(queries), _dtype_code(queries), nq, k,
                                      nprobe_max, ctypes.byref(o), _ptr(ids), _ptr(scores), _ptr(t),
                                      _ptr(rq) if trace else None, _ptr(ema) if trace else None,
                                      _stream_ptr(stream)))
        if trace:
            return ids, scores, t, rq, ema
        return ids, scores, t

    # sa_index_build_graph / sa_search_graph / sa_index_export_graph (proximity graph)
    def build_graph(self, knn_k: int = 64, degree: int = 32, nprobe_build: int = 8,
                    keep_knn: bool = False, stream=None):
        _check(lib().sa_index_build_graph(self.handle, knn_k, degree, nprobe_build,
                                          1 if keep_knn else 0, _stream_ptr(stream)))
        return self

    def search_graph(self, queries: torch.Tensor, k: int, search_range: int, *,
                     search_width: int = 4, n_entries: int = 8, max_iters: int = 1 << 30,
                     expanded: bool = False, fp8: bool = False, stream=None):
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        nq = queries.shape[0]
        ids = torch.empty(nq, k, dtype=torch.int64, device=queries.device)
        scores = torch.empty(nq, k, dtype=torch.float32, device=queries.device)
        ex = torch.empty(2, nq, dtype=torch.int32, device=queries.device) if expanded else None
        _check(lib().sa_search_graph_ex(self.handle, _ptr(queries), _dtype_code(queries), nq, k,
                                        search_range, search_width, n_entries,
                                        min(max_iters, 2**31 - 1), SA_GRAPH_FP8 if fp8 else 0,
                                        _ptr(ids), _ptr(scores), _ptr(ex) if expanded else None,
                                        _stream_ptr(stream)))
        # expanded: (entries expanded [nq], rows scored [nq])
        return (ids, scores, ex[0], ex[1]) if expanded else (ids, scores)

    def search_graph_host(self, queries: torch.Tensor, k: int, search_range: int, *,
                          search_width: int = 4, n_entries: int = 8, fp8: bool = False, out=None,
                          stream=None):
        """sa_search_graph_host: queries a (pinned) CPU tensor; results in CPU tensors."""
        if queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CPU tensor")
        nq = queries.shape[0]
        if out is None:
            ids = torch.empty(nq, k, dtype=torch.int64)
            scores = torch.empty(nq, k, dtype=torch.float32)
        else:
            ids, scores = out
        _check(lib().sa_search_graph_host(self.handle, _ptr(queries), _dtype_code(queries), nq, k,
                                          search_range, search_width, n_entries,
                                          SA_GRAPH_FP8 if fp8 else 0, _ptr(ids), _ptr(scores),
                                          _stream_ptr(stream)))
        return ids, scores

    def search_graph_mature(self, queries: torch.Tensor, k: int, search_range: int, *,
                            tau: float, window: int, check_every: int = 1,
                            engine_ready: torch.Tensor | None = None, search_width: int = 4,
                            n_entries: int = 8, max_iters: int = 1 << 30, trace_cols: int = 0,
                            stream=None):
        """sa_search_graph_mature.  Returns (ids, scores, steps[, rq, ema]) -- rq / ema
        [nq, trace_cols] fp64 when trace_cols > 0."""
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        nq = queries.shape[0]
        dev = queries.device
        ids = torch.empty(nq, k, dtype=torch.int64, device=dev)
        scores = torch.empty(nq, k, dtype=torch.float32, device=dev)
        steps = torch.empty(nq, dtype=torch.int32, device=dev)
        rq = ema = None
        if trace_cols > 0:
            rq = torch.empty(nq, trace_cols, dtype=torch.float64, device=dev)
            ema = torch.empty(nq, trace_cols, dtype=torch.float64, device=dev)
        o = _maturity_opts(tau, window, check_every, engine_ready)
        _check(lib().sa_search_graph_mature(self.handle, _ptr(queries), _dtype_code(queries), nq, k,
                                            search_range, search_width, n_entries,
                                            min(max_iters, 2**31 - 1), ctypes.byref(o), _ptr(ids),
                                            _ptr(scores), _ptr(steps),
                                            _ptr(rq) if rq is not None else None,
                                            _ptr(ema) if ema is not None else None,
                                            trace_cols, _stream_ptr(stream)))
        return (ids, scores, steps, rq, ema) if trace_cols > 0 else (ids, scores, steps)

    # sa_index_build_fp8 / sa_search_fp8 / sa_index_export_fp8 (e4m3 scan + bf16 re-rank)
    def build_fp8(self, stream=None):
        _check(lib().sa_index_build_fp8(self.handle, _stream_ptr(stream)))
        return self

    def search_fp8(self, queries: torch.Tensor, k: int, n_cand: int = 16, nprobe: int = 0,
                   out=None, stream=None):
        if not queries.is_cuda or queries.dim() != 2 or not queries.is_contiguous():
            raise ValueError("queries must be a contiguous 2-D CUDA tensor")
        if queries.shape[1] != self.d:
            raise SAError(SA_ERR_INVALID_ARG, f"queries have d={queries.shape[1]}, index d={self.d}")
        nq = queries.shape[0]
        if out is None:
            ids = torch.empty(nq, k, dtype=torch.int64, device=queries.device)
            scores = torch.empty(nq, k, dtype=torch.float32, device=queries.device)
        else:
            ids, scores = out
        _check(lib().sa_search_fp8(self.handle, _ptr(queries), _dtype_code(queries), nq, k, nprobe,
                                   n_cand, _ptr(ids), _ptr(scores), _stream_ptr(stream)))
        return ids, scores

    def export_fp8(self):
        """(uint8 [n_local, d] e4m3 bytes by local id, scale exponent e)."""
        e = ctypes.c_int32()
        out = np.empty((self.info()["n_local"], self.d), dtype=np.uint8)
        _check(lib().sa_index_export_fp8(self.handle, out.ctypes.data_as(ctypes.c_void_p),
                                         ctypes.byref(e)))
        return out, e.value

    def import_graph(self, nbr: np.ndarray):
        """sa_index_import_graph: nbr int64 [n_local, degree] of global ids (-1 padded)."""
        nbr = np.ascontiguousarray(nbr, dtype=np.int64)
        _check(lib().sa_index_import_graph(self.handle, nbr.shape[1],
                                           nbr.ctypes.data_as(ctypes.c_void_p)))
        return self

    def export_graph(self, knn: bool = False):
        inf = self.info()
        deg, kk = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().sa_index_export_graph(self.handle, ctypes.byref(deg), ctypes.byref(kk),
                                           None, None))
        nbr = np.empty((inf["n_local"], deg.value), dtype=np.int64)
        kn = np.empty((inf["n_local"], kk.value), dtype=np.int64) if knn else None
        _check(lib().sa_index_export_graph(self.handle, ctypes.byref(deg), ctypes.byref(kk),
                                           nbr.ctypes.data_as(ctypes.c_void_p),
                                           kn.ctypes.data_as(ctypes.c_void_p) if knn else None))
        return (nbr, kn) if knn else nbr

    def info(self):
        n = ctypes.c_int64()
        d = ctypes.c_int32()
        nl = ctypes.c_int32()
        off = ctypes.c_int64()
        _check(lib().sa_index_info(self.handle, ctypes.byref(n), ctypes.byref(d), ctypes.byref(nl),
                                   ctypes.byref(off)))
        return dict(n_local=n.value, d=d.value, nlist=nl.value, row_offset=off.value)

    def export_centroids(self) -> np.ndarray:
        inf = self.info()
        out = np.empty((inf["nlist"], inf["d"]), dtype=np.float32)
        _check(lib().sa_index_export_centroids(self.handle, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def export_lists(self):
        inf = self.info()
        off = np.empty(inf["nlist"] + 1, dtype=np.int64)
        ids = np.empty(inf["n_local"], dtype=np.int64)
        _check(lib().sa_index_export_lists(self.handle, off.ctypes.data_as(ctypes.c_void_p),
                                           ids.ctypes.data_as(ctypes.c_void_p)))
        return off, ids

    def probes(self, queries: torch.Tensor, nprobe: int, stream=None) -> torch.Tensor:
        out = torch.empty(queries.shape[0], nprobe, dtype=torch.int32, device=queries.device)
        _check(lib().sa_search_probes(self.handle, _ptr(queries), queries.shape[0], nprobe,
                                      _ptr(out), _stream_ptr(stream)))
        return out

    def debug_small_phases(self, queries: torch.Tensor, k: int, nprobe: int, stream=None):
        """The one-launch agent-step search with per-CTA phase timestamps (ns, [grid, 8])."""
        nq = queries.shape[0]
        ids = torch.empty(nq, k, dtype=torch.int64, device=queries.device)
        sc = torch.empty(nq, k, dtype=torch.float32, device=queries.device)
        ns = np.zeros(1024 * 8, dtype=np.int64)
        grid = ctypes.c_int32(0)
        _check(lib().sa_debug_small_phases(self.handle, _ptr(queries), nq, k, nprobe, _ptr(ids),
                                           _ptr(sc), ns.ctypes.data_as(ctypes.c_void_p),
                                           ctypes.byref(grid), _stream_ptr(stream)))
        return ids, sc, ns[:grid.value * 8].reshape(grid.value, 8)

    def debug_mature_stages(self, queries: torch.Tensor, k: int, nprobe_max: int, *, tau: float,
                            window: int, check_every: int = 1, stream=None):
        """One-launch maturity search with per-stage timestamps (ns, [64, 4])."""
        nq = queries.shape[0]
        ids = torch.empty(nq, k, dtype=torch.int64, device=queries.device)
        sc = torch.empty(nq, k, dtype=torch.float32, device=queries.device)
        t = torch.empty(nq, dtype=torch.int32, device=queries.device)
        ns = np.zeros(64 * 4, dtype=np.int64)
        o = _maturity_opts(tau, window, check_every, None)
        _check(lib().sa_debug_mature_stages(self.handle, _ptr(queries), nq, k, nprobe_max,
                                            ctypes.byref(o), _ptr(ids), _ptr(sc), _ptr(t),
                                            ns.ctypes.data_as(ctypes.c_void_p),
                                            _stream_ptr(stream)))
        return ids, sc, t, ns.reshape(64, 4)

    def debug_scores(self, queries: torch.Tensor, stream=None) -> torch.Tensor:
        n = self.info()["n_local"]
        out = torch.empty(queries.shape[0], n, dtype=torch.float32, device=queries.device)
        _check(lib().sa_debug_scores(self.handle, _ptr(queries), queries.shape[0], _ptr(out),
                                     _stream_ptr(stream)))
        return out

    def free(self):
        if self.handle:
            lib().sa_index_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sa_merge_keys(keys: torch.Tensor, stream=None):
    """Final merge of per-rank key lists: keys int64 (uint64 bits) CUDA [w, nq, k]."""
    w, nq, k = keys.shape
    keys = keys.contiguous()
    ids = torch.empty(nq, k, dtype=torch.int64, device=keys.device)
    scores = torch.empty(nq, k, dtype=torch.float32, device=keys.device)
    _check(lib().sa_merge_keys(_ptr(keys), w, nq, k, _ptr(ids), _ptr(scores), _stream_ptr(stream)))
    return ids, scores


# C-ABI-named aliases
def sa_index_build(corpus, nlist=0, **kw) -> Index:
    return Index.build(corpus, nlist, **kw)


def sa_search(index: Index, queries, k, nprobe=0, out=None, stream=None):
    return index.search(queries, k, nprobe, out, stream)


def sa_search_host(index: Index, queries, k, nprobe=0, out=None, stream=None):
    return index.search_host(queries, k, nprobe, out, stream)


def sa_search_mature(index: Index, queries, k, nprobe_max, **kw):
    return index.search_mature(queries, k, nprobe_max, **kw)


def sa_priority_order(R, W_us, C, Wcur_us, ids, G: int = 6):
    """PAPER §3.2 Eq. 1-2 priority order of waiting sequences (host).  Returns (order as
    input positions, levels)."""
    arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in (R, W_us, C, Wcur_us, ids)]
    n = arrs[0].shape[0]
    lv = np.empty(n, dtype=np.int32)
    order = np.empty(n, dtype=np.int64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib().sa_priority_order(n, *[ptr(a) for a in arrs], G, ptr(lv), ptr(order)))
    return order, lv


class Retriever:
    """Asynchronous retrieval tasks (Alg. 1 LaunchAsyncRetrievalTask / getResult) over an
    index: submit() never blocks; poll() is an event query; result() copies out."""

    def __init__(self, index: Index, streams: int = 1, slots: int = 8, max_nq: int = 64,
                 max_k: int = 16):
        self.index = index
        self.max_k = max_k
        h = ctypes.c_void_p()
        _check(lib().sa_retriever_create(index.handle, streams, slots, max_nq, max_k,
                                         ctypes.byref(h)))
        self.handle = h
        self._shape = {}

    def submit(self, queries: np.ndarray, k: int, nprobe_max: int, *, mature: bool = False,
               tau: float = 0.0, window: int = 1, check_every: int = 1) -> int:
        q = np.ascontiguousarray(queries, dtype=np.float32)
        o = _MaturityOpts()
        o.tau, o.window, o.check_every = float(tau), int(window), int(check_every)
        t = ctypes.c_int64()
        _check(lib().sa_retriever_submit(self.handle, q.ctypes.data_as(ctypes.c_void_p),
                                         q.shape[0], k, nprobe_max, int(mature), ctypes.byref(o),
                                         ctypes.byref(t)))
        self._shape[t.value] = (q.shape[0], k)
        return t.value

    def submit_graph(self, queries: np.ndarray, k: int, search_range: int, *,
                     search_width: int = 4, n_entries: int = 16, mature: bool = False,
                     tau: float = 0.0, window: int = 1, check_every: int = 1) -> int:
        q = np.ascontiguousarray(queries, dtype=np.float32)
        o = _MaturityOpts()
        o.tau, o.window, o.check_every = float(tau), int(window), int(check_every)
        t = ctypes.c_int64()
        _check(lib().sa_retriever_submit_graph(self.handle, q.ctypes.data_as(ctypes.c_void_p),
                                               q.shape[0], k, search_range, search_width,
                                               n_entries, int(mature), ctypes.byref(o),
                                               ctypes.byref(t)))
        self._shape[t.value] = (q.shape[0], k)
        return t.value

    def poll(self, task: int) -> bool:
        done = ctypes.c_int32()
        _check(lib().sa_retriever_poll(self.handle, task, ctypes.byref(done)))
        return bool(done.value)

    def result(self, task: int):
        nq, k = self._shape.pop(task)
        ids = np.empty((nq, k), dtype=np.int64)
        sc = np.empty((nq, k), dtype=np.float32)
        lists = np.empty(nq, dtype=np.int32)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _check(lib().sa_retriever_result(self.handle, task, ptr(ids), ptr(sc), ptr(lists)))
        return ids, sc, lists

    def set_engine_ready(self, ready: bool):
        _check(lib().sa_retriever_set_engine_ready(self.handle, int(bool(ready))))

    def free(self):
        if self.handle:
            lib().sa_retriever_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sa_index_free(index: Index):
    index.free()


# ----------------------------------------------------------------- accounting
def profile_enable(on: bool = True):
    _check(lib().sa_profile_enable(1 if on else 0))


def profile_read(kind: str | int):
    kid = KERNEL_KINDS.index(kind) if isinstance(kind, str) else int(kind)
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(lib().sa_profile_read(kid, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value
