"""paper_2201_01257_b200 -- thin Python binding of libtt (include/tt.h).

Argument marshalling only: every step of the hot path runs in libtt's sm_100a kernels.  There is no
CPU fallback: importing this package fails loudly if ``libtt.so`` is missing (build it with
``python -m paper_2201_01257_b200.build`` or ``__graft_entry__.build()``), and every device call on
a machine without a B200 returns an error from the library.

Names follow the C ABI (and the paper's vocabulary, P111-174): IndexSpace, TiledIndexSpace, Tensor,
set_/add/contract/contract_scalar, task_list, partition_lpt, gather_plan.  Device memory is supplied
by the caller (e.g. a torch tensor); pointers are passed as integers (``t.data_ptr()``).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtt.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtt.so not found at {LIB_PATH}: build it with `python -m paper_2201_01257_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

TT_OK = 0
ERRORS = {-1: "TT_E_ARG", -2: "TT_E_COVERAGE", -3: "TT_E_LABEL", -4: "TT_E_TILING", -5: "TT_E_ZERO_BLOCK",
          -6: "TT_E_UNBOUND", -7: "TT_E_OOM", -8: "TT_E_CUDA", -9: "TT_E_NCCL", -10: "TT_E_STATE",
          -11: "TT_E_UNSUPPORTED", -12: "TT_E_WORKSPACE"}
TT_E_WORKSPACE = -12
HOST_C_IN, HOST_C_OUT = 1, 2
# default device workspace per context (tt_workspace_bind): plan metadata and scratch; cached plans are
# evicted least-recently-used when it is full.  Override with Context(workspace_bytes=...) or TT_WORKSPACE_MB.
DEFAULT_WORKSPACE_BYTES = int(os.environ.get("TT_WORKSPACE_MB", "256")) << 20
TT_REPLICATED = -2
TT_SPLIT = -3
KIND_UNIFORM, KIND_INTEGER = 0, 1

_vp, _i32, _i64, _u32, _u64, _dbl = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                     ctypes.c_uint64, ctypes.c_double)
_P = ctypes.POINTER


class Stats(ctypes.Structure):
    _fields_ = [("c_blocks", _i64), ("tasks", _i64), ("work_items", _i64), ("flops", _dbl), ("bytes", _dbl),
                ("gathered_bytes", _i64), ("launches", _i64), ("plan_cached", _i32), ("kernel_variant", _i32),
                ("producer", _i32), ("aux_flops", _dbl)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Contract3Info(ctypes.Structure):
    _fields_ = [("pair", _i32), ("i_lbl", ctypes.c_char * 9), ("flops", _dbl * 3), ("naive_macs", _dbl),
                ("ws_elems", _i64)]

    def as_dict(self):
        return {"pair": self.pair, "i_lbl": self.i_lbl.decode(), "flops": list(self.flops),
                "naive_macs": self.naive_macs, "ws_elems": self.ws_elems}


class TriplesInfo(ctypes.Structure):
    _fields_ = [("w_blocks_total", _i64), ("w_blocks", _i64), ("batches", _i64), ("flops_alg", _dbl),
                ("flops_exec", _dbl), ("ws_elems", _i64), ("cost_rank", _dbl), ("cost_total", _dbl),
                ("cost_max_unit", _dbl)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "tt_ctx_create": [_i32, _vp, _i32, _i32, _vp, _P(_vp)],
    "tt_ctx_destroy": [_vp],
    "tt_sim_create": [_i32, _i32, _P(_vp)],
    "tt_sim_destroy": [_vp],
    "tt_ctx_create_sim": [_vp, _i32, _vp, _P(_vp)],
    "tt_nccl_unique_id": [_vp],
    "tt_ctx_set_profiling": [_vp, _i32],
    "tt_profile_read": [_vp, ctypes.c_char_p, _P(_dbl), _P(_i64)],
    "tt_profile_reset": [_vp],
    "tt_last_stats": [_vp, _P(Stats)],
    "tt_launch_count": [_vp, _P(_i64)],
    "tt_sync": [_vp],
    "tt_workspace_bind": [_vp, _vp, _i64],
    "tt_workspace_bytes": [_vp, _P(_i64)],
    "tt_workspace_info": [_vp, _P(_i64), _P(_i64), _P(_i64)],
    "tt_ctx_set_plan_limit": [_vp, _i64],
    "tt_ctx_clear_plans": [_vp],
    "tt_is_create": [_i64, _i32, _vp, _vp, _P(_vp)],
    "tt_is_destroy": [_vp],
    "tt_tis_fixed": [_vp, _i64, _P(_vp)],
    "tt_tis_custom": [_vp, _i32, _vp, _P(_vp)],
    "tt_tis_info": [_vp, _P(_i32), _P(_P(_i64)), _P(_P(ctypes.c_int8))],
    "tt_tis_destroy": [_vp],
    "tt_tis_sub": [_vp, _i64, _i64, _P(_vp)],
    "tt_tis_range": [_vp, _i32, _P(_vp)],
    "tt_tensor_view": [_vp, _vp, _P(_vp)],
    "tt_tensor_create": [_vp, _i32, _vp, _vp, _P(_vp)],
    "tt_tensor_create_spin": [_vp, _i32, _vp, _u32, _u32, _P(_vp)],
    "tt_tensor_info": [_vp, _P(_i32), _P(_i64), _P(_i64)],
    "tt_tensor_layout": [_vp, _P(_i64), _P(_P(_i64)), _P(_P(_i32)), _P(_P(ctypes.c_uint8))],
    "tt_tensor_set_owner": [_vp, _vp],
    "tt_tensor_set_parts": [_vp, _i64, _vp, _vp, _vp, _vp],
    "tt_tensor_parts": [_vp, _P(_i64), _P(_P(_i64)), _P(_P(_i32)), _P(_P(_i32)), _P(_P(_i32))],
    "tt_tensor_bind": [_vp, _vp, _i64],
    "tt_tensor_upload": [_vp, _vp, _vp],
    "tt_tensor_download": [_vp, _vp, _vp],
    "tt_tensor_destroy": [_vp],
    "tt_fill_synthetic": [_vp, _vp, _u64, _u32, _i32],
    "tt_set": [_vp, _vp, _dbl],
    "tt_add": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p],
    "tt_contract": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p],
    "tt_contract_cholesky": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp,
                             _i64],
    "tt_contract_prefetch": [_vp, _vp, ctypes.c_char_p, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p],
    "tt_contract_host": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, _vp,
                         _vp, _i32],
    "tt_contract3": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp,
                     ctypes.c_char_p, _vp, _i64, _vp],
    "tt_triples_energy": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _P(_dbl), _vp],
    "tt_contract_scalar": [_vp, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _P(_dbl)],
    "tt_task_list": [_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _i32, _vp, _vp, _vp,
                     _vp, _vp, _i64, _P(_i64), _P(_i64)],
    "tt_partition_lpt": [_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _u32, _vp],
    "tt_partition_split": [_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _u32],
    "tt_partition_split_cost": [_vp, _vp, _vp, _u32],
    "tt_partition_split_cholesky": [_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _u32],
    "tt_tensor_set_compact": [_vp, _i32],
    "tt_tensor_storage": [_vp, _P(_i64), _P(_P(_i64))],
    "tt_gather_plan": [_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, _P(_i64), _vp,
                       _P(_i64), _i64],
    "tt_sched_create": [_vp, _i32, _P(_vp)],
    "tt_sched_destroy": [_vp],
    "tt_sched_set": [_vp, _vp, _dbl],
    "tt_sched_add": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p],
    "tt_sched_contract": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p],
    "tt_sched_contract_cholesky": [_vp, _vp, ctypes.c_char_p, _dbl, _dbl, _vp, ctypes.c_char_p, _vp,
                                   ctypes.c_char_p, _vp, _i64],
    "tt_sched_scalar": [_vp, _dbl, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _P(_dbl)],
    "tt_sched_levels": [_vp, _vp, _P(_i64), _P(_i32)],
    "tt_sched_execute": [_vp],
    "tt_sched_capture": [_vp],
    "tt_sched_replay": [_vp],
    "tt_sched_stats": [_vp, _P(_i64), _P(_i64)],
    "tt_last_error": [],
    "tt_version": [],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _i32
_lib.tt_last_error.restype = ctypes.c_char_p

EXPORTED = tuple(_SIGS)


class TTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.name = ERRORS.get(code, str(code))


def _check(status: int):
    if status != TT_OK:
        raise TTError(status, _lib.tt_last_error().decode(errors="replace"))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp) if a is not None else None


def _b(s: str) -> bytes:
    return s.encode()


def _devptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def version() -> int:
    return _lib.tt_version()


def last_error() -> str:
    return _lib.tt_last_error().decode(errors="replace")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.tt_nccl_unique_id(buf))
    return buf.raw


class SimGroup:
    """Simulated ranks on one GPU (tt_sim_create): ``Context(stream=..., rank=r, sim=group)`` per rank,
    each rank driven by its own host thread (SPMD); gathers become device copies between the ranks'
    buffers, the all-reduce a rank-order sum."""

    def __init__(self, device: int, nranks: int):
        h = _vp()
        _check(_lib.tt_sim_create(device, nranks, ctypes.byref(h)))
        self.h, self.device, self.nranks = h, device, nranks

    def close(self):
        if self.h:
            _check(_lib.tt_sim_destroy(self.h))
            self.h = None


class Context:
    """ExecutionContext (P178-188).  device=-1 gives a host-only context (metadata only); ``sim`` = a
    SimGroup: simulated rank ``rank`` of that group (device and nranks come from the group).  A device
    context gets its workspace (tt_workspace_bind) from torch: ``workspace_bytes`` (default
    DEFAULT_WORKSPACE_BYTES); ``bind_workspace`` re-binds a larger one."""

    def __init__(self, device: int = 0, stream: int = 0, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, sim: Optional[SimGroup] = None,
                 workspace_bytes: Optional[int] = None):
        h = _vp()
        if sim is not None:
            _check(_lib.tt_ctx_create_sim(_vp(stream or 0), rank, sim.h, ctypes.byref(h)))
            device, nranks = sim.device, sim.nranks
        else:
            idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            _check(_lib.tt_ctx_create(device, _vp(stream or 0), rank, nranks, idbuf, ctypes.byref(h)))
        self.h, self.device, self.rank, self.nranks, self.sim = h, device, rank, nranks, sim
        self._ws = None
        if device >= 0:
            self.bind_workspace(workspace_bytes or DEFAULT_WORKSPACE_BYTES)

    def bind_workspace(self, nbytes: int):
        """tt_workspace_bind with a fresh torch buffer of ``nbytes`` on the context's device (the old
        buffer is released after the library has re-bound; it synchronises the device first)."""
        import torch
        buf = torch.empty(int(nbytes), dtype=torch.uint8, device=f"cuda:{self.device}")
        _check(_lib.tt_workspace_bind(self.h, _vp(buf.data_ptr()), int(nbytes)))
        self._ws = buf

    def workspace_bytes(self) -> int:
        n = _i64()
        _check(_lib.tt_workspace_bytes(self.h, ctypes.byref(n)))
        return n.value

    def workspace_info(self) -> dict:
        b, l, h = _i64(), _i64(), _i64()
        _check(_lib.tt_workspace_info(self.h, ctypes.byref(b), ctypes.byref(l), ctypes.byref(h)))
        return {"bound": b.value, "live": l.value, "high": h.value}

    def set_plan_limit(self, n: int):
        _check(_lib.tt_ctx_set_plan_limit(self.h, int(n)))

    def clear_plans(self):
        _check(_lib.tt_ctx_clear_plans(self.h))

    def close(self):
        if self.h:
            _check(_lib.tt_ctx_destroy(self.h))
            self.h = None
            self._ws = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        _check(_lib.tt_sync(self.h))

    def set_profiling(self, on: bool):
        _check(_lib.tt_ctx_set_profiling(self.h, 1 if on else 0))

    def profile(self, kernel: str = ""):
        ms, n = _dbl(), _i64()
        _check(_lib.tt_profile_read(self.h, _b(kernel), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def profile_reset(self):
        _check(_lib.tt_profile_reset(self.h))

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.tt_last_stats(self.h, ctypes.byref(s)))
        return s.as_dict()

    def launches(self) -> int:
        n = _i64()
        _check(_lib.tt_launch_count(self.h, ctypes.byref(n)))
        return n.value


class IndexSpace:
    """IndexSpace (P116-122).  ``ranges`` = [(begin, end)], ``spins`` = [+1/-1] per range (P138),
    ``names`` = optional names of the ranges (P120-121 "first"/"second"; used by TiledIndexSpace(name))."""

    def __init__(self, extent: int, ranges: Optional[Sequence] = None, spins: Optional[Sequence[int]] = None,
                 names: Optional[Sequence[str]] = None):
        self.names = list(names or [])
        h = _vp()
        be = np.asarray([x for r in (ranges or []) for x in r], dtype=np.int64)
        sp = np.asarray(spins, dtype=np.int8) if spins is not None else None
        _check(_lib.tt_is_create(extent, len(ranges or []), _ptr(be) if len(be) else None, _ptr(sp),
                                 ctypes.byref(h)))
        self.h, self.extent = h, extent

    def __del__(self):  # pragma: no cover
        try:
            _lib.tt_is_destroy(self.h)
        except Exception:
            pass


class TiledIndexSpace:
    """TiledIndexSpace (P125-127): fixed ``tile`` or custom ``sizes``.  ``tis("first")`` / ``tis.sub(b, e)``
    give the sub-space of a named range / of [b, e) (P152, P159; tt_tis_range / tt_tis_sub)."""

    def __init__(self, space: IndexSpace, tile: Optional[int] = None, sizes: Optional[Sequence[int]] = None,
                 _handle=None, _parent=None):
        h = _vp()
        self.parent = _parent
        if _handle is not None:
            h = _handle
        elif sizes is not None:
            s = np.asarray(sizes, dtype=np.int64)
            _check(_lib.tt_tis_custom(space.h, len(s), _ptr(s), ctypes.byref(h)))
        else:
            _check(_lib.tt_tis_fixed(space.h, int(tile), ctypes.byref(h)))
        self.h, self.space = h, space
        n = _i32()
        off = _P(_i64)()
        sp = _P(ctypes.c_int8)()
        _check(_lib.tt_tis_info(h, ctypes.byref(n), ctypes.byref(off), ctypes.byref(sp)))
        self.ntiles = n.value
        self.offsets = np.ctypeslib.as_array(off, (n.value + 1,)).copy()
        self.spin = np.ctypeslib.as_array(sp, (n.value,)).copy() if n.value else np.zeros(0, np.int8)
        self.extent = int(self.offsets[-1])

    def sub(self, begin: int, end: int) -> "TiledIndexSpace":
        h = _vp()
        _check(_lib.tt_tis_sub(self.h, int(begin), int(end), ctypes.byref(h)))
        return TiledIndexSpace(self.space, _handle=h, _parent=self)

    def __call__(self, name) -> "TiledIndexSpace":
        r = self.space.names.index(name) if isinstance(name, str) else int(name)
        h = _vp()
        _check(_lib.tt_tis_range(self.h, r, ctypes.byref(h)))
        return TiledIndexSpace(self.space, _handle=h, _parent=self)

    def __del__(self):  # pragma: no cover
        try:
            _lib.tt_tis_destroy(self.h)
        except Exception:
            pass


class Tensor:
    """Tensor<double> (P129-140) with a non-zero block map: explicit ``nz`` (u8 per block, row-major)
    or the spin rule ``spin=(upper_dims, lower_dims)`` (reading R7)."""

    def __init__(self, ctx: Context, dims: Sequence[TiledIndexSpace], nz=None, spin=None, _view_of=None):
        h = _vp()
        arr = (_vp * len(dims))(*[d.h.value if isinstance(d.h, _vp) else d.h for d in dims])
        self.parent = _view_of
        if _view_of is not None:
            _check(_lib.tt_tensor_view(_view_of.h, arr, ctypes.byref(h)))
        elif spin is not None:
            up = sum(1 << d for d in spin[0])
            lo = sum(1 << d for d in spin[1])
            _check(_lib.tt_tensor_create_spin(ctx.h, len(dims), arr, up, lo, ctypes.byref(h)))
        else:
            z = np.ascontiguousarray(nz, dtype=np.uint8) if nz is not None else None
            _check(_lib.tt_tensor_create(ctx.h, len(dims), arr, _ptr(z), ctypes.byref(h)))
        self.h, self.ctx, self.dims = h, ctx, list(dims)
        self._refresh()
        self.storage = None

    def _refresh(self):
        order, nb, nnz = _i32(), _i64(), _i64()
        _check(_lib.tt_tensor_info(self.h, ctypes.byref(order), ctypes.byref(nb), ctypes.byref(nnz)))
        pe = _i64()
        bo, ow, z = _P(_i64)(), _P(_i32)(), _P(ctypes.c_uint8)()
        _check(_lib.tt_tensor_layout(self.h, ctypes.byref(pe), ctypes.byref(bo), ctypes.byref(ow), ctypes.byref(z)))
        self.order, self.nblocks, self.nnz, self.packed_elems = order.value, nb.value, nnz.value, pe.value
        self.blk_off = np.ctypeslib.as_array(bo, (nb.value,)).copy()
        self.owner = np.ctypeslib.as_array(ow, (nb.value,)).copy()
        self.nz = np.ctypeslib.as_array(z, (nb.value,)).copy()
        n = _i64()
        pb, plo, phi, pow_ = _P(_i64)(), _P(_i32)(), _P(_i32)(), _P(_i32)()
        _check(_lib.tt_tensor_parts(self.h, ctypes.byref(n), ctypes.byref(pb), ctypes.byref(plo), ctypes.byref(phi),
                                    ctypes.byref(pow_)))
        se, so = _i64(), _P(_i64)()
        _check(_lib.tt_tensor_storage(self.h, ctypes.byref(se), ctypes.byref(so)))
        self.storage_elems = se.value
        self.storage_off = np.ctypeslib.as_array(so, (nb.value,)).copy()
        k = n.value
        self.parts = [tuple(int(x) for x in row) for row in zip(
            np.ctypeslib.as_array(pb, (k,)) if k else [], np.ctypeslib.as_array(plo, (k,)) if k else [],
            np.ctypeslib.as_array(phi, (k,)) if k else [], np.ctypeslib.as_array(pow_, (k,)) if k else [])]

    def view(self, dims: Sequence[TiledIndexSpace]) -> "Tensor":
        """Sliced view over sub-spaces of this tensor's dims (P152, P159; tt_tensor_view): no copy, the
        view reads and writes this tensor's storage."""
        v = Tensor(self.ctx, dims, _view_of=self)
        v.storage = self.storage
        return v

    @property
    def shape(self):
        return tuple(int(d.extent) for d in self.dims)

    @property
    def grid(self):
        return tuple(int(d.ntiles) for d in self.dims)

    def set_owner(self, owner):
        o = np.ascontiguousarray(owner, dtype=np.int32)
        _check(_lib.tt_tensor_set_owner(self.h, _ptr(o)))
        self._refresh()

    def set_parts(self, parts):
        """Row-range ownership: ``parts`` = [(block, lo, hi, owner)] (see tt_tensor_set_parts)."""
        a = np.asarray(parts, dtype=np.int64).reshape(-1, 4)
        blk = np.ascontiguousarray(a[:, 0])
        lo, hi, ow = (np.ascontiguousarray(a[:, i], dtype=np.int32) for i in (1, 2, 3))
        _check(_lib.tt_tensor_set_parts(self.h, len(a), _ptr(blk), _ptr(lo), _ptr(hi), _ptr(ow)))
        self._refresh()

    def set_compact(self, on: bool = True):
        """Compact storage: the buffer holds only this rank's parts (tt_tensor_set_compact)."""
        _check(_lib.tt_tensor_set_compact(self.h, 1 if on else 0))
        self._refresh()

    def bind(self, storage, capacity: Optional[int] = None):
        """Bind caller-owned device memory (a torch tensor, or an int pointer with ``capacity``)."""
        if capacity is None:
            capacity = int(storage.numel())
        _check(_lib.tt_tensor_bind(self.h, _vp(_devptr(storage)), int(capacity)))
        self.storage = storage

    def upload(self, host: np.ndarray):
        assert host.dtype == np.float64 and host.size >= self.storage_elems
        _check(_lib.tt_tensor_upload(self.ctx.h, self.h, _vp(host.ctypes.data)))

    def upload_ptr(self, host_ptr: int):
        _check(_lib.tt_tensor_upload(self.ctx.h, self.h, _vp(host_ptr)))

    def download(self, host: Optional[np.ndarray] = None) -> np.ndarray:
        if host is None:
            host = np.empty(self.storage_elems, dtype=np.float64)
        _check(_lib.tt_tensor_download(self.ctx.h, self.h, _vp(host.ctypes.data)))
        return host

    def download_ptr(self, host_ptr: int):
        _check(_lib.tt_tensor_download(self.ctx.h, self.h, _vp(host_ptr)))

    def close(self):
        """Destroys the handle now (a view: releases its parent's layout, see tt_tensor_view)."""
        if getattr(self, "h", None) is not None:
            _lib.tt_tensor_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def fill_synthetic(ctx: Context, T: Tensor, seed: int, tag: int, kind: int = KIND_UNIFORM):
    _check(_lib.tt_fill_synthetic(ctx.h, T.h, seed, tag, kind))


def set_(ctx: Context, C: Tensor, alpha: float):
    """P172 rule 5: C = alpha."""
    _check(_lib.tt_set(ctx.h, C.h, float(alpha)))


def add(ctx: Context, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str):
    """P173 rule 6: C(c_lbl) = beta*C + alpha*A(a_lbl)."""
    _check(_lib.tt_add(ctx.h, C.h, _b(c_lbl), float(beta), float(alpha), A.h, _b(a_lbl)))


def contract(ctx: Context, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str, B: Tensor,
             b_lbl: str):
    """P174 rule 7: C(c_lbl) = beta*C + alpha*A(a_lbl)*B(b_lbl)."""
    _check(_lib.tt_contract(ctx.h, C.h, _b(c_lbl), float(beta), float(alpha), A.h, _b(a_lbl), B.h, _b(b_lbl)))


def contract_cholesky(ctx: Context, C: Tensor, c_lbl: str, beta: float, alpha: float, X: Tensor, v_lbl: str,
                      B: Tensor, b_lbl: str, workspace, ws_elems: Optional[int] = None):
    """C = beta*C + alpha * V(v_lbl) * B(b_lbl), V(p,q,r,s) = sum_L X(p,r,L)X(q,s,L) - X(p,s,L)X(q,r,L)
    built batch by batch in ``workspace`` (Eq. cc12; tt_contract_cholesky)."""
    if ws_elems is None:
        ws_elems = int(workspace.numel())
    _check(_lib.tt_contract_cholesky(ctx.h, C.h, _b(c_lbl), float(beta), float(alpha), X.h, _b(v_lbl), B.h,
                                     _b(b_lbl), _vp(_devptr(workspace)), int(ws_elems)))


def contract_prefetch(ctx: Context, C: Tensor, c_lbl: str, beta: float, A: Tensor, a_lbl: str, B: Tensor,
                      b_lbl: str):
    """Issue the input gather of a later ``contract`` with the same arguments on the comm stream
    (tt_contract_prefetch): it overlaps the kernels issued in between."""
    _check(_lib.tt_contract_prefetch(ctx.h, C.h, _b(c_lbl), beta, A.h, _b(a_lbl), B.h, _b(b_lbl)))


def contract_host(ctx: Context, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str, B: Tensor,
                  b_lbl: str, hA=None, hB=None, hC=None, c_in: bool = False, c_out: bool = False):
    """tt_contract_host: the contraction from host buffers (pinned torch tensors or addresses; None = the
    operand is resident), pipelined inside the library (per chunk of C, see include/tt.h)."""
    flags = (HOST_C_IN if c_in else 0) | (HOST_C_OUT if c_out else 0)
    _check(_lib.tt_contract_host(ctx.h, C.h, _b(c_lbl), float(beta), float(alpha), A.h, _b(a_lbl), B.h, _b(b_lbl),
                                 _vp(_devptr(hA)) if hA is not None else None,
                                 _vp(_devptr(hB)) if hB is not None else None,
                                 _vp(_devptr(hC)) if hC is not None else None, flags))


def contract3(ctx: Context, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str, B: Tensor,
              b_lbl: str, D: Tensor, d_lbl: str, workspace=None, ws_elems: Optional[int] = None) -> dict:
    """Three-operand contraction through the cheapest intermediate (PAPER Eqs. cc9-cc11; tt_contract3).
    ``workspace=None`` only plans: returns the pairing, its costs and the workspace size."""
    info = Contract3Info()
    ws = _vp(_devptr(workspace)) if workspace is not None else None
    n = int(ws_elems if ws_elems is not None else (workspace.numel() if workspace is not None else 0))
    _check(_lib.tt_contract3(ctx.h, C.h, _b(c_lbl), beta, alpha, A.h, _b(a_lbl), B.h, _b(b_lbl), D.h, _b(d_lbl),
                             ws, n, ctypes.byref(info)))
    return info.as_dict()


def triples_energy(ctx: Context, T1: Tensor, T2: Tensor, Vooov: Tensor, Vvovv: Tensor, Voovv: Tensor,
                   eps_o=None, eps_v=None, workspace=None, ws_elems: Optional[int] = None):
    """(T) energy, PAPER Eq. cc14 (tt_triples_energy).  ``eps_o``/``eps_v`` device arrays (torch); with
    ``workspace=None`` only plans and returns (None, info)."""
    info = TriplesInfo()
    e = _dbl(0.0)
    ws = _vp(_devptr(workspace)) if workspace is not None else None
    n = int(ws_elems if ws_elems is not None else (workspace.numel() if workspace is not None else 0))
    _check(_lib.tt_triples_energy(ctx.h, T1.h, T2.h, Vooov.h, Vvovv.h, Voovv.h,
                                  _vp(_devptr(eps_o)) if eps_o is not None else None,
                                  _vp(_devptr(eps_v)) if eps_v is not None else None, ws, n, ctypes.byref(e),
                                  ctypes.byref(info)))
    return (e.value if workspace is not None else None), info.as_dict()


def contract_scalar(ctx: Context, alpha: float, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str) -> float:
    r = _dbl()
    _check(_lib.tt_contract_scalar(ctx.h, float(alpha), A.h, _b(a_lbl), B.h, _b(b_lbl), ctypes.byref(r)))
    return r.value


def task_list(ctx: Context, C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str,
              device: bool = False):
    """Canonical task list (R11): returns dict cblk, ptr, a_blk, b_blk, cost (numpy int64)."""
    nc, nt = _i64(), _i64()
    args = (ctx.h, C.h, _b(c_lbl), A.h, _b(a_lbl), B.h, _b(b_lbl), 1 if device else 0)
    _check(_lib.tt_task_list(*args, None, None, None, None, None, 0, ctypes.byref(nc), ctypes.byref(nt)))
    cb = np.empty(nc.value, np.int64)
    ptr = np.empty(nc.value + 1, np.int64)
    ab = np.empty(max(nt.value, 1), np.int64)
    bb = np.empty(max(nt.value, 1), np.int64)
    cost = np.empty(nc.value, np.int64)
    _check(_lib.tt_task_list(*args, _ptr(cb), _ptr(ptr), _ptr(ab), _ptr(bb), _ptr(cost), len(ab), ctypes.byref(nc),
                             ctypes.byref(nt)))
    return {"cblk": cb, "ptr": ptr, "a_blk": ab[:nt.value], "b_blk": bb[:nt.value], "cost": cost}


def partition_lpt(ctx: Context, C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str,
                  group_dims: Sequence[int] = ()) -> np.ndarray:
    """LPT owner partition (R24); ``group_dims`` = C dims whose tile coordinates define a unit."""
    own = np.empty(C.nblocks, np.int32)
    mask = sum(1 << d for d in group_dims)
    _check(_lib.tt_partition_lpt(ctx.h, C.h, _b(c_lbl), A.h, _b(a_lbl), B.h, _b(b_lbl), mask, _ptr(own)))
    return own


def partition_split(ctx: Context, C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str,
                    group_dims: Sequence[int] = ()):
    """Balanced partition with row splitting (tt_partition_split); updates C's ownership in place."""
    mask = sum(1 << d for d in group_dims)
    _check(_lib.tt_partition_split(ctx.h, C.h, _b(c_lbl), A.h, _b(a_lbl), B.h, _b(b_lbl), mask))
    C._refresh()


def partition_split_cost(ctx: Context, C: Tensor, cost, group_dims: Sequence[int] = ()):
    """tt_partition_split with caller-supplied costs (one per non-zero C block, block-id order)."""
    c = np.ascontiguousarray(cost, dtype=np.int64)
    if c.shape != (int((C.nz > 0).sum()),):
        raise ValueError("cost needs one entry per non-zero block of C")
    mask = sum(1 << d for d in group_dims)
    _check(_lib.tt_partition_split_cost(ctx.h, C.h, _ptr(c), mask))
    C._refresh()


def partition_split_cholesky(ctx: Context, C: Tensor, c_lbl: str, X: Tensor, v_lbl: str, B: Tensor, b_lbl: str,
                             group_dims: Sequence[int] = ()):
    """tt_partition_split on the executed cost of the implicit-operand ladder (tt_contract_cholesky)."""
    mask = sum(1 << d for d in group_dims)
    _check(_lib.tt_partition_split_cholesky(ctx.h, C.h, _b(c_lbl), X.h, _b(v_lbl), B.h, _b(b_lbl), mask))
    C._refresh()


def gather_plan(ctx: Context, C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str):
    """(recv, send) arrays of (operand, block, peer, e0, e1) rows for this rank."""
    nr, ns = _i64(), _i64()
    args = (ctx.h, C.h, _b(c_lbl), A.h, _b(a_lbl), B.h, _b(b_lbl))
    _check(_lib.tt_gather_plan(*args, None, ctypes.byref(nr), None, ctypes.byref(ns), 0))
    cap = max(nr.value, ns.value, 1)
    r = np.empty(5 * cap, np.int64)
    s = np.empty(5 * cap, np.int64)
    _check(_lib.tt_gather_plan(*args, _ptr(r), ctypes.byref(nr), _ptr(s), ctypes.byref(ns), cap))
    return r[:5 * nr.value].reshape(-1, 5), s[:5 * ns.value].reshape(-1, 5)


class Scheduler:
    """Scheduler (P178, P191-199, P215): queue operations, levelize by conflicts, execute level by
    level (concurrent streams inside a level).  Mirrors ``sch(op)(op)...execute()``."""

    def __init__(self, ctx: Context, nstreams: int = 4):
        h = _vp()
        _check(_lib.tt_sched_create(ctx.h, nstreams, ctypes.byref(h)))
        self.h, self.ctx = h, ctx
        self._results = []
        self._keep = []

    def close(self):
        if self.h:
            _check(_lib.tt_sched_destroy(self.h))
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def set_(self, C: Tensor, alpha: float):
        _check(_lib.tt_sched_set(self.h, C.h, float(alpha)))
        return self

    def add(self, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str):
        _check(_lib.tt_sched_add(self.h, C.h, _b(c_lbl), float(beta), float(alpha), A.h, _b(a_lbl)))
        return self

    def contract(self, C: Tensor, c_lbl: str, beta: float, alpha: float, A: Tensor, a_lbl: str, B: Tensor,
                 b_lbl: str):
        _check(_lib.tt_sched_contract(self.h, C.h, _b(c_lbl), float(beta), float(alpha), A.h, _b(a_lbl), B.h,
                                      _b(b_lbl)))
        return self

    def contract_cholesky(self, C: Tensor, c_lbl: str, beta: float, alpha: float, X: Tensor, v_lbl: str,
                          B: Tensor, b_lbl: str, workspace, ws_elems: Optional[int] = None):
        if ws_elems is None:
            ws_elems = int(workspace.numel())
        self._keep.append(workspace)
        _check(_lib.tt_sched_contract_cholesky(self.h, C.h, _b(c_lbl), float(beta), float(alpha), X.h, _b(v_lbl),
                                               B.h, _b(b_lbl), _vp(_devptr(workspace)), int(ws_elems)))
        return self

    def scalar(self, alpha: float, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str):
        """Queues an order-0 contraction; its value is in ``results[i]`` after execute()."""
        r = _dbl()
        self._results.append(r)
        _check(_lib.tt_sched_scalar(self.h, float(alpha), A.h, _b(a_lbl), B.h, _b(b_lbl), ctypes.byref(r)))
        return self

    def levels(self):
        n, L = _i64(), _i32()
        _check(_lib.tt_sched_levels(self.h, None, ctypes.byref(n), ctypes.byref(L)))
        lv = np.empty(max(n.value, 1), np.int32)
        _check(_lib.tt_sched_levels(self.h, _ptr(lv), ctypes.byref(n), ctypes.byref(L)))
        return lv[:n.value].tolist(), L.value

    def execute(self):
        _check(_lib.tt_sched_execute(self.h))
        out = [r.value for r in self._results]
        self._results = []
        self._keep = []
        return out

    def capture(self):
        """Record the queue into a CUDA graph (plans are built first); the queue is kept."""
        _check(_lib.tt_sched_capture(self.h))
        return self

    def replay(self):
        """Launch the captured graph; returns the scalar results (in queue order)."""
        _check(_lib.tt_sched_replay(self.h))
        return [r.value for r in self._results]

    def stats(self):
        q, lv = _i64(), _i64()
        _check(_lib.tt_sched_stats(self.h, ctypes.byref(q), ctypes.byref(lv)))
        return {"queued": q.value, "levels_executed": lv.value}
