"""Thin Python binding of liblco.so (include/lco.h) — argument marshalling only.

Every step of the permutation runs in the library's CUDA kernels; this module only
turns torch tensors into pointers, allocates outputs and the workspace through
PyTorch's caching allocator, and maps status codes to exceptions.  There is no CPU
fallback: if liblco.so is missing or the tensors are not on a CUDA device, calls fail.

Names follow the C ABI: ``permute`` (lco_permute), ``sort`` (lco_sort),
``permute_host`` (lco_permute_host), ``partition`` (lco_partition),
``key_histogram`` (lco_key_histogram), ``Plan.info`` (lco_plan_query).
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblco.so")

FLAG_VALIDATE = 1
FLAG_HIERARCHICAL = 2
MAX_ORDER = 16
PATHS = {0: "copy", 1: "lsd", 2: "leaf", 3: "msd", 4: "tile", 5: "seg", 6: "hier", 7: "block",
         8: "single"}

_STATUS = {
    0: "LCO_OK", 1: "LCO_ERR_NULL", 2: "LCO_ERR_ORDER", 3: "LCO_ERR_DIM", 4: "LCO_ERR_PERM",
    5: "LCO_ERR_OVERFLOW", 6: "LCO_ERR_CAPACITY", 7: "LCO_ERR_WORKSPACE", 8: "LCO_ERR_ALIAS",
    9: "LCO_ERR_UNSORTED", 10: "LCO_ERR_KEY_RANGE", 11: "LCO_ERR_CUDA", 12: "LCO_ERR_ARG",
}


class LcoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class LcoValueError(LcoError, ValueError):
    pass


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int),
        ("rearrangement", ctypes.c_int32 * MAX_ORDER),
        ("norm_order", ctypes.c_int),
        ("norm_dims", ctypes.c_uint64 * MAX_ORDER),
        ("norm_perm", ctypes.c_int32 * MAX_ORDER),
        ("prefix_len", ctypes.c_int),
        ("suffix_start", ctypes.c_int),
        ("segment_divisor", ctypes.c_uint64),
        ("trailing", ctypes.c_uint64),
        ("middle_size", ctypes.c_uint64),
        ("num_segments", ctypes.c_uint64),
        ("sort_bits", ctypes.c_int),
        ("passes", ctypes.c_int),
        ("digit_bits", ctypes.c_int * 8),
        ("radix_bits", ctypes.c_int),
        ("path", ctypes.c_int),
        ("launches", ctypes.c_int),
        ("tile", ctypes.c_int),
        ("msd_levels", ctypes.c_int),
        ("leaf_bits", ctypes.c_int),
        ("leaf_kind", ctypes.c_int),
        ("model_bytes", ctypes.c_double),
        ("stages", ctypes.c_int),
        ("stage_path", ctypes.c_int * 8),
        ("stage_sort_bits", ctypes.c_int * 8),
        ("flat_model_bytes", ctypes.c_double),
        ("block_grid", ctypes.c_uint64 * 5),
    ]


_lib = None
_lib_lock = threading.Lock()

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_SIGS = {
    "lco_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.POINTER(_U64),
                                  ctypes.POINTER(ctypes.c_int32), _U64, ctypes.c_uint32]),
    "lco_destroy": (ctypes.c_int, [_P]),
    "lco_workspace_size": (ctypes.c_int, [_P, _U64, ctypes.POINTER(ctypes.c_size_t)]),
    "lco_host_workspace_size": (ctypes.c_int, [_P, _U64, ctypes.POINTER(ctypes.c_size_t)]),
    "lco_permute": (ctypes.c_int, [_P, _U64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "lco_sort": (ctypes.c_int, [_P, _U64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "lco_permute_host": (ctypes.c_int, [_P, _U64, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "lco_partition": (ctypes.c_int, [_P, _U64, _P, _P, ctypes.c_uint32, ctypes.c_int, _P, _P, _P,
                                     _P, _P, _P, ctypes.c_size_t, _P]),
    "lco_key_histogram": (ctypes.c_int, [_P, _U64, _P, ctypes.c_int, _P, _P]),
    "lco_partition_counts": (ctypes.c_int, [_P, _U64, _P, ctypes.c_int, _P, _P, _P,
                                            ctypes.c_size_t, _P]),
    "lco_partition_direct": (ctypes.c_int, [_P, _U64, _P, _P, ctypes.c_uint32, ctypes.c_int, _P,
                                            _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "lco_add_workspace_size": (ctypes.c_int, [_P, _U64, _U64, ctypes.POINTER(ctypes.c_size_t)]),
    "lco_compress_workspace_size": (ctypes.c_int, [_U64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "lco_compress": (ctypes.c_int, [_U64, _P, _U64, _U64, ctypes.c_int, _P, _P, _P, _P, _P,
                                    ctypes.c_size_t, _P]),
    "lco_sparsity_class": (ctypes.c_int, [_U64, _U64, _U64, ctypes.c_double]),
    "lco_mdt_choice": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "lco_mdt_name": (ctypes.c_char_p, [ctypes.c_int]),
    "lco_add": (ctypes.c_int, [_P, _U64, _P, _P, _U64, _P, _P, ctypes.c_double, _P, _P, _P, _P,
                               ctypes.c_size_t, _P]),
    "lco_plan_query": (ctypes.c_int, [_P, _U64, ctypes.c_int, ctypes.POINTER(PlanInfo)]),
    "lco_plan_stage": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_U64),
                                      ctypes.POINTER(ctypes.c_int32)]),
    "lco_fastdiv_host": (ctypes.c_int, [_U64, _U64, _P, _P]),
    "lco_profile_enable": (ctypes.c_int, [_P, ctypes.c_int]),
    "lco_profile_read": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P,
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.c_char_p, ctypes.c_size_t]),
    "lco_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "lco_last_error": (ctypes.c_char_p, []),
    "lco_version": (ctypes.c_char_p, []),
}


def lib():
    """Load liblco.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing; build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'`")
                from . import _build
                if not _build.up_to_date():
                    # the .so does not match the sources (content hash): never run a stale
                    # binary; rebuild in place (nvcc is part of the image)
                    import sys
                    print(f"[lco] {LIB_PATH} is stale for the current sources; rebuilding",
                          file=sys.stderr, flush=True)
                    _build.build(force=True)
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    f = getattr(L, name)
                    f.restype = res
                    f.argtypes = args
                _lib = L
    return _lib


def _check(status):
    if status != 0:
        msg = lib().lco_last_error().decode(errors="replace")
        cls = LcoValueError if status in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12) else LcoError
        raise cls(status, msg)


def version() -> str:
    return lib().lco_version().decode()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _workspace(nbytes, device):
    if nbytes == 0:
        return None, 0
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 256
    return buf, off


def _on(stream, device):
    """Allocate on and launch into `stream` (default: the current stream): workspace and
    outputs this module allocates then belong to that stream in the caching allocator,
    so their memory is never reused while the call's kernels run, and zero-fills are
    ordered before them."""
    return _Ctx(stream, device)


class _Ctx:
    def __init__(self, stream, device):
        cuda = torch.device(device).type == "cuda"  # else the call itself raises
        self.d = torch.cuda.device(device) if cuda else None
        self.s = torch.cuda.stream(stream) if (stream is not None and cuda) else None

    def __enter__(self):
        if self.d is not None:
            self.d.__enter__()
        if self.s is not None:
            self.s.__enter__()
        return self

    def __exit__(self, *exc):
        if self.s is not None:
            self.s.__exit__(*exc)
        if self.d is not None:
            self.d.__exit__(*exc)
        return False


class Plan:
    """An lco_handle: the host plan for (dims, perm).  Immutable; reusable."""

    def __init__(self, dims, perm=None, max_nnz=(1 << 32) - 1, validate=False, hierarchical=False):
        self.dims = tuple(int(d) for d in dims)
        order = len(self.dims)
        self.perm = tuple(range(order)) if perm is None else tuple(int(p) for p in perm)
        d = (ctypes.c_uint64 * max(order, 1))(*self.dims)
        p = (ctypes.c_int32 * max(order, 1))(*self.perm)
        h = ctypes.c_void_p()
        _check(lib().lco_create(ctypes.byref(h), order, d, p, int(max_nnz),
                                (FLAG_VALIDATE if validate else 0)
                                | (FLAG_HIERARCHICAL if hierarchical else 0)))
        self._h = h
        self.max_nnz = int(max_nnz)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.lco_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def new_dims(self):
        return tuple(self.dims[p] for p in self.perm)

    def workspace_size(self, nnz: int) -> int:
        n = ctypes.c_size_t()
        _check(lib().lco_workspace_size(self._h, int(nnz), ctypes.byref(n)))
        return n.value

    def host_workspace_size(self, nnz: int) -> int:
        n = ctypes.c_size_t()
        _check(lib().lco_host_workspace_size(self._h, int(nnz), ctypes.byref(n)))
        return n.value

    def stages(self) -> list:
        """The hierarchical plan (lco_plan_stage): [(dims, perm)] per stage, in the
        normalized key space; composing them gives this plan's permutation."""
        out, j, ns = [], 0, 1
        while j < ns:
            n_st, order = ctypes.c_int(), ctypes.c_int()
            dims = (_U64 * 16)()
            perm = (ctypes.c_int32 * 16)()
            _check(lib().lco_plan_stage(self._h, j, ctypes.byref(n_st), ctypes.byref(order), dims, perm))
            ns = n_st.value
            out.append((tuple(int(x) for x in dims[:order.value]), tuple(perm[:order.value])))
            j += 1
        return out

    def info(self, nnz: int, sort: bool = False) -> dict:
        pi = PlanInfo()
        _check(lib().lco_plan_query(self._h, int(nnz), 1 if sort else 0, ctypes.byref(pi)))
        n = pi.norm_order
        return {
            "order": pi.order,
            "rearrangement": list(pi.rearrangement[:pi.order]),
            "norm_dims": [int(x) for x in pi.norm_dims[:n]],
            "norm_perm": list(pi.norm_perm[:n]),
            "prefix_len": pi.prefix_len,
            "suffix_start": pi.suffix_start,
            "segment_divisor": int(pi.segment_divisor),
            "trailing": int(pi.trailing),
            "middle_size": int(pi.middle_size),
            "num_segments": int(pi.num_segments),
            "sort_bits": pi.sort_bits,
            "passes": pi.passes,
            "digit_bits": list(pi.digit_bits[:pi.passes]),
            "radix_bits": pi.radix_bits,
            "path": PATHS.get(pi.path, pi.path),
            "launches": pi.launches,
            "tile": pi.tile,
            "msd_levels": pi.msd_levels,
            "leaf_bits": pi.leaf_bits,
            "leaf_kind": {0: None, 1: "warp", 2: "cta"}.get(pi.leaf_kind, pi.leaf_kind),
            "model_bytes": pi.model_bytes,
            "stages": pi.stages,
            "stage_paths": [PATHS.get(x, x) for x in pi.stage_path[:pi.stages]] if pi.stages > 1 else [],
            "stage_sort_bits": list(pi.stage_sort_bits[:pi.stages]) if pi.stages > 1 else [],
            "flat_model_bytes": pi.flat_model_bytes,
            "block_grid": list(pi.block_grid) if pi.path == 7 else None,
        }

    # ---------------------------------------------------------------- device calls
    def _run(self, fn, keys, vals, idx, return_perm, stream, out, workspace):
        if not keys.is_cuda:
            raise ValueError("keys must be a CUDA tensor (no CPU fallback)")
        if keys.dtype not in (torch.int64, torch.uint64) or keys.dim() != 1:
            raise ValueError("keys must be a 1-D int64/uint64 tensor")
        keys = keys.contiguous()
        dev = keys.device
        n = keys.numel()
        if vals is not None:
            if vals.dtype != torch.float64 or vals.numel() != n or vals.device != dev:
                raise ValueError("vals must be float64, same length and device as keys")
            vals = vals.contiguous()
        if idx is not None:
            if idx.dtype not in (torch.int32, torch.uint32) or idx.numel() != n or idx.device != dev:
                raise ValueError("idx must be int32/uint32, same length and device as keys")
            idx = idx.contiguous()
        if out is None:
            ko = torch.empty_like(keys)
            vo = None if vals is None else torch.empty_like(vals)
            po = torch.empty(n, dtype=torch.int32, device=dev) if return_perm else None
        else:
            ko, vo, po = out
        if workspace is None:
            ws, off = _workspace(self.workspace_size(n), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        with torch.cuda.device(dev):
            _check(fn(self._h, n, _ptr(keys), _ptr(vals), _ptr(idx), _ptr(ko), _ptr(vo), _ptr(po),
                      wptr, wlen, _stream_ptr(stream, dev)))
        return ko, vo, po

    def add_workspace_size(self, nnz_a: int, nnz_b: int) -> int:
        b = ctypes.c_size_t()
        _check(lib().lco_add_workspace_size(self._h, int(nnz_a), int(nnz_b), ctypes.byref(b)))
        return b.value

    def add(self, keys_a, vals_a, keys_b, vals_b, sign=1.0, stream=None, out=None,
            workspace=None, trim=True):
        """Index-matched addition (lco_add): A + sign * permute(B, match) where this plan
        holds B's dims and the match.  Returns (keys_c, vals_c, nnz_c); with trim=True the
        outputs are cut to nnz_c (one device->host read of the count)."""
        with _on(stream, keys_a.device):
            return self._add_impl(keys_a=keys_a, vals_a=vals_a, keys_b=keys_b, vals_b=vals_b,
                                  sign=sign, stream=stream, out=out, workspace=workspace, trim=trim)

    def _add_impl(self, keys_a, vals_a, keys_b, vals_b, sign=1.0, stream=None, out=None,
            workspace=None, trim=True):
        for t in (keys_a, vals_a, keys_b, vals_b):
            if not t.is_cuda:
                raise ValueError("operands must be CUDA tensors (no CPU fallback)")
        dev = keys_a.device
        na, nb = keys_a.numel(), keys_b.numel()
        if vals_a.numel() != na or vals_b.numel() != nb:
            raise ValueError("keys and values of an operand must have the same length")
        if vals_a.dtype != torch.float64 or vals_b.dtype != torch.float64:
            raise ValueError("values must be float64")
        keys_a, vals_a = keys_a.contiguous(), vals_a.contiguous()
        keys_b, vals_b = keys_b.contiguous(), vals_b.contiguous()
        if out is None:
            kc = torch.empty(na + nb, dtype=keys_a.dtype, device=dev)
            vc = torch.empty(na + nb, dtype=torch.float64, device=dev)
            nc = torch.zeros(1, dtype=torch.int64, device=dev)
        else:
            kc, vc, nc = out
        if workspace is None:
            ws, off = _workspace(self.add_workspace_size(na, nb), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        with torch.cuda.device(dev):
            _check(lib().lco_add(self._h, na, _ptr(keys_a), _ptr(vals_a), nb, _ptr(keys_b),
                                 _ptr(vals_b), float(sign), _ptr(kc), _ptr(vc), _ptr(nc), wptr,
                                 wlen, _stream_ptr(stream, dev)))
        if trim:
            m = int(nc.item())
            return kc[:m], vc[:m], m
        return kc, vc, nc

    def permute(self, keys, vals=None, idx=None, return_perm=True, stream=None, out=None,
                workspace=None):
        with _on(stream, keys.device):
            return self._run(lib().lco_permute, keys, vals, idx, return_perm, stream, out,
                             workspace)

    def sort(self, keys, vals=None, idx=None, return_perm=True, stream=None, out=None,
             workspace=None):
        with _on(stream, keys.device):
            return self._run(lib().lco_sort, keys, vals, idx, return_perm, stream, out, workspace)

    def permute_host(self, keys, vals=None, return_perm=True, device=None, stream=None,
                     out=None, workspace=None):
        """Host (ideally pinned) tensors in and out; copies run inside the call."""
        with _on(stream, torch.device(device or 'cuda')):
            return self._permute_host_impl(keys=keys, vals=vals, return_perm=return_perm,
                                           device=device, stream=stream, out=out,
                                           workspace=workspace)

    def _permute_host_impl(self, keys, vals=None, return_perm=True, device=None, stream=None,
                     out=None, workspace=None):
        if keys.is_cuda:
            raise ValueError("permute_host takes host tensors")
        dev = torch.device(device or "cuda")
        n = keys.numel()
        if out is None:
            pin = keys.is_pinned()
            ko = torch.empty(n, dtype=keys.dtype, pin_memory=pin)
            vo = None if vals is None else torch.empty(n, dtype=torch.float64, pin_memory=pin)
            po = torch.empty(n, dtype=torch.int32, pin_memory=pin) if return_perm else None
        else:
            ko, vo, po = out
        if workspace is None:
            ws, off = _workspace(self.host_workspace_size(n), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        with torch.cuda.device(dev):
            _check(lib().lco_permute_host(self._h, n, _ptr(keys), _ptr(vals), _ptr(ko), _ptr(vo),
                                          _ptr(po), wptr, wlen, _stream_ptr(stream, dev)))
        return ko, vo, po

    def partition(self, keys, vals, idx_base, splitters, stream=None, workspace=None):
        """Stable multisplit by new-key range: returns (send_keys, send_vals, send_idx,
        send_counts) on the device; send_keys are OLD keys."""
        with _on(stream, keys.device):
            return self._partition_impl(keys=keys, vals=vals, idx_base=idx_base,
                                        splitters=splitters, stream=stream, workspace=workspace)

    def _partition_impl(self, keys, vals, idx_base, splitters, stream=None, workspace=None):
        dev = keys.device
        n = keys.numel()
        world = 1 if splitters is None else splitters.numel() + 1
        sk = torch.empty_like(keys)
        sv = None if vals is None else torch.empty_like(vals)
        si = torch.empty(n, dtype=torch.int32, device=dev)
        cnt = torch.zeros(world, dtype=torch.int64, device=dev)
        if workspace is None:
            ws, off = _workspace(self.workspace_size(n), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        sp = None if splitters is None else splitters.contiguous()
        with torch.cuda.device(dev):
            _check(lib().lco_partition(self._h, n, _ptr(keys), _ptr(vals), int(idx_base), world,
                                       _ptr(sp), _ptr(sk), _ptr(sv), _ptr(si), _ptr(cnt), wptr,
                                       wlen, _stream_ptr(stream, dev)))
        return sk, sv, si, cnt

    def partition_counts(self, keys, splitters, stream=None, workspace=None):
        """Records per destination rank of the multisplit (device int64[world])."""
        with _on(stream, keys.device):
            return self._partition_counts_impl(keys=keys, splitters=splitters, stream=stream,
                                               workspace=workspace)

    def _partition_counts_impl(self, keys, splitters, stream=None, workspace=None):
        dev = keys.device
        n = keys.numel()
        world = 1 if splitters is None else splitters.numel() + 1
        cnt = torch.zeros(world, dtype=torch.int64, device=dev)
        if workspace is None:
            ws, off = _workspace(self.workspace_size(n), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        sp = None if splitters is None else splitters.contiguous()
        with torch.cuda.device(dev):
            _check(lib().lco_partition_counts(self._h, n, _ptr(keys), world, _ptr(sp), _ptr(cnt),
                                              wptr, wlen, _stream_ptr(stream, dev)))
        return cnt

    def partition_direct(self, keys, vals, idx_base, splitters, recv_keys, recv_vals, recv_idx,
                         recv_offsets, stream=None, workspace=None):
        """The partition with the exchange fused in: records go straight into the
        receivers' buffers (lists of device tensors, peer-mapped on a multi-GPU box) at
        recv_offsets[d] + index.  Returns the device send counts."""
        with _on(stream, keys.device):
            return self._partition_direct_impl(keys=keys, vals=vals, idx_base=idx_base,
                                               splitters=splitters, recv_keys=recv_keys,
                                               recv_vals=recv_vals, recv_idx=recv_idx,
                                               recv_offsets=recv_offsets, stream=stream,
                                               workspace=workspace)

    def _partition_direct_impl(self, keys, vals, idx_base, splitters, recv_keys, recv_vals, recv_idx,
                         recv_offsets, stream=None, workspace=None):
        dev = keys.device
        n = keys.numel()
        world = 1 if splitters is None else splitters.numel() + 1
        cnt = torch.zeros(world, dtype=torch.int64, device=dev)
        if workspace is None:
            ws, off = _workspace(self.workspace_size(n), dev)
        else:
            ws, off = workspace, (-workspace.data_ptr()) % 256
        wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
        wlen = 0 if ws is None else ws.numel() - off
        sp = None if splitters is None else splitters.contiguous()
        arr = ctypes.c_void_p * world
        rk = arr(*[t.data_ptr() for t in recv_keys])
        rv = None if vals is None else arr(*[t.data_ptr() for t in recv_vals])
        ri = arr(*[t.data_ptr() for t in recv_idx])
        ro = (ctypes.c_uint64 * world)(*[int(x) for x in recv_offsets])
        with torch.cuda.device(dev):
            _check(lib().lco_partition_direct(
                self._h, n, _ptr(keys), _ptr(vals), int(idx_base), world, _ptr(sp),
                ctypes.cast(rk, _P), None if rv is None else ctypes.cast(rv, _P),
                ctypes.cast(ri, _P), ctypes.cast(ro, _P), _ptr(cnt), wptr, wlen,
                _stream_ptr(stream, dev)))
        return cnt

    def key_histogram(self, keys, bits, counts=None, stream=None):
        dev = keys.device
        with _on(stream, dev):
            if counts is None:
                counts = torch.zeros(1 << bits, dtype=torch.int64, device=dev)
            _check(lib().lco_key_histogram(self._h, keys.numel(), _ptr(keys), int(bits),
                                           _ptr(counts), _stream_ptr(stream, dev)))
        return counts

    def graph(self, keys, vals=None, idx=None, out=None, workspace=None, sort=False):
        """Capture one lco_permute (or lco_sort) call on fixed device buffers into a CUDA
        graph and return it: ``g.replay()`` re-runs the whole call -- every kernel the
        library launches for it, on the same inputs, outputs and workspace -- as one graph
        launch, which removes the per-kernel launch latency and host overhead that bound
        small tensors (SURVEY.md §7 "launch-latency-bound" configs).  The buffers must stay
        alive and in place while the graph is used."""
        fn = self.sort if sort else self.permute
        n = keys.numel()
        dev = keys.device
        if out is None:
            out = (torch.empty_like(keys), None if vals is None else torch.empty_like(vals),
                   torch.empty(n, dtype=torch.int32, device=dev))
        if workspace is None:
            workspace = torch.empty(self.workspace_size(n) + 256, dtype=torch.uint8, device=dev)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up: kernel attributes set before capture
            fn(keys, vals, idx, out=out, workspace=workspace)
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(keys, vals, idx, out=out, workspace=workspace)
        g.out = out
        g.workspace = workspace
        return g

    # ---------------------------------------------------------------- measurement hook
    def profile_enable(self, calls: int):
        _check(lib().lco_profile_enable(self._h, int(calls)))

    def profile_read(self, max_calls=64, max_stages=49):
        ms = (ctypes.c_float * (max_calls * max_stages))()
        nc, ns = ctypes.c_int(), ctypes.c_int()
        names = ctypes.create_string_buffer(4096)
        _check(lib().lco_profile_read(self._h, max_calls, max_stages, ctypes.cast(ms, _P),
                                      ctypes.byref(nc), ctypes.byref(ns), names, 4096))
        stage_names = names.value.decode().split(";") if names.value else []
        rows = [[ms[c * max_stages + s] for s in range(ns.value)] for c in range(nc.value)]
        return stage_names, rows


_plan_cache: dict = {}


def plan(dims, perm=None, max_nnz=(1 << 32) - 1, validate=False, hierarchical=False) -> Plan:
    # the library reads its LCO_* schedule overrides once per handle (lco_create): a
    # cached handle is only reused under the same overrides
    env = tuple(sorted((k, v) for k, v in os.environ.items() if k.startswith("LCO_")))
    key = (tuple(int(d) for d in dims), None if perm is None else tuple(int(p) for p in perm),
           int(max_nnz), bool(validate), bool(hierarchical), env)
    p = _plan_cache.get(key)
    if p is None:
        p = _plan_cache[key] = Plan(dims, perm, max_nnz, validate, hierarchical)
    return p


def permute(keys, vals, dims, perm, idx=None, return_perm=True, validate=False, stream=None,
            hierarchical=False):
    """Permute a sorted LCO tensor: returns (keys_out, vals_out, perm_out)."""
    return plan(dims, perm, validate=validate, hierarchical=hierarchical).permute(
        keys, vals, idx, return_perm, stream)


def add(keys_a, vals_a, keys_b, vals_b, dims_b, match, sign=1.0, stream=None):
    """Index-matched addition A + sign * permute(B, match): B has dims
    dims_b and is sorted in its own order; A is sorted in the matched order.  Returns the
    trimmed (keys_c, vals_c, nnz_c)."""
    return plan(dims_b, match).add(keys_a, vals_a, keys_b, vals_b, sign, stream)


def sort(keys, vals, dims, perm=None, idx=None, return_perm=True, validate=False, stream=None):
    """Sort an LCO tensor in any order into the order given by perm (stable)."""
    return plan(dims, perm, validate=validate).sort(keys, vals, idx, return_perm, stream)


def fastdiv_host(d: int, xs) -> list:
    """Host reference of the device fast divisor (test hook)."""
    n = len(xs)
    xa = (ctypes.c_uint64 * max(n, 1))(*[int(x) for x in xs])
    qa = (ctypes.c_uint64 * max(n, 1))()
    _check(lib().lco_fastdiv_host(int(d), n, ctypes.cast(xa, _P), ctypes.cast(qa, _P)))
    return [int(qa[i]) for i in range(n)]


# ------------------------------------------------------------ matrix datatypes (§5.2)
SPARSITY = ("sparse", "row-sparse", "column-sparse", "index-sparse")


def flatten(keys, vals, dims, rows, cols, major="row", stream=None):
    """Flatten (matricize) a sorted LCO tensor (§5.2 step 1): `rows` / `cols`
    are the modes mapped to the matrix rows / columns (disjoint, covering all modes, in
    the order wanted).  The permutation into (rows, cols) (row-major) or (cols, rows)
    (column-major) order runs on the GPU (lco_permute; the identity is a copy); the LIV
    of the result is row * n + col, resp. col * m + row.  Returns (keys, vals, m, n)."""
    rows, cols = tuple(int(x) for x in rows), tuple(int(x) for x in cols)
    if sorted(rows + cols) != list(range(len(dims))):
        raise ValueError("rows and cols must partition the modes")
    m = math.prod(int(dims[r]) for r in rows)
    n = math.prod(int(dims[c]) for c in cols)
    perm = rows + cols if major == "row" else cols + rows
    ko, vo, _ = plan(dims, perm).permute(keys, vals, return_perm=False, stream=stream)
    return ko, vo, m, n


def compress(keys, n_major, n_minor, doubly=False, stream=None):
    """Compress a major-first LCO matrix (lco_compress): CSR/CSC (doubly=False) returns
    {"ptr": [n_major+1], "minor": [nnz]}; DCSR/DCSC returns {"ids", "ptr", "minor", "nz"}
    with ids / ptr trimmed to the nz non-empty majors (one count read back)."""
    if not keys.is_cuda:
        raise ValueError("keys must be a CUDA tensor (no CPU fallback)")
    keys = keys.contiguous()
    dev, nnz = keys.device, keys.numel()
    minor = torch.empty(nnz, dtype=torch.int64, device=dev)
    b = ctypes.c_size_t()
    _check(lib().lco_compress_workspace_size(nnz, 1 if doubly else 0, ctypes.byref(b)))
    ws, off = _workspace(b.value, dev) if b.value else (None, 0)
    wptr = None if ws is None else ctypes.c_void_p(ws.data_ptr() + off)
    wlen = 0 if ws is None else ws.numel() - off
    if doubly:
        ids = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        ptr = torch.empty(nnz + 1, dtype=torch.int64, device=dev)
        nz = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        ids = nz = None
        ptr = torch.empty(int(n_major) + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _check(lib().lco_compress(nnz, _ptr(keys), int(n_major), int(n_minor), 1 if doubly else 0,
                                  _ptr(ptr), _ptr(ids), _ptr(minor), _ptr(nz), wptr, wlen,
                                  _stream_ptr(stream, dev)))
    if not doubly:
        return {"ptr": ptr, "minor": minor}
    k = int(nz.item())
    return {"ids": ids[:k], "ptr": ptr[:k + 1], "minor": minor, "nz": k}


def sparsity_class(m, n, nnz, threshold=3.0) -> str:
    """Hyper-sparsity of an m x n matrix (LibNT's ratio test)."""
    return SPARSITY[lib().lco_sparsity_class(int(m), int(n), int(nnz), float(threshold))]


def mdt_choice(class_a: str, class_b: str) -> str:
    """The poly-algorithm's MDT / algorithm for A (class_a) times B (class_b), PAPER.md
    Table "Multiplication possibilities"."""
    c = lib().lco_mdt_choice(SPARSITY.index(class_a), SPARSITY.index(class_b))
    return lib().lco_mdt_name(c).decode()
