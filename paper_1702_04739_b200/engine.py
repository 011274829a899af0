"""Device backend: torch CUDA tensors as buffers, libisoclust_b200.so as compute.

PyTorch is plumbing only (allocation, the current stream, torch.distributed
for the per-round key all-reduce); every arithmetic step on the hot path is
one of our sm_100a kernels behind the C ABI.  There is no CPU path: the
backend raises when CUDA or the library is unavailable.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check
from .types import Extrema

NO_KEY = 0x7FFFFFFFFFFFFFFF


def _torch():
    import torch

    return torch


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class Comm:
    """Row sharding over torch.distributed ranks (one process per GPU)."""

    def __init__(self):
        torch = _torch()
        dist = torch.distributed
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank()
            self.world = dist.get_world_size()
        else:
            self.rank, self.world = 0, 1
        self.dist = dist

    def rows(self, n: int, rank: Optional[int] = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        return n * r // self.world, n * (r + 1) // self.world

    def allreduce_min_(self, t) -> None:
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)

    def allreduce_sum_(self, t) -> None:
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)

    def allgather_rows(self, local, n: int):
        """Concatenate per-rank row blocks (rank order) into one n-row tensor."""
        if self.world == 1:
            return local
        torch = _torch()
        sizes = [self.rows(n, r) for r in range(self.world)]
        mx = max(h - l for l, h in sizes)
        pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad)
        return torch.cat([p[: h - l] for p, (l, h) in zip(parts, sizes)])

    def alltoall_rows(self, t, n: int):
        """Rows of `t` (n rows, any trailing shape) sent to their owners; the
        result holds, rank-major, every rank's rows of this rank's shard:
        shape (world, hi - lo, ...).  Ranks exchange equal padded blocks."""
        torch = _torch()
        lo, hi = self.rows(n)
        if self.world == 1:
            return t[lo:hi].unsqueeze(0)
        sizes = [self.rows(n, r) for r in range(self.world)]
        mx = max(h - l for l, h in sizes)
        send = torch.zeros((self.world, mx) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        for r, (l, h) in enumerate(sizes):
            send[r, : h - l] = t[l:h]
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send)
        return recv[:, : hi - lo].contiguous()

    def alltoall_chunks(self, t):
        """t: (world, ...) contiguous, chunk r for rank r; returns (world, ...)
        with chunk s = what rank s sent here."""
        if self.world == 1:
            return t
        out = _torch().empty_like(t)
        self.dist.all_to_all_single(out, t)
        return out

    def alltoall_var(self, t, send_counts, recv_counts):
        """1-d `t` = this rank's messages to ranks 0..world-1 (send_counts
        elements each, in rank order); returns the concatenation of the
        messages every rank sent here (recv_counts elements each)."""
        if self.world == 1:
            return t
        out = _torch().empty((max(1, sum(recv_counts)),), dtype=t.dtype, device=t.device)
        self.dist.all_to_all_single(out[: sum(recv_counts)], t[: sum(send_counts)],
                                    output_split_sizes=list(recv_counts), input_split_sizes=list(send_counts))
        return out

    def allgather_stack(self, stack):
        """Fold stacks of every rank, in rank (= row) order."""
        if self.world == 1:
            return stack.view(1, -1)
        torch = _torch()
        parts = [torch.empty_like(stack) for _ in range(self.world)]
        self.dist.all_gather(parts, stack)
        return torch.stack(parts)


class CudaBackend:
    """Stage calls into libisoclust_b200.so on torch's current CUDA stream."""

    name = "cuda"

    def __init__(self, device: Optional[int] = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1702_04739_b200 needs a CUDA device (B200); no CPU fallback")
        self.lib = _lib.load()
        if device is not None:
            torch.cuda.set_device(device)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.torch = torch

    # -- plumbing -----------------------------------------------------
    @property
    def stream(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    _STAGE_THREADS = 8
    _STAGE_MIN = 64 << 20

    def to_device(self, x: np.ndarray):
        """Host array -> HBM through a page-locked staging buffer (torch's
        caching host allocator); large arrays are staged by several threads
        (numpy copies release the GIL), then one async H2D copy."""
        torch = self.torch
        a = np.ascontiguousarray(x)
        t = torch.from_numpy(a)
        if t.is_pinned():
            return t.to(self.device, non_blocking=True)
        if a.nbytes < self._STAGE_MIN:
            return t.pin_memory().to(self.device, non_blocking=True)
        staged = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        dst = staged.numpy().reshape(-1)
        src = a.reshape(-1)
        k = self._STAGE_THREADS
        step = -(-src.shape[0] // k)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(k) as ex:
            list(ex.map(lambda i: np.copyto(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]),
                        range(k)))
        return staged.to(self.device, non_blocking=True)

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.device)

    _NP2TORCH = {np.dtype(np.int64): "int64", np.dtype(np.float64): "float64", np.dtype(np.int8): "int8",
                 np.dtype(np.int32): "int32"}

    def pinned_empty(self, n: int, dtype) -> np.ndarray:
        """numpy view of a page-locked host buffer (the array keeps it alive)."""
        tdt = getattr(self.torch, self._NP2TORCH[np.dtype(dtype)])
        return self.torch.empty(n, dtype=tdt, pin_memory=True).numpy()

    # -- exact passes -------------------------------------------------
    def sigma_partial(self, X, n: int, d: int, lo: int, hi: int, alpha: float, want_nn: bool = True):
        torch = self.torch
        rows = hi - lo
        stack = self.empty((_lib.FOLD_STACK_BYTES,), torch.uint8)
        p = self.empty((rows,), torch.float64)
        if want_nn:
            nn_j = self.empty((rows,), torch.int32)
            nn_d = self.empty((rows,), torch.float64)
            nn_tie = self.empty((rows,), torch.int8)
            ptrs = (_ptr(nn_j), _ptr(nn_d), _ptr(nn_tie))
        else:
            ptrs = (None, None, None)
        check(self.lib.isoc_sigma_partial(_ptr(X), n, d, lo, hi, float(alpha), _ptr(stack), *ptrs, _ptr(p),
                                          self.stream))
        return stack, ((nn_j, nn_d, nn_tie) if want_nn else None), p

    def sigma_finish(self, stacks) -> float:
        total = ctypes.c_double(0.0)
        check(self.lib.isoc_sigma_finish(_ptr(stacks), stacks.shape[0], ctypes.byref(total),
                                         self.stream))
        return total.value

    def sym_block_range(self, n: int, rank: int, world: int) -> tuple:
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.isoc_sym_block_range(n, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
        return int(lo.value), int(hi.value)

    def omega_block_range(self, n: int, rank: int, world: int) -> tuple:
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.isoc_omega_block_range(n, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
        return int(lo.value), int(hi.value)

    def sigma_sym_range(self, X, n: int, d: int, jlo: int, jhi: int, want_nn: bool = True):
        """This rank's partial leaf stacks and neighbours for all n rows."""
        torch = self.torch
        vals = self.empty((n, _lib.ROW_CAP), torch.float64)
        ids = self.empty((n, _lib.ROW_CAP), torch.int64)
        cnt = self.empty((n,), torch.int32)
        if want_nn:
            m1, m2, j1 = (self.empty((n,), torch.float64), self.empty((n,), torch.float64),
                          self.empty((n,), torch.int32))
            nnp = (_ptr(m1), _ptr(m2), _ptr(j1))
        else:
            m1 = m2 = j1 = None
            nnp = (None, None, None)
        check(self.lib.isoc_sigma_sym_range(_ptr(X), n, d, jlo, jhi, _ptr(vals), _ptr(ids), _ptr(cnt), *nnp,
                                            self.stream))
        return vals, ids, cnt, m1, m2, j1

    def sigma_rank_merge(self, X, n: int, d: int, lo: int, hi: int, parts, want_nn: bool = True):
        """Owner side: parts = (vals, ids, cnt, m1, m2, j1) rank-major for
        rows [lo, hi); returns (fold stack, nn) like sigma_partial."""
        torch = self.torch
        vals, ids, cnt, m1, m2, j1 = parts
        G = vals.shape[0]
        rows = hi - lo
        stack = self.empty((_lib.FOLD_STACK_BYTES,), torch.uint8)
        if want_nn and m1 is not None:
            nn_j = self.empty((rows,), torch.int32)
            nn_d = self.empty((rows,), torch.float64)
            nn_tie = self.empty((rows,), torch.int8)
            nnin = (_ptr(m1), _ptr(m2), _ptr(j1))
            nnout = (_ptr(nn_j), _ptr(nn_d), _ptr(nn_tie))
        else:
            nnin = (None, None, None)
            nnout = (None, None, None)
        check(self.lib.isoc_sigma_rank_merge(_ptr(X), n, d, lo, hi, G, _ptr(vals), _ptr(ids), _ptr(cnt), *nnin,
                                             _ptr(stack), *nnout, self.stream))
        return stack, ((nn_j, nn_d, nn_tie) if (want_nn and m1 is not None) else None)

    def omega(self, X, n: int, d: int, lo: int, hi: int, sigma: float):
        out = self.empty((hi - lo,), self.torch.float64)
        check(self.lib.isoc_omega(_ptr(X), n, d, lo, hi, float(sigma), _ptr(out), self.stream))
        return out

    def omega_mst(self, X, n: int, d: int, lo: int, hi: int, sigma: float, h):
        """omega rows plus the fused Boruvka round-2 minima (exact)."""
        torch = self.torch
        rows = hi - lo
        out = self.empty((rows,), torch.float64)
        nn_j = self.empty((rows,), torch.int32)
        nn_d = self.empty((rows,), torch.float64)
        nn_tie = self.empty((rows,), torch.int8)
        check(self.lib.isoc_omega_mst(_ptr(X), n, d, lo, hi, float(sigma), h, _ptr(out), _ptr(nn_j),
                                      _ptr(nn_d), _ptr(nn_tie), self.stream))
        return out, (nn_j, nn_d, nn_tie)

    def omega_shard_counts(self, n: int, G: int, rank: int) -> tuple:
        """Slots this rank sends to each owner / receives from each sender."""
        send = (ctypes.c_int64 * G)()
        recv = (ctypes.c_int64 * G)()
        check(self.lib.isoc_omega_shard_counts(n, G, rank, send, recv))
        return [int(v) for v in send], [int(v) for v in recv]

    def omega_sym_range(self, X, n: int, d: int, rank: int, G: int, sigma: float, h=None):
        """This rank's flow subtrees (and, with the MST handle h, round-2
        minima): exactly the slots it produces, grouped by owner -- the send
        buffers of one all-to-all with per-peer split sizes."""
        torch = self.torch
        send, _ = self.omega_shard_counts(n, G, rank)
        tot = max(1, sum(send))
        ps = self.empty((tot,), torch.float64)
        psm = self.empty((tot,), torch.float64) if h is not None else None
        psj = self.empty((tot,), torch.int32) if h is not None else None
        check(self.lib.isoc_omega_sym_range(_ptr(X), n, d, rank, G, float(sigma), h, _ptr(ps),
                                             None if psm is None else _ptr(psm),
                                             None if psj is None else _ptr(psj), self.stream))
        return ps, psm, psj

    def omega_rank_merge(self, n: int, rank: int, G: int, ps, psm=None, psj=None):
        """Owner side: the senders' messages for this rank's rows -> (omega, nn)."""
        torch = self.torch
        lo, hi = n * rank // G, n * (rank + 1) // G
        rows = hi - lo
        out = self.empty((rows,), torch.float64)
        nn = None
        if psm is not None:
            nn = (self.empty((rows,), torch.int32), self.empty((rows,), torch.float64),
                  self.empty((rows,), torch.int8))
        check(self.lib.isoc_omega_rank_merge(n, rank, G, _ptr(ps), None if psm is None else _ptr(psm),
                                             None if psj is None else _ptr(psj), _ptr(out),
                                             *((None, None, None) if nn is None else tuple(_ptr(t) for t in nn)),
                                             self.stream))
        return out, nn

    # -- Boruvka ------------------------------------------------------
    def mst_create(self, X, n: int, d: int, lo: int, hi: int):
        h = ctypes.c_void_p()
        check(self.lib.isoc_mst_create(_ptr(X), n, d, lo, hi, self.stream, ctypes.byref(h)))
        return h

    def mst_round_local(self, h, n: int, nn=None):
        """Local rows' per-component exact minimum weight keys (int64, n)."""
        cmin = self.empty((n,), self.torch.int64)
        if nn is not None:
            check(self.lib.isoc_mst_round_local(h, 1, _ptr(nn[0]), _ptr(nn[1]), _ptr(nn[2]), _ptr(cmin)))
        else:
            check(self.lib.isoc_mst_round_local(h, 0, None, None, None, _ptr(cmin)))
        return cmin

    def mst_round_edges(self, h, cmin):
        """Packed endpoint keys of local rows attaining the (global) minima."""
        cedge = self.empty(tuple(cmin.shape), self.torch.int64)
        check(self.lib.isoc_mst_round_edges(h, _ptr(cmin), _ptr(cedge)))
        return cedge

    def mst_round_finish(self, h, cmin, cedge):
        """Hook + contract with the global keys; (components, ties, rescans)."""
        comps, ties, rescans = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.isoc_mst_round_finish(h, _ptr(cmin), _ptr(cedge), ctypes.byref(comps),
                                             ctypes.byref(ties), ctypes.byref(rescans)))
        return comps.value, ties.value, rescans.value

    def mst_edges(self, h, n: int):
        torch = self.torch
        u = self.empty((n - 1,), torch.int32)
        v = self.empty((n - 1,), torch.int32)
        w = self.empty((n - 1,), torch.float64)
        check(self.lib.isoc_mst_edges(h, _ptr(u), _ptr(v), _ptr(w)))
        return u, v, w

    def prim_edges(self, X, n: int, d: int, root: int):
        """isoc_prim_edges: the reference's Prim tree (tie rule included)."""
        torch = self.torch
        u = self.empty((n - 1,), torch.int32)
        v = self.empty((n - 1,), torch.int32)
        w = self.empty((n - 1,), torch.float64)
        check(self.lib.isoc_prim_edges(_ptr(X), n, d, root, _ptr(u), _ptr(v), _ptr(w), self.stream))
        return u, v, w

    def mst_filter_stats(self, h):
        """(256-row blocks scanned by the tc filter, blocks x filter rounds,
        rows whose candidate list ran out)."""
        if not hasattr(self.lib, "isoc_mst_filter_stats"):   # an older variant build (ISOC_LIB_PATH)
            return None
        run, tot, rows = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.isoc_mst_filter_stats(h, ctypes.byref(run), ctypes.byref(tot), ctypes.byref(rows)))
        return run.value, tot.value, rows.value

    def mst_destroy(self, h) -> None:
        self.lib.isoc_mst_destroy(h)

    # -- trees ----------------------------------------------------------
    def tree_from_edges(self, u, v, w, n: int, root: int, sigma: float) -> "DeviceTree":
        h = ctypes.c_void_p()
        check(self.lib.isoc_tree_from_edges(_ptr(u), _ptr(v), _ptr(w), n, root, float(sigma),
                                             self.stream, ctypes.byref(h)))
        return DeviceTree(self, h, n)

    def tree_from_parent(self, parent: np.ndarray, flows: np.ndarray, root: Optional[int],
                         child_id: Optional[np.ndarray] = None) -> "DeviceTree":
        """root None: the array's unique sentinel, found (and every index
        validated) on the device; DeviceTree.root holds it."""
        n = parent.shape[0]
        par = self.to_device(np.ascontiguousarray(parent, dtype=np.int64))
        fl = self.to_device(np.ascontiguousarray(flows, dtype=np.float64))
        cid = None if child_id is None else self.to_device(np.ascontiguousarray(child_id, dtype=np.int64))
        h = ctypes.c_void_p()
        check(self.lib.isoc_tree_from_parent(_ptr(par), _ptr(fl), None if cid is None else _ptr(cid),
                                             n, -1 if root is None else int(root), self.stream, ctypes.byref(h)))
        dt = DeviceTree(self, h, n)
        r = ctypes.c_int64()
        check(self.lib.isoc_tree_root(h, ctypes.byref(r)))
        dt.root = int(r.value)
        return dt


@dataclass
class Witness:
    labels: np.ndarray
    cut: np.ndarray
    eta: np.ndarray
    sparsities: list
    miso: float


class DeviceTree:
    """Owner of an isoc_tree handle (BFS-position layout on the device)."""

    def __init__(self, backend: CudaBackend, handle, n: int):
        self.b = backend
        self.h = handle
        self.n = n
        self.weights_set = False

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            try:
                self.b.lib.isoc_tree_destroy(h)
            except Exception:
                pass

    def _host(self, n: int, dtype):
        """Page-locked host array (device->host copies at full PCIe/C2C rate)."""
        return self.b.pinned_empty(n, dtype)

    def export(self):
        n = self.n
        parent = self._host(n, np.int64)
        flow = self._host(n, np.float64)
        depth = self._host(n, np.int64)
        cid = self._host(n, np.int64)
        order = self._host(n, np.int64)
        pdist = self._host(n, np.float64)
        md = ctypes.c_int64()
        check(self.b.lib.isoc_tree_export(self.h, parent.ctypes.data, flow.ctypes.data, depth.ctypes.data,
                                          cid.ctypes.data, order.ctypes.data, ctypes.byref(md),
                                          pdist.ctypes.data))
        return parent, flow, depth, cid, order, int(md.value), pdist

    def set_weights(self, omega_dev, p_dev) -> Extrema:
        ext = np.empty(6, np.float64)
        check(self.b.lib.isoc_tree_set_weights(self.h, _ptr(omega_dev), _ptr(p_dev), ext.ctypes.data))
        self.weights_set = True
        return Extrema(*[float(v) for v in ext])

    def decide(self, N: float, k: int, slot: int) -> int:
        j = ctypes.c_int64()
        check(self.b.lib.isoc_decide(self.h, float(N), int(k), int(slot), ctypes.byref(j)))
        return int(j.value)

    def decide_batch(self, thresholds, k: int) -> list:
        """Cut counts j at up to batch_capacity() thresholds in one level-synchronous pass."""
        thr = np.ascontiguousarray(thresholds, dtype=np.float64)
        j = np.empty(thr.shape[0], np.int64)
        check(self.b.lib.isoc_decide_batch(self.h, thr.ctypes.data, int(thr.shape[0]), int(k), j.ctypes.data))
        return [int(v) for v in j]

    def cost(self, labels: np.ndarray, k: int) -> float:
        """subpartition_cost of given labels on this tree's weights."""
        lab = self.b.to_device(np.ascontiguousarray(labels, dtype=np.int64))
        miso = ctypes.c_double()
        check(self.b.lib.isoc_tree_cost(self.h, _ptr(lab), int(k), ctypes.byref(miso)))
        return float(miso.value)

    def batch_capacity(self) -> int:
        """Thresholds per isoc_decide_batch: 63 on trees that fit one CTA's
        shared memory (one warp each), else 16."""
        cap = ctypes.c_int32()
        check(self.b.lib.isoc_decide_batch_capacity(self.h, ctypes.byref(cap)))
        return int(cap.value)

    def shape(self) -> tuple:
        lv, mw = ctypes.c_int64(), ctypes.c_int64()
        check(self.b.lib.isoc_tree_shape(self.h, ctypes.byref(lv), ctypes.byref(mw)))
        return int(lv.value), int(mw.value)

    def witness(self, slot: int, k: int) -> Witness:
        n = self.n
        labels = self._host(n, np.int64)
        cut = self._host(n, np.int8)
        eta = self._host(n, np.int64)
        sp = np.empty(k, np.float64)
        miso = ctypes.c_double()
        check(self.b.lib.isoc_witness(self.h, int(slot), int(k), labels.ctypes.data, cut.ctypes.data,
                                      eta.ctypes.data, sp.ctypes.data, ctypes.byref(miso)))
        return Witness(labels, cut, eta, [float(v) for v in sp], float(miso.value))
