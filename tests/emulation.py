"""CPU stand-in for the device backend (TEST INFRASTRUCTURE ONLY).

Implements the per-shard primitives of engine.CudaBackend with the CPU
oracle so that the product's multi-rank orchestration in
paper_1702_04739_b200.pipeline (row sharding, fold-stack exchange in rank
order, the two MIN all-reduces per Boruvka round, hook/contract replicated on
every rank) can run under torch.distributed with the gloo backend on a
machine without a GPU.  The fold-stack wire format is the library's
(ISOC_FOLD_STACK_BYTES: count, overflow, uint64 id[96], double value[96]).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle as orc

CAP = 96
NO_KEY = 0x7FFFFFFFFFFFFFFF


def _split(n):
    n2 = n // 2
    return n2 - n2 % 8


def find_leaf(total, pos):
    s, n, hid = 0, total, 1
    while n > 128:
        n2 = _split(n)
        if pos < s + n2:
            n, hid = n2, hid * 2
        else:
            s, n, hid = s + n2, n - n2, hid * 2 + 1
    return s, n, hid


def leaf_sum(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += x
        return r
    r = [float(x) for x in a[:8]]
    i = 8
    while i < n - n % 8:
        for j in range(8):
            r[j] += a[i + j]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        res += a[i]
        i += 1
    return res


def push(st, v, h):
    while st and (h & 1) and st[-1][1] == h - 1:
        v = st[-1][0] + v
        st.pop()
        h >>= 1
    st.append((v, h))


def pack_stack(st) -> torch.Tensor:
    buf = np.zeros(8 + 16 * CAP, dtype=np.uint8)
    hdr = np.array([len(st), 0], dtype=np.int32)
    ids = np.zeros(CAP, dtype=np.uint64)
    vals = np.zeros(CAP, dtype=np.float64)
    for i, (v, h) in enumerate(st):
        ids[i], vals[i] = h, v
    buf[:8] = hdr.view(np.uint8)
    buf[8:8 + 8 * CAP] = ids.view(np.uint8)
    buf[8 + 8 * CAP:] = vals.view(np.uint8)
    return torch.from_numpy(buf)


def unpack_stack(t: torch.Tensor):
    b = t.numpy()
    cnt = int(b[:8].view(np.int32)[0])
    ids = b[8:8 + 8 * CAP].view(np.uint64)
    vals = b[8 + 8 * CAP:].view(np.float64)
    return [(float(vals[i]), int(ids[i])) for i in range(cnt)]


class MstState:
    def __init__(self, X, n, lo, hi):
        self.X, self.n, self.lo, self.hi = X, n, lo, hi
        self.comp = np.arange(n, dtype=np.int64)
        self.edges = []
        self.cand = {}


class EmuBackend:
    name = "emulated-cpu"
    device = "cpu"
    torch = torch

    def to_device(self, x):
        return torch.from_numpy(np.ascontiguousarray(x))

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype)

    # K1 restated per shard: row stacks, straddle leaves, merge (the CUDA
    # algorithm of exact_passes.cu, in Python)
    def sigma_partial(self, X, n, d, lo, hi, alpha, want_nn=True):
        Xn = X.numpy()
        total = n * n
        rows = orc.distance_rows(Xn, lo, hi)
        flat_row = lambda i: rows[i - lo]  # noqa: E731
        st = []
        nn_j = np.zeros(hi - lo, np.int32)
        nn_d = np.zeros(hi - lo)
        nn_tie = np.zeros(hi - lo, np.int8)
        for i in range(lo, hi):
            rs, re = i * n, (i + 1) * n
            if i > lo:
                self._straddle(Xn, n, total, i, st)
            s, l, h = find_leaf(total, rs)
            if s < rs:
                if s + l < re:
                    s, l, h = find_leaf(total, s + l)
                else:
                    l = 0
            while l > 0 and s + l <= re and not (s + l == total and total % 8):
                push(st, leaf_sum(flat_row(i)[s - rs:s + l - rs]), h)
                if s + l >= re:
                    break
                s, l, h = find_leaf(total, s + l)
            r = flat_row(i).copy()
            r[i] = np.inf
            j = int(np.argmin(r))
            nn_j[i - lo], nn_d[i - lo] = j, r[j]
            r2 = r.copy()
            r2[j] = np.inf
            nn_tie[i - lo] = int(r2.min() == r[j])
        self._straddle(Xn, n, total, hi, st)
        p = np.zeros(hi - lo) if alpha == 0 else orc.row_folds(Xn, 1.0, alpha, lo, hi)[1]
        nn = (torch.from_numpy(nn_j), torch.from_numpy(nn_d), torch.from_numpy(nn_tie)) if want_nn else None
        return pack_stack(st), nn, torch.from_numpy(p)

    # sharded symmetric sigma (pipeline._sigma_pass with world > 1): the
    # rank's per-row partial stacks over its column-block range, restated
    SYM_BLOCK = 2048      # sigma_sym.cu YB
    OMEGA_BLOCK = 1024    # omega_sym.cu SB

    def sym_block_range(self, n, rank, world, block=None):
        import math
        nbs = -(-n // (block or self.SYM_BLOCK))
        tot = nbs * (nbs + 1) / 2.0

        def bound(k):
            if k <= 0:
                return 0
            if k >= world:
                return nbs
            target = tot * k / world
            return max(0, min(nbs, int(math.ceil((math.sqrt(8.0 * target + 1.0) - 1.0) / 2.0))))
        return bound(rank), bound(rank + 1)

    def sigma_sym_range(self, X, n, d, jlo, jhi, want_nn=True):
        Xn = X.numpy()
        total, B = n * n, self.SYM_BLOCK
        cap = 40
        vals = np.zeros((n, cap))
        ids = np.zeros((n, cap), np.int64)
        cnt = np.zeros(n, np.int32)
        m1 = np.full(n, np.inf)
        m2 = np.full(n, np.inf)
        j1 = np.full(n, 2**31 - 1, np.int32)
        rows = orc.distance_rows(Xn, 0, n)
        for r in range(n):
            K = r // B
            if K < jlo:
                a, b = jlo, jhi
            elif K < jhi:
                a, b = 0, jhi
            else:
                continue
            rs, re = r * n, (r + 1) * n
            # internal leaves of the row (as sigma_partial) starting in [a*B, b*B)
            st = []
            s_, l, h = find_leaf(total, rs)
            if s_ < rs:
                s_, l, h = find_leaf(total, s_ + l) if s_ + l < re else (re, 0, 0)
            while l > 0 and s_ + l <= re and not (s_ + l == total and total % 8):
                if rs + a * B <= s_ < rs + b * B:
                    push(st, leaf_sum(rows[r][s_ - rs:s_ + l - rs]), h)
                if s_ + l >= re:
                    break
                s_, l, h = find_leaf(total, s_ + l)
            cnt[r] = len(st)
            for e, (v, hh) in enumerate(st):
                vals[r, e], ids[r, e] = v, np.uint64(hh).view(np.int64)
            if want_nn:
                row = rows[r][a * B:min(b * B, n)].copy()
                if a * B <= r < b * B:
                    row[r - a * B] = np.inf
                if row.size and np.isfinite(row.min()):
                    j = int(np.argmin(row))
                    m1[r], j1[r] = row[j], a * B + j
                    rr = row.copy()
                    rr[j] = np.inf
                    m2[r] = rr.min()
        t = torch.from_numpy
        nnp = (t(m1), t(m2), t(j1)) if want_nn else (None, None, None)
        return (t(vals), t(ids), t(cnt)) + nnp

    def sigma_rank_merge(self, X, n, d, lo, hi, parts, want_nn=True):
        Xn = X.numpy()
        total = n * n
        vals, ids, cnt, m1, m2, j1 = parts
        G = vals.shape[0]
        st = []
        nn_j = np.zeros(hi - lo, np.int32)
        nn_d = np.zeros(hi - lo)
        nn_tie = np.zeros(hi - lo, np.int8)
        for i in range(lo, hi):
            q = i - lo
            if i > lo:
                self._straddle(Xn, n, total, i, st)
            for g in range(G):
                for e in range(int(cnt[g, q])):
                    push(st, float(vals[g, q, e]), int(np.int64(ids[g, q, e]).view(np.uint64)))
            if want_nn and m1 is not None:
                best = (np.inf, 2**31 - 1)
                sec = np.inf
                for g in range(G):
                    c = (float(m1[g, q]), int(j1[g, q]))
                    if c < best:
                        sec = min(sec, best[0], float(m2[g, q]))
                        best = c
                    else:
                        sec = min(sec, c[0])
                nn_j[q] = -1 if best[1] == 2**31 - 1 else best[1]
                nn_d[q] = best[0]
                nn_tie[q] = int(sec == best[0])
        self._straddle(Xn, n, total, hi, st)
        nn = (torch.from_numpy(nn_j), torch.from_numpy(nn_d), torch.from_numpy(nn_tie)) if want_nn else None
        return pack_stack(st), nn

    @staticmethod
    def _straddle(Xn, n, total, b, st):
        if b < n:
            s, l, h = find_leaf(total, b * n)
            own = s < b * n and s // n == b - 1
        else:
            s, l, h = find_leaf(total, total - 1)
            own = total % 8 != 0 and s >= (n - 1) * n
        if own:
            vals = [orc.pair_distance(Xn, f // n, f % n) for f in range(s, s + l)]
            push(st, leaf_sum(vals), h)

    def sigma_finish(self, stacks):
        st = []
        for q in range(stacks.shape[0]):
            for v, h in unpack_stack(stacks[q]):
                push(st, v, h)
        assert len(st) == 1 and st[0][1] == 1, st
        return 0.0 + st[0][0]

    def omega(self, X, n, d, lo, hi, sigma):
        return torch.from_numpy(orc.row_folds(X.numpy(), sigma, 0.0, lo, hi)[0])

    def omega_mst(self, X, n, d, lo, hi, sigma, h):
        om = self.omega(X, n, d, lo, hi, sigma)
        self.mst_round_local(h, n)   # exact per-row minima for round 2
        return om, "fused"

    # sharded symmetric omega (pipeline._omega_pass with world > 1): complete
    # 1024-wide flow subtrees per (row, super-block) into owner-major slots
    def omega_block_range(self, n, rank, world):
        return self.sym_block_range(n, rank, world, self.OMEGA_BLOCK)

    def _omega_plan(self, n, G):
        """omega_sym.cu omega_plan_build: per (sender s, owner g) message
        offsets of the first row of g in each block, message sizes, send /
        receive displacements."""
        B = self.OMEGA_BLOCK
        nbs = -(-n // B)
        rng = [self.omega_block_range(n, s, G) for s in range(G)]
        T = np.zeros((G, G, nbs + 1), np.int64)
        for s, (jlo, jhi) in enumerate(rng):
            for g in range(G):
                lo_g, hi_g = n * g // G, n * (g + 1) // G
                acc = 0
                for blk in range(nbs + 1):
                    T[s, g, blk] = acc
                    if blk == nbs:
                        break
                    rows = max(0, min(hi_g, (blk + 1) * B) - max(lo_g, blk * B))
                    cnt = jhi - jlo if blk < jlo else (jhi if blk < jhi else 0)
                    acc += rows * cnt
        MC = T[:, :, nbs]
        return rng, T, MC, nbs

    def omega_shard_counts(self, n, G, rank):
        _, _, MC, _ = self._omega_plan(n, G)
        return [int(v) for v in MC[rank, :]], [int(v) for v in MC[:, rank]]

    def _msg_off(self, plan, n, G, s, g, i, b):
        rng, T, _, _ = plan
        B = self.OMEGA_BLOCK
        blk = i // B
        jlo, jhi = rng[s]
        cnt = jhi - jlo if blk < jlo else (jhi if blk < jhi else 0)
        bst = jlo if blk < jlo else 0
        r0 = max(n * g // G, blk * B)
        return int(T[s, g, blk]) + (i - r0) * cnt + (b - bst)

    def omega_sym_range(self, X, n, d, rank, G, sigma, h=None):
        Xn = X.numpy()
        B = self.OMEGA_BLOCK
        plan = self._omega_plan(n, G)
        rng, _, MC, nbs = plan
        jlo, jhi = rng[rank]
        sd = np.concatenate([[0], np.cumsum(MC[rank, :])])
        tot = max(1, int(sd[-1]))
        ps = np.zeros(tot)
        psm = np.full(tot, np.inf)
        psj = np.full(tot, 2**31 - 1, np.int32)
        D = orc.distance_rows(Xn, 0, n)
        F = orc.exp(np.negative(D) / sigma)
        np.fill_diagonal(F, 0.0)
        Fp = np.zeros((n, nbs * B))
        Fp[:, :n] = F

        def owner(i):
            r = i * G // n
            while n * (r + 1) // G <= i:
                r += 1
            while n * r // G > i:
                r -= 1
            return r

        def put(i, b):
            seg = Fp[i, b * B:(b + 1) * B]
            while seg.size > 1:
                seg = seg[0::2] + seg[1::2]
            g = owner(i)
            o = int(sd[g]) + self._msg_off(plan, n, G, rank, g, i, b)
            ps[o] = seg[0]
            if h is not None:
                row = D[i, b * B:min((b + 1) * B, n)].copy()
                row[h.comp[b * B:b * B + row.size] == h.comp[i]] = np.inf
                if row.size and np.isfinite(row.min()):
                    j = int(np.argmin(row))
                    psm[o] = row[j]
                    # exact tie flag in the index's sign bit (omega_sym.cu TIEBIT)
                    tie = int(np.count_nonzero(row == row[j]) > 1)
                    psj[o] = np.int32(np.uint32((b * B + j) | (tie << 31)).view(np.int32))

        for J in range(jlo, jhi):
            for I in range(J + 1):
                for i in range(I * B, min((I + 1) * B, n)):
                    put(i, J)
                if I < J:
                    for j in range(J * B, min((J + 1) * B, n)):
                        put(j, I)
        t = torch.from_numpy
        return t(ps), (t(psm) if h is not None else None), (t(psj) if h is not None else None)

    def omega_rank_merge(self, n, rank, G, ps, psm=None, psj=None):
        plan = self._omega_plan(n, G)
        rng, _, MC, nbs = plan
        rd = np.concatenate([[0], np.cumsum(MC[:, rank])])
        P = ps.numpy()
        lo, hi = n * rank // G, n * (rank + 1) // G
        om = np.empty(hi - lo)
        nn_j = np.full(hi - lo, -1, np.int32)
        nn_d = np.full(hi - lo, np.inf)
        nn_t = np.zeros(hi - lo, np.int8)
        B = self.OMEGA_BLOCK
        for q in range(hi - lo):
            i = lo + q
            blk = i // B
            offs = []
            for b in range(nbs):
                m = max(b, blk)
                s = next(s for s, (a, e) in enumerate(rng) if a <= m < e)
                offs.append(int(rd[s]) + self._msg_off(plan, n, G, s, rank, i, b))
            w = np.zeros(1 << max(0, (nbs - 1).bit_length()))
            w[:nbs] = P[offs]
            while w.size > 1:
                w = w[0::2] + w[1::2]
            om[q] = w[0]
            if psm is not None:
                m, mj, tie = np.inf, 2**31 - 1, 0
                for o in offs:
                    x = float(psm[o])
                    raw = int(np.int32(psj[o]).view(np.uint32))
                    xj, xt = raw & 0x7FFFFFFF, raw >> 31
                    if x < m:
                        m, mj, tie = x, xj, xt
                    elif x == m and np.isfinite(x):
                        mj, tie = min(mj, xj), 1
                if mj != 2**31 - 1:
                    nn_j[q], nn_d[q], nn_t[q] = mj, m, tie
        nn = None
        if psm is not None:
            nn = (torch.from_numpy(nn_j), torch.from_numpy(nn_d), torch.from_numpy(nn_t))
        return torch.from_numpy(om), nn

    # Boruvka primitives on the shard's rows (exact per-row minima)
    def mst_create(self, X, n, d, lo, hi):
        return MstState(X.numpy(), n, lo, hi)

    def mst_round_local(self, h, n, nn=None):
        cmin = np.full(n, NO_KEY, dtype=np.int64)
        h.cand = {}
        if getattr(h, "D", None) is None:
            h.D = orc.distance_rows(h.X, h.lo, h.hi)
        R = h.D.copy()
        R[h.comp[h.lo:h.hi, None] == h.comp[None, :]] = np.inf
        js = np.argmin(R, axis=1)
        for q, j in enumerate(js.tolist()):
            i = h.lo + q
            if not np.isfinite(R[q, j]):
                continue
            h.cand[i] = (R[q, j], j)
            key = int(np.float64(R[q, j]).view(np.int64))
            c = h.comp[i]
            cmin[c] = min(cmin[c], key)
        if isinstance(nn, tuple):
            # minima handed in by a fused pass (sharded omega's round 2)
            # must be the exact per-row minima recomputed here
            for i, (w, j) in h.cand.items():
                assert int(nn[0][i - h.lo]) == j and float(nn[1][i - h.lo]) == w, (i, j, w)
        return torch.from_numpy(cmin)

    def mst_round_edges(self, h, cmin):
        cm = cmin.numpy()
        ce = np.full(h.n, NO_KEY, dtype=np.int64)
        for i, (w, j) in h.cand.items():
            c = h.comp[i]
            if int(np.float64(w).view(np.int64)) == cm[c]:
                ce[c] = min(ce[c], (min(i, j) << 32) | max(i, j))
        return torch.from_numpy(ce)

    def mst_round_finish(self, h, cmin, cedge):
        cm, ce = cmin.numpy(), cedge.numpy()
        comp = h.comp
        reps = np.flatnonzero(comp == np.arange(h.n))
        succ = np.arange(h.n)
        for c in reps:
            if ce[c] == NO_KEY:
                continue
            a, b = int(ce[c]) >> 32, int(ce[c]) & 0xFFFFFFFF
            succ[c] = comp[b] if comp[a] == c else comp[a]
        succ2 = succ.copy()
        for c in reps:
            s = succ[c]
            if s != c and succ[s] == c and c < s:
                s = c
            succ2[c] = s
            if s != c:
                a, b = int(ce[c]) >> 32, int(ce[c]) & 0xFFFFFFFF
                h.edges.append((a, b, float(np.int64(cm[c]).view(np.float64))))
        for _ in range(64):
            nxt = succ2[succ2]
            if np.array_equal(nxt, succ2):
                break
            succ2 = nxt
        h.comp = succ2[comp]
        return int(np.sum(h.comp == np.arange(h.n))), 0, 0

    def mst_edges(self, h, n):
        e = sorted(h.edges)
        u = torch.tensor([a for a, _, _ in e], dtype=torch.int32)
        v = torch.tensor([b for _, b, _ in e], dtype=torch.int32)
        w = torch.tensor([x for _, _, x in e], dtype=torch.float64)
        return u, v, w

    def mst_destroy(self, h):
        pass
