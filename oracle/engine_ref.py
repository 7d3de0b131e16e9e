"""ORACLE — test infrastructure only (tests/, smoke(), bench cpu_baseline).

CPU restatement (numpy / scipy) of the reference's generalized LDL^T engine,
`/root/reference/pkg/src/h2slice/gldl.py:179-633`.  It is the checker the
CUDA engine is compared with, and the CPU baseline bench.py times
(`cpu_baseline.kind = "port"`); it is never called by the product path.

Pinned against the reference itself: tests/test_oracle.py replays the
reference's own inertia counts recorded in tests/golden/*.npz (made by
tests/golden/make_golden.py with the reference imported from
/root/reference) on the identical exported H payloads.

Structure of one run (reference line numbers):
  * leaf assembly, skeleton congruences Q^T A Q      gldl.py:229-256, compress.py:99-127
  * per level, ascending clusters:
      - recompression of fill rows (pivoted QR, abs. Frobenius tail)  gldl.py:67-79, 296-347
      - BK of the redundant block, inertia, panel solve, Schur/fill   gldl.py:349-426
  * fill -> coupling fold on the level's low-rank pairs             gldl.py:284-294
  * pairwise merge with parent bases / flat merge / root BK          gldl.py:429-602
  * retry wrapper with mu <- mu(1+d)+d                              gldl.py:615-633
"""

import time
from collections import defaultdict
from itertools import combinations

import numpy as np
import scipy.linalg

from .dense_ref import Breakdown, inertia_of, ldl_symmetric

RETRY_DELTA = 1e-11
MAX_SHIFT_RETRIES = 3


class ShiftHit(Exception):
    pass


class Unstable(Exception):
    pass


class Deadline(Exception):
    """Bounded-sample stop (bench cpu_baseline): work done when the time ran out."""

    def __init__(self, elim_flops, seconds, clusters):
        super().__init__(f"deadline after {clusters} clusters, {seconds:.1f} s")
        self.elim_flops, self.seconds, self.clusters = elim_flops, seconds, clusters


def abs_split(G, tol):
    """Pivoted QR of G; rank = first r with ||R[r:, :]||_F <= tol (gldl.py:67-79)."""
    Q, R, _ = scipy.linalg.qr(G, mode="full", pivoting=True)
    k = min(G.shape)
    rows = np.sum(R[:k] ** 2, axis=1)
    tail = np.sqrt(np.append(np.cumsum(rows[::-1])[::-1], 0.0))
    rank = int(np.searchsorted(-tail, -tol))
    return rank, Q[:, :rank], Q[:, rank:], float(tail[rank])


class _Node:
    __slots__ = ("m", "nR", "nS", "r0")

    def __init__(self, m, nR, nS):
        self.m, self.nR, self.nS, self.r0 = m, nR, nS, nS


def _key(a, b):
    return (a, b) if a < b else (b, a)


class OracleEngine:
    """One factorization of origin(H) - shift*I; counts accumulate in self.counts."""

    def __init__(self, H, shift, skel_cache=None, deadline_s=None):
        self.deadline_s = deadline_s
        self.elim_flops = 0.0   # survey §8d count, live rows (== the engine's elim_flops)
        self.done = set()       # eliminated clusters of the current level
        self.H = H.origin()
        self.tree = self.H.tree
        self.st = self.H.structure
        self.shift = float(shift)
        self.delta = self.shift - self.H.shift
        self.counts = [0, 0, 0]
        self.stats = dict(fill_blocks=0, recompressions=0, rank_added=0, dropped_fro=0.0,
                          max_front=0)
        self.tol = self.H.eps * (self.H.scale0() + abs(self.delta))
        self.cache = skel_cache if skel_cache is not None else {}

    # -------------------------------------------------- skeleton prologue (K1)
    def _skel(self, key):
        got = self.cache.get(key)
        if got is None:
            L = self.tree.depth
            if key[0] == "d":
                i = key[1]
                bs = self.H.bases.get((L, i))
                base = self.H.leaf_diag[i]
                got = base if bs is None else bs.square().T @ base @ bs.square()
            else:
                _, i, j = key
                got = (self.H.bases[(L, i)].square().T @ self.H.leaf_offdiag[(i, j)]
                       @ self.H.bases[(L, j)].square())
            self.cache[key] = got
        return got

    def _skel_diag(self, i):
        S = self._skel(("d", i))
        return S - self.delta * np.eye(S.shape[0]) if self.delta else S.copy()

    def run(self):
        if self.tree.depth == 0:
            self._root(self._skel_diag(0))
            return self
        self._leaf_level()
        self._t0 = time.perf_counter()
        self._nclus = 0
        level = self.tree.depth
        while True:
            self._sweep(level)
            if self.st.kind == "flat":
                root = self._merge_flat()
                break
            if level == 1:
                root = self._merge_up(1, root=True)
                break
            self._merge_up(level, root=False)
            level -= 1
        self._root(root)
        return self

    # ------------------------------------------------------------ leaf level
    def _leaf_level(self):
        L = self.tree.depth
        self.node, self.D = {}, {}
        self.off, self.cp, self.fl = {}, {}, {}
        self.adj = {"off": defaultdict(set), "fl": defaultdict(set), "cp": defaultdict(set)}
        for i in range(self.tree.num_clusters(L)):
            m = self.tree.size(L, i)
            if m == 0:
                self.node[i] = _Node(0, 0, 0)
                self.D[i] = np.zeros((0, 0))
                continue
            r = self.H.bases[(L, i)].rank
            self.node[i] = _Node(m, m - r, r)
            self.D[i] = self._skel_diag(i)
        for (i, j) in self.st.dense:
            self.off[(i, j)] = self._skel(("o", i, j)).copy()
            self.adj["off"][i].add((i, j))
            self.adj["off"][j].add((i, j))
        for (i, j) in self.st.lowrank_at(L):
            self.cp[(i, j)] = self.H.couplings[(L, i, j)].copy()
            self.adj["cp"][i].add((i, j))
            self.adj["cp"][j].add((i, j))

    # ------------------------------------------------------------ level sweep
    def _sweep(self, level):
        self.done = set()
        for i in range(self.tree.num_clusters(level)):
            if self.node[i].m:
                self._recompress(i)
                self._eliminate(i)
                self._nclus += 1
                if self.deadline_s is not None:
                    dt = time.perf_counter() - self._t0
                    if dt > self.deadline_s:
                        raise Deadline(self.elim_flops, dt, self._nclus)
        low = set(self.st.lowrank_at(level))
        for key in [k for k in self.fl if k in low]:
            a, b = key
            F = self.fl.pop(key)
            self.cp[key] = self.cp[key] + F[self.node[a].nR:, self.node[b].nR:]
            self.adj["fl"][a].discard(key)
            self.adj["fl"][b].discard(key)

    def _recompress(self, i):
        nd = self.node[i]
        nR = nd.nR
        keys = self.adj["fl"][i]
        if nR == 0 or not keys:
            return
        parts = []
        for k in keys:
            piece = self.fl[k][:nR, :] if k[0] == i else self.fl[k][:, :nR].T
            if piece.any():
                parts.append(piece)
        if parts:
            t, Us, Ur, dropped = abs_split(np.hstack(parts), self.tol)
            self.stats["recompressions"] += 1
            self.stats["dropped_fro"] += dropped
            if t:
                new_nR = nR - t
                # new coordinates: [Ur^T R ; S ; Us^T R]  (gldl.py:316-319)
                T = np.zeros((nd.m, nd.m))
                T[:new_nR, :nR] = Ur.T
                T[new_nR:new_nR + nd.nS, nR:] = np.eye(nd.nS)
                T[new_nR + nd.nS:, :nR] = Us.T
                self.D[i] = T @ self.D[i] @ T.T
                for store, kind in ((self.off, "off"), (self.fl, "fl")):
                    for k in self.adj[kind][i]:
                        store[k] = T @ store[k] if k[0] == i else store[k] @ T.T
                for k in self.adj["cp"][i]:
                    pad = ((0, t), (0, 0)) if k[0] == i else ((0, 0), (0, t))
                    self.cp[k] = np.pad(self.cp[k], pad)
                nd.nR, nd.nS = new_nR, nd.nS + t
                self.stats["rank_added"] += t
        for k in keys:
            if k[0] == i:
                self.fl[k][:nd.nR, :] = 0.0
            else:
                self.fl[k][:, :nd.nR] = 0.0

    def _eliminate(self, i):
        nd = self.node[i]
        nR = nd.nR
        if nR == 0:
            return
        D = self.D[i]
        self.stats["max_front"] = max(self.stats["max_front"], nd.m)
        try:
            f = ldl_symmetric(D[:nR, :nR])
        except Breakdown as exc:
            raise ShiftHit(self.shift) from exc
        for q, c in enumerate(inertia_of(f)):
            self.counts[q] += c
        partners = sorted(b if a == i else a for a, b in self.adj["off"][i])
        rows = [D[nR:, :nR]]
        for j in partners:
            O = self.off[_key(i, j)]
            rows.append(O[:nR, :].T if i < j else O[:, :nR])
        B = np.vstack(rows)
        if B.shape[0]:
            W = scipy.linalg.solve_triangular(f.L, B[:, f.perm].T, lower=True,
                                              unit_diagonal=True).T
            X = np.linalg.solve(f.D, W.T).T
        else:
            W = X = np.zeros((0, nR))
        # algorithmic count on live rows: BK nR^3/3, panel R nR^2 + R nR, Schur nR R^2
        live = nd.nS + sum(self.node[j].m - (self.node[j].nR if j in self.done else 0)
                           for j in partners)
        self.elim_flops += nR ** 3 / 3.0 + live * nR * nR + live * nR + nR * float(live) ** 2
        seg = {i: (0, nd.nS)}
        pos = nd.nS
        for j in partners:
            seg[j] = (pos, pos + self.node[j].m)
            pos += self.node[j].m

        def xw(a, b):
            (a0, a1), (b0, b1) = seg[a], seg[b]
            return X[a0:a1] @ W[b0:b1].T

        D[nR:, nR:] -= xw(i, i)
        for j in partners:
            self.D[j] -= xw(j, j)
            if i < j:
                self.off[(i, j)][nR:, :] -= xw(i, j)
            else:
                self.off[(j, i)][:, nR:] -= xw(j, i)
        for j, k in combinations(partners, 2):
            upd = xw(j, k)
            if (j, k) in self.off:
                self.off[(j, k)] -= upd
                continue
            F = self.fl.get((j, k))
            if F is None:
                F = np.zeros((self.node[j].m, self.node[k].m))
                self.fl[(j, k)] = F
                self.adj["fl"][j].add((j, k))
                self.adj["fl"][k].add((j, k))
                self.stats["fill_blocks"] += 1
            F -= upd
        D[:nR, :] = 0.0
        D[:, :nR] = 0.0
        for k in self.adj["off"][i]:
            if k[0] == i:
                self.off[k][:nR, :] = 0.0
            else:
                self.off[k][:, :nR] = 0.0
        self.done.add(i)

    # ------------------------------------------------------------------ merge
    def _content(self, key):
        """Skeleton-skeleton content of a finished pair (gldl.py:429-438)."""
        if key in self.cp:
            return self.cp[key]
        a, b = key
        src = self.off.get(key)
        if src is None:
            src = self.fl.get(key)
        if src is None:
            return None
        return src[self.node[a].nR:, self.node[b].nR:]

    def _merge_flat(self):
        L = self.tree.depth
        order = range(self.tree.num_clusters(L))
        start, pos = {}, 0
        for i in order:
            start[i] = pos
            pos += self.node[i].nS
        R = np.zeros((pos, pos))
        for i in order:
            nd = self.node[i]
            R[start[i]:start[i] + nd.nS, start[i]:start[i] + nd.nS] = self.D[i][nd.nR:, nd.nR:]
        for key in set(self.cp) | set(self.off) | set(self.fl):
            C = self._content(key)
            if C is None or C.size == 0:
                continue
            a, b = key
            R[start[a]:start[a] + C.shape[0], start[b]:start[b] + C.shape[1]] = C
            R[start[b]:start[b] + C.shape[1], start[a]:start[a] + C.shape[0]] = C.T
        return R

    def _merge_up(self, level, root):
        nparent = self.tree.num_clusters(level - 1)
        loc = {}  # child -> row offset inside its parent
        raw = {}
        for p in range(nparent):
            c1, c2 = 2 * p, 2 * p + 1
            s1, s2 = self.node[c1].nS, self.node[c2].nS
            loc[c1], loc[c2] = 0, s1
            R = np.zeros((s1 + s2, s1 + s2))
            R[:s1, :s1] = self.D[c1][self.node[c1].nR:, self.node[c1].nR:]
            R[s1:, s1:] = self.D[c2][self.node[c2].nR:, self.node[c2].nR:]
            C = self._content((c1, c2))
            if C is not None and C.size:
                R[:s1, s1:] = C
                R[s1:, :s1] = C.T
            raw[p] = R
        between = {}
        for key in set(self.cp) | set(self.off) | set(self.fl):
            a, b = key
            p, q = a >> 1, b >> 1
            if p == q:
                continue
            C = self._content(key)
            if C is None or C.size == 0:
                continue
            acc = between.get((p, q))
            if acc is None:
                acc = between[(p, q)] = np.zeros((raw[p].shape[0], raw[q].shape[0]))
            acc[loc[a]:loc[a] + C.shape[0], loc[b]:loc[b] + C.shape[1]] += C
        if root:
            return raw[0]
        plevel = level - 1
        node, D, Qs = {}, {}, {}
        for p in range(nparent):
            mp = raw[p].shape[0]
            if mp == 0:
                node[p], D[p], Qs[p] = _Node(0, 0, 0), np.zeros((0, 0)), np.zeros((0, 0))
                continue
            Q, rk = self._parent_basis(level, p)
            node[p] = _Node(mp, mp - rk, rk)
            Qs[p] = Q
            D[p] = Q.T @ raw[p] @ Q
        adj = {"off": defaultdict(set), "fl": defaultdict(set), "cp": defaultdict(set)}
        off, fl, cp = {}, {}, {}
        for key in self.st.deferred_at(plevel):
            p, q = key
            R = between.pop(key, None)
            if R is None:
                R = np.zeros((node[p].m, node[q].m))
            off[key] = Qs[p].T @ R @ Qs[q]
            adj["off"][p].add(key)
            adj["off"][q].add(key)
        for key, R in between.items():
            p, q = key
            fl[key] = Qs[p].T @ R @ Qs[q]
            adj["fl"][p].add(key)
            adj["fl"][q].add(key)
            self.stats["fill_blocks"] += 1
        for key in self.st.lowrank_at(plevel):
            cp[key] = self.H.couplings[(plevel,) + key].copy()
            adj["cp"][key[0]].add(key)
            adj["cp"][key[1]].add(key)
        self.node, self.D, self.off, self.fl, self.cp, self.adj = node, D, off, fl, cp, adj

    def _parent_basis(self, level, p):
        """Parent [U_R | extras | U_S] over the merged child skeletons (gldl.py:561-588)."""
        a, b = self.node[2 * p], self.node[2 * p + 1]
        bs = self.H.bases[(level - 1, p)]
        e1, e2 = a.nS - a.r0, b.nS - b.r0
        if e1 == 0 and e2 == 0:
            return bs.square(), bs.rank
        mp = a.nS + b.nS
        rk = bs.rank
        nRh = a.r0 + b.r0 - rk
        orig = list(range(a.r0)) + list(range(a.nS, a.nS + b.r0))
        extra = list(range(a.r0, a.nS)) + list(range(a.nS + b.r0, mp))
        Q = np.zeros((mp, mp))
        if nRh:
            Q[np.ix_(orig, range(nRh))] = bs.U_R
        if extra:
            Q[np.ix_(extra, range(nRh, nRh + len(extra)))] = np.eye(len(extra))
        if rk:
            Q[np.ix_(orig, range(mp - rk, mp))] = bs.U_S
        return Q, rk

    def _root(self, M):
        if M.size == 0:
            return
        try:
            f = ldl_symmetric(M)
        except Breakdown as exc:
            raise ShiftHit(self.shift) from exc
        for q, c in enumerate(inertia_of(f)):
            self.counts[q] += c


def generalized_ldl(H, shift=None, skel_cache=None):
    """One factorization; returns (neg, zero, pos), stats.  Raises ShiftHit."""
    mu = H.shift if shift is None else shift
    eng = OracleEngine(H, mu, skel_cache).run()
    return tuple(eng.counts), eng.stats


def inertia(H, mu=0.0, max_retries=MAX_SHIFT_RETRIES, skel_cache=None):
    """Retry wrapper of gldl.py:615-633 (mu is relative to H's own shift)."""
    delta = RETRY_DELTA * max(1.0, abs(mu))
    m = mu
    for _ in range(max_retries + 1):
        try:
            c, _ = generalized_ldl(H, H.shift + m, skel_cache)
            if c[1]:
                raise ShiftHit(m)
            return c
        except ShiftHit:
            m = m * (1.0 + delta) + delta
    raise Unstable(mu)


def slice_spectrum(H, k, interval, eps_ev, skel_cache=None):
    """Bisection of spectrum.py:127-178 with a monotone count cache.

    Returns (value, half_width, iterations, evaluations, [(mu, count), ...])."""
    cache = {}
    trace = []
    a, b = float(interval[0]), float(interval[1])

    def branch(mu):
        below = [x for x in cache if x <= mu]
        if below and cache[max(below)] >= k:
            return True
        above = [x for x in cache if x >= mu]
        if above and cache[min(above)] < k:
            return False
        v = inertia(H, mu, skel_cache=skel_cache)[0]
        cache[mu] = v
        trace.append((mu, v))
        return v >= k

    it = 0
    while b - a >= eps_ev:
        it += 1
        mu = 0.5 * (a + b)
        if branch(mu):
            b = mu
        else:
            a = mu
    return 0.5 * (a + b), 0.5 * (b - a), it, len(trace), trace
