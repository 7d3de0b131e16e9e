"""Device-side H2 / HSS / BLR2 construction.

The reference builds its rank-structured matrices by dense sampling on the
CPU (`h2slice/compress.py:146-279`), which takes ~500 s for config 2 and hours
for configs 4-5.  This module runs the same algorithm on the GPU so configs
2-5 can be instantiated in seconds:

* leaf bases: the row block of all admissible same-level partners
  (`construction_partners`, `partition.py:233-249`) is sampled on the device,
  reduced by a QR of its transpose and rank-revealed by an SVD of the small
  triangular factor; rank = first r with Frobenius tail <= eps * (largest
  column norm), the reference's relative rule (`dense.py:195-221`, |R00| of a
  column-pivoted QR is the largest column norm);
* transfer bases: the far field projected on the children's expanded skeleton
  bases, in column slabs (`compress.py:162-184`), same rank rule;
* couplings: E_i^T K(I, J) E_j in slabs (`compress.py:207-226`);
* dense leaf blocks: evaluated straight into the upload arena.

The kernel matrix is generated on the fly from the point coordinates; all
dense linear algebra is fp64 (cuBLAS / cuSOLVER through torch: this is
shift-independent preprocessing, not the factorization hot path).  The
result is an ordinary RankStructuredMatrix whose payload lives in one device
arena that `h2l_upload` copies device-to-device; `to_host()` exports it to
numpy for the oracle (parity is always checked on the identical H).
"""

import numpy as np

from .errors import ConfigError
from .h2matrix import BasisSplit, RankStructuredMatrix

SLAB = 8192


def _torch():
    import torch

    return torch


# ----------------------------------------------------------------- kernels
def _radial(kind, r, kernel, t):
    if kind == "laplace_offset":
        return 1.0 / (r + 1e-3)
    if kind == "inv_r":
        return 1.0 / r
    if kind == "neg_log":
        return -t.log(r)
    if kind == "yukawa":
        return t.exp(-r) / r
    if kind == "hopping":
        return -t.exp(-r / kernel.a0)
    raise ConfigError(f"kernel kind {kind!r} has no device evaluator")


class DeviceKernel:
    """K(I, J) on the device for contiguous index ranges of an ordered cloud."""

    def __init__(self, kernel, device="cuda"):
        t = _torch()
        self.t = t
        self.kernel = kernel
        self.kind = kernel.kind
        self.dev = t.device(device)
        if self.kind is None:
            A = getattr(kernel, "A", None)
            if A is None:
                raise ConfigError("kernel has neither a device formula nor a dense matrix")
            self.A = t.as_tensor(np.ascontiguousarray(A), dtype=t.float64, device=self.dev)
            self.X = None
        else:
            self.X = t.as_tensor(np.ascontiguousarray(kernel.cloud.coords), dtype=t.float64,
                                 device=self.dev)
        self.diag = getattr(kernel, "diag_value", None)

    def block(self, i0, i1, j0, j1, out=None):
        t = self.t
        if self.X is None:
            blk = self.A[i0:i1, j0:j1]
            if out is not None:
                out.copy_(blk)
                return out
            return blk.clone()
        a = self.X[i0:i1]
        b = self.X[j0:j1]
        d = a[:, None, :] - b[None, :, :]
        r = t.sqrt((d * d).sum(dim=2))
        lo, hi = max(i0, j0), min(i1, j1)
        if self.diag is not None and lo < hi:
            k = t.arange(lo, hi, device=self.dev)
            r[k - i0, k - j0] = 1.0
            f = _radial(self.kind, r, self.kernel, t)
            f[k - i0, k - j0] = self.diag
        else:
            f = _radial(self.kind, r, self.kernel, t)
        if out is not None:
            out.copy_(f)
            return out
        return f

    def rows_at(self, idx, j0, j1):
        """K(idx, j0:j1) for a device index vector idx disjoint from [j0, j1) (no diagonal)."""
        t = self.t
        if self.X is None:
            return self.A[idx, j0:j1]
        d = self.X[idx][:, None, :] - self.X[j0:j1][None, :, :]
        return _radial(self.kind, t.sqrt((d * d).sum(dim=2)), self.kernel, t)

    def block_ranges(self, I, J):
        """K over unions of ranges: I, J lists of (start, stop)."""
        t = self.t
        rows = []
        for (i0, i1) in I:
            rows.append(t.cat([self.block(i0, i1, j0, j1) for (j0, j1) in J], dim=1)
                        if J else t.zeros((i1 - i0, 0), dtype=t.float64, device=self.dev))
        return t.cat(rows, dim=0)


# ----------------------------------------------------------- admissibility
def _admissible_matrix(tree, level, eta):
    """Vectorised `admissible(box_i, box_j, eta)` over all pairs of one level."""
    N = tree.num_clusters(level)
    boxes = tree.boxes[level]
    d = len(next(b for b in boxes if b is not None)[0])
    lo = np.full((N, d), np.nan)
    hi = np.full((N, d), np.nan)
    for i, b in enumerate(boxes):
        if b is not None:
            lo[i], hi[i] = b
    gap = np.maximum(0.0, np.maximum(lo[None, :, :] - hi[:, None, :],
                                     lo[:, None, :] - hi[None, :, :]))
    dist = np.sqrt(np.sum(gap * gap, axis=2))
    diam = np.sqrt(np.sum((hi - lo) ** 2, axis=1))
    dmax = np.maximum(diam[:, None], diam[None, :])
    ok = (dist > 0.0) & (dmax <= eta * dist)
    empty = np.isnan(lo[:, 0])
    ok[empty, :] = False
    ok[:, empty] = False
    np.fill_diagonal(ok, False)
    return ok


def _partners(tree, st, level):
    N = tree.num_clusters(level)
    if st.kind in ("weak", "flat"):
        sizes = np.array([tree.size(level, i) for i in range(N)])
        ok = (sizes[:, None] > 0) & (sizes[None, :] > 0)
        np.fill_diagonal(ok, False)
        return ok
    return _admissible_matrix(tree, level, st.eta)


def _index_vector(ranges, t, dev):
    if not ranges:
        return t.zeros(0, dtype=t.int64, device=dev)
    return t.cat([t.arange(a, b, device=dev) for (a, b) in ranges])


# ------------------------------------------------------------- rank reveal
class _Prof:
    """Phase timer of the construction (H2L_BUILD_PROFILE=1: synchronising, diagnostics only)."""

    def __init__(self, t):
        import os
        import time

        self.on = bool(os.environ.get("H2L_BUILD_PROFILE"))
        self.t, self.time = t, time
        self.acc = {}
        self.last = None

    def __call__(self, what):
        if not self.on:
            return
        self.t.cuda.synchronize()
        now = self.time.perf_counter()
        if self.last is not None:
            self.acc[self.last[0]] = self.acc.get(self.last[0], 0.0) + now - self.last[1]
        self.last = (what, now)


_PROF = None


def _split(M_T, eps, t):
    """Basis split of M (rows x cols) given M^T (cols x rows); reference rank rule."""
    m = M_T.shape[1]
    dev = M_T.device
    if M_T.shape[0] == 0 or not bool((M_T != 0).any()):
        return t.zeros((m, 0), dtype=t.float64, device=dev), t.eye(m, dtype=t.float64, device=dev)
    colmax = float(t.linalg.vector_norm(M_T, dim=1).max())
    if _PROF:
        _PROF("qr")
    if M_T.shape[0] > m:
        R = t.linalg.qr(M_T, mode="r")[1]          # M^T = Q R  ->  M = R^T Q^T
        core = R.T
    else:
        core = M_T.T
    if _PROF:
        _PROF("svd")
    U, S, _ = t.linalg.svd(core, full_matrices=True)
    tail = t.sqrt(t.flip(t.cumsum(t.flip(S * S, [0]), 0), [0]))
    hits = t.nonzero(tail <= eps * colmax)
    rank = int(hits[0]) if hits.numel() else int(S.numel())
    return U[:, :rank].contiguous(), U[:, rank:].contiguous()


# ------------------------------------------------------------ construction
def construct_device(kernel, tree, structure, eps, device="cuda", verbose=False):
    """H2 / HSS / BLR2 construction on the GPU (same algorithm as `construct`).

    Returns a RankStructuredMatrix whose blocks are torch views into a single
    device arena (attached as `H._arena`, `H._arena_offsets`), ready for a
    device-to-device `h2l_upload`."""
    t = _torch()
    if eps <= 0:
        raise ConfigError("eps must be positive")
    st = structure
    fmt = {"flat": "blr2", "strong": "h2"}.get(st.kind) or (
        "hss" if len(st.lowrank_levels()) > 1 else "blr2")
    K = DeviceKernel(kernel, device)
    dev = K.dev
    L = tree.depth
    rng = tree.ranges
    global _PROF
    prof = _PROF = _Prof(t)

    # ---- bases
    bases = {}
    expanded = {}
    if L > 0:
        part = _partners(tree, st, L)
        for i in range(tree.num_clusters(L)):
            i0, i1 = rng[L][i]
            if i1 == i0:
                bases[(L, i)] = (t.zeros((0, 0), dtype=t.float64, device=dev),
                                 t.zeros((0, 0), dtype=t.float64, device=dev))
                expanded[(L, i)] = t.zeros((0, 0), dtype=t.float64, device=dev)
                continue
            prof("leaf_sample")
            J = [rng[L][j] for j in np.nonzero(part[i])[0]]
            jidx = _index_vector(J, t, dev)                        # K(J, I) = K(I, J)^T
            MT = K.rows_at(jidx, i0, i1) if jidx.numel() else t.zeros((0, i1 - i0), dtype=t.float64,
                                                                        device=dev)
            US, UR = _split(MT, eps, t)
            bases[(L, i)] = (US, UR)
            expanded[(L, i)] = US
        if st.kind != "flat":
            for level in range(L - 1, 0, -1):
                part = _partners(tree, st, level)
                for i in range(tree.num_clusters(level)):
                    prof("transfer_sample")
                    c1, c2 = 2 * i, 2 * i + 1
                    e1, e2 = expanded[(level + 1, c1)], expanded[(level + 1, c2)]
                    (a0, a1), (b0, b1) = rng[level + 1][c1], rng[level + 1][c2]
                    r1, r2 = e1.shape[1], e2.shape[1]
                    cols = []
                    # all partners' columns at once, in slabs (K(J, I) with I = the two
                    # children's contiguous rows, split into e1^T / e2^T projections)
                    jidx = _index_vector([rng[level][j] for j in np.nonzero(part[i])[0]], t, dev)
                    for s0 in range(0, jidx.numel(), SLAB):
                        KT = K.rows_at(jidx[s0:s0 + SLAB], a0, b1)      # slab x (m1 + m2)
                        cols.append(t.cat([KT[:, :a1 - a0] @ e1, KT[:, b0 - a0:] @ e2], dim=1))
                    ZT = t.cat(cols, dim=0) if cols else t.zeros((0, r1 + r2), dtype=t.float64,
                                                                   device=dev)
                    if r1 + r2 == 0:
                        US = t.zeros((0, 0), dtype=t.float64, device=dev)
                        UR = t.zeros((0, 0), dtype=t.float64, device=dev)
                    else:
                        US, UR = _split(ZT, eps, t)
                    bases[(level, i)] = (US, UR)
                    prof("transfer_expand")
                    expanded[(level, i)] = t.cat([e1 @ US[:r1], e2 @ US[r1:]], dim=0)

    prof("arena")
    # ---- arena layout (the order of _native.build_plan)
    sizes = []
    nleaf = tree.num_clusters(L)
    for i in range(nleaf):
        m = tree.size(L, i)
        sizes.append(("D", i, m * m))
    for (i, j) in st.dense:
        sizes.append(("O", (i, j), tree.size(L, i) * tree.size(L, j)))
    low = [(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]]
    for key in low:
        l, i, j = key
        sizes.append(("C", key, bases[(l, i)][0].shape[1] * bases[(l, j)][0].shape[1]))
    for key in sorted(bases):
        US, UR = bases[key]
        m = US.shape[0] if US.numel() else UR.shape[0]
        sizes.append(("B", key, m * m))
    total = sum(s[2] for s in sizes)
    arena = t.empty(max(1, total), dtype=t.float64, device=dev)
    offsets = {}
    pos = 0
    for kind, key, sz in sizes:
        offsets[(kind, key)] = pos
        pos += sz

    def view(kind, key, shape):
        o = offsets[(kind, key)]
        return arena[o:o + shape[0] * shape[1]].view(shape)

    leaf_diag, leaf_offdiag, couplings, bsplit = {}, {}, {}, {}
    prof("dense_blocks")
    for i in range(nleaf):
        i0, i1 = rng[L][i]
        v = view("D", i, (i1 - i0, i1 - i0))
        if i1 > i0:
            K.block(i0, i1, i0, i1, out=v)
        leaf_diag[i] = v
    for (i, j) in st.dense:
        (i0, i1), (j0, j1) = rng[L][i], rng[L][j]
        v = view("O", (i, j), (i1 - i0, j1 - j0))
        K.block(i0, i1, j0, j1, out=v)
        leaf_offdiag[(i, j)] = v
    prof("couplings")
    for key in low:
        l, i, j = key
        ei, ej = expanded[(l, i)], expanded[(l, j)]
        (i0, i1), (j0, j1) = rng[l][i], rng[l][j]
        v = view("C", key, (ei.shape[1], ej.shape[1]))
        acc = t.zeros((i1 - i0, ej.shape[1]), dtype=t.float64, device=dev)
        for s0 in range(j0, j1, SLAB):
            s1 = min(j1, s0 + SLAB)
            acc += K.block(i0, i1, s0, s1) @ ej[s0 - j0:s1 - j0]
        v.copy_(ei.T @ acc)
        couplings[key] = v
    prof("bases_out")
    for key in sorted(bases):
        US, UR = bases[key]
        m = US.shape[0] if US.numel() else UR.shape[0]
        v = view("B", key, (m, m))
        if m:
            v.copy_(t.cat([UR, US], dim=1))
        bsplit[key] = DeviceBasis(v, US.shape[1])
        if verbose and key[0] == L and key[1] < 2:
            print(f"basis {key}: m={m} rank={US.shape[1]}", flush=True)
    H = RankStructuredMatrix(fmt=fmt, tree=tree, structure=st, eps=eps, leaf_diag=leaf_diag,
                             leaf_offdiag=leaf_offdiag, bases=bsplit, couplings=couplings)
    H._arena = arena
    H._arena_offsets = offsets
    prof("end")
    H._build_profile = dict(prof.acc)
    _PROF = None
    scale = max((float(b.abs().max()) for b in leaf_diag.values() if b.numel()), default=0.0)
    H._scale0 = scale
    # hand the construction's temporaries back to the device: the engine allocates
    # from its own stream-ordered pools, not from torch's cache
    del bases, expanded
    t.cuda.empty_cache()
    return H


class DeviceBasis(BasisSplit):
    """BasisSplit whose square [U_R | U_S] lives in the device arena."""

    def __init__(self, square, rank):
        self._sq = square
        self._rank = int(rank)

    @property
    def rank(self):
        return self._rank

    @property
    def m(self):
        return int(self._sq.shape[0])

    @property
    def U_S(self):
        return self._sq[:, self.m - self._rank:]

    @property
    def U_R(self):
        return self._sq[:, :self.m - self._rank]

    def square(self):
        return self._sq


def to_host(H):
    """Copy a device-built H into an ordinary numpy RankStructuredMatrix.

    The arena crosses PCIe once; blocks become numpy views of the host copy."""
    arena = getattr(H, "_arena", None)
    offs = getattr(H, "_arena_offsets", None)
    if arena is not None and offs is not None:
        host = arena.detach().cpu().numpy()

        def hv(kind, key, shape):
            o = offs[(kind, key)]
            return host[o:o + shape[0] * shape[1]].reshape(shape)
    else:
        hv = None

    def h(kind, key, v):
        if hv is not None and (kind, key) in offs:
            return hv(kind, key, tuple(v.shape))
        return v.detach().cpu().numpy().copy()

    bases = {}
    for k, b in H.bases.items():
        sq = h("B", k, b.square())
        m, r = sq.shape[0], b.rank
        bases[k] = BasisSplit(U_S=sq[:, m - r:].copy(), U_R=sq[:, :m - r].copy())
    out = RankStructuredMatrix(
        fmt=H.fmt, tree=H.tree, structure=H.structure, eps=H.eps,
        leaf_diag={k: h("D", k, v) for k, v in H.leaf_diag.items()},
        leaf_offdiag={k: h("O", k, v) for k, v in H.leaf_offdiag.items()},
        bases=bases, couplings={k: h("C", k, v) for k, v in H.couplings.items()})
    return out


def gershgorin_device(kernel, rows=1024, pad=1e-6, device="cuda"):
    """Search interval of BASELINE's configs: Gershgorin discs of the kernel matrix.

    Row sums of |A_ij| are evaluated on the device in row slabs (the n x n
    matrix is never stored).  The H2 approximation differs from A by about
    eps * |A|, so both ends are widened by pad * max(|lo|, |hi|)."""
    t = _torch()
    K = DeviceKernel(kernel, device)
    n = kernel.cloud.n if kernel.kind is not None else K.A.shape[0]
    lo, hi = np.inf, -np.inf
    for i0 in range(0, n, rows):
        i1 = min(n, i0 + rows)
        rad = t.zeros(i1 - i0, dtype=t.float64, device=K.dev)
        for j0 in range(0, n, SLAB):
            j1 = min(n, j0 + SLAB)
            rad += K.block(i0, i1, j0, j1).abs().sum(dim=1)
        d = t.diagonal(K.block(i0, i1, i0, i1))
        rad -= d.abs()
        lo = min(lo, float((d - rad).min()))
        hi = max(hi, float((d + rad).max()))
    w = pad * max(abs(lo), abs(hi), 1.0)
    return lo - w, hi + w


def config_device(name, seed=0, n=None, leaf=None, device="cuda", verbose=False):
    """(H on device, cloud) for a BASELINE config or a same-recipe mini-config."""
    from . import configs

    cfg = configs.CONFIGS[name]
    cloud, kern, tree, st = configs.config_problem(name, seed=seed, n=n, leaf=leaf)
    H = construct_device(kern, tree, st, cfg.eps, device=device, verbose=verbose)
    H._kernel = kern
    return H, cloud


def reconstruct_dense_device(H, device="cuda"):
    """Dense realisation of an unshifted device-built H on the GPU (validation only:
    the reference's `reconstruct_dense`, compress.py / h2matrix.reconstruct_dense, for
    sizes whose n x n fp64 matrix fits in HBM -- config 2 is 34 GB)."""
    t = _torch()
    tree = H.tree
    L = tree.depth
    n = H.n
    dev = t.device(device)
    A = t.zeros((n, n), dtype=t.float64, device=dev)

    def dv(x):
        return x if isinstance(x, t.Tensor) else t.as_tensor(np.asarray(x), dtype=t.float64,
                                                              device=dev)

    for i, blk in H.leaf_diag.items():
        lo, hi = tree.index_range(L, i)
        A[lo:hi, lo:hi] = dv(blk)
    for (i, j), blk in H.leaf_offdiag.items():
        (a0, a1), (b0, b1) = tree.index_range(L, i), tree.index_range(L, j)
        b = dv(blk)
        A[a0:a1, b0:b1] = b
        A[b0:b1, a0:a1] = b.T
    memo = {}

    def expanded(level, i):
        key = (level, i)
        if key not in memo:
            bs = H.bases[key]
            if tree.is_leaf_level(level):
                memo[key] = dv(bs.U_S)
            else:
                (lc, c1), (_, c2) = tree.children(level, i)
                e1, e2 = expanded(lc, c1), expanded(lc, c2)
                r1 = e1.shape[1]
                us = dv(bs.U_S)
                memo[key] = t.cat([e1 @ us[:r1], e2 @ us[r1:]], dim=0)
        return memo[key]

    for (level, i, j), S in sorted(H.couplings.items(), key=lambda kv: -kv[0][0]):
        ei, ej = expanded(level, i), expanded(level, j)
        (a0, a1), (b0, b1) = tree.index_range(level, i), tree.index_range(level, j)
        blk = ei @ dv(S) @ ej.T
        A[a0:a1, b0:b1] = blk
        A[b0:b1, a0:a1] = blk.T
        del blk
    memo.clear()
    return A
