"""Rank-structured (BLR2 / HSS / H2) symmetric matrices: container and build.

The container mirrors the reference's `RankStructuredMatrix`
(`h2slice/compress.py:24-143`): dense leaf diagonal blocks, dense inadmissible
leaf off-diagonal blocks (strong admissibility), nested bases per (level, i)
stored as orthogonal splits `[U_R | U_S]`, and skeleton couplings per
(level, i, j).  `shift_diagonal` records a diagonal shift without touching the
shared payload, which is what the CUDA engine consumes: the payload is uploaded
once per unshifted origin and every shift is applied on the device.

`construct` is the reference's dense-sampling construction
(`compress.py:146-279`): leaf bases by truncated column-pivoted QR of the
concatenated far-field rows, transfer bases by projecting the far field onto
the children's expanded skeletons, couplings by two-sided projection.  It is
host-side numpy and O(n^2); it is not part of the factorization hot path
(SURVEY.md §8f lists GPU construction as the next row).
"""

from dataclasses import dataclass, field
import os

import numpy as np
import scipy.linalg

from .cluster import construction_partners
from .errors import ConfigError, OracleTooLarge

COLUMN_SLAB = 1024
ORACLE_CAP_ENV = "H2SPEC_ORACLE_CAP"
_DEFAULT_ORACLE_CAP = 4096


def oracle_cap():
    raw = os.environ.get(ORACLE_CAP_ENV)
    return int(raw) if raw else _DEFAULT_ORACLE_CAP


@dataclass
class BasisSplit:
    """Orthogonal split of R^m into skeleton U_S (kept) and redundant U_R."""

    U_S: np.ndarray
    U_R: np.ndarray

    @property
    def rank(self):
        return int(self.U_S.shape[1])

    @property
    def m(self):
        return int(self.U_S.shape[0])

    def square(self):
        """[U_R | U_S]: redundant directions first (reference `dense.py:190-192`)."""
        return np.hstack([self.U_R, self.U_S])


def rrqr_truncated(M, eps):
    """Column-pivoted QR split with relative Frobenius-tail truncation.

    rank = first r with ||R[r:, :]||_F <= eps * |R[0, 0]| (else min(M.shape)),
    the rule of the reference `dense.py:195-221`.
    """
    M = np.asarray(M, dtype=np.float64)
    m = M.shape[0]
    if M.size == 0 or not M.any():
        return BasisSplit(U_S=np.zeros((m, 0)), U_R=np.eye(m))
    Q, R, _ = scipy.linalg.qr(M, mode="full", pivoting=True)
    k = min(M.shape)
    mass = np.sum(R[:k, :] ** 2, axis=1)
    tail = np.sqrt(np.maximum(0.0, np.cumsum(mass[::-1])[::-1]))
    bound = eps * abs(R[0, 0])
    hits = np.nonzero(tail <= bound)[0]
    rank = int(hits[0]) if hits.size else k
    return BasisSplit(U_S=Q[:, :rank].copy(), U_R=Q[:, rank:].copy())


@dataclass
class RankStructuredMatrix:
    """Symmetric matrix in BLR2 / HSS / H2 form over a cluster tree."""

    fmt: str
    tree: object
    structure: object
    eps: float
    leaf_diag: dict
    leaf_offdiag: dict = field(default_factory=dict)
    bases: dict = field(default_factory=dict)
    couplings: dict = field(default_factory=dict)
    shift: float = 0.0
    _origin: object = None
    _scale0: float = -1.0
    _device: dict = field(default_factory=dict)  # per-device native uploads (origin only)

    @property
    def n(self):
        return self.tree.n

    def origin(self):
        return self._origin if self._origin is not None else self

    def max_rank(self):
        return max((bs.rank for bs in self.bases.values()), default=0)

    def storage_bytes(self):
        tot = sum(a.nbytes for a in self.leaf_diag.values())
        tot += sum(a.nbytes for a in self.leaf_offdiag.values())
        tot += sum(b.U_S.nbytes + b.U_R.nbytes for b in self.bases.values())
        tot += sum(a.nbytes for a in self.couplings.values())
        return tot

    def scale0(self):
        """max |entry| over the origin's leaf diagonal blocks (`compress.py:71-82`)."""
        org = self.origin()
        if org._scale0 < 0.0:
            vals = [float(np.abs(b).max()) for b in org.leaf_diag.values() if b.size]
            org._scale0 = max(vals) if vals else 0.0
        return org._scale0

    def scale_estimate(self):
        org = self.origin()
        return self.scale0() + abs(self.shift - org.shift)

    def copy(self):
        """Independent replica of the numeric payload (shares tree and bases)."""
        return RankStructuredMatrix(
            fmt=self.fmt, tree=self.tree, structure=self.structure, eps=self.eps,
            leaf_diag={k: v.copy() for k, v in self.leaf_diag.items()},
            leaf_offdiag={k: v.copy() for k, v in self.leaf_offdiag.items()},
            bases=dict(self.bases), couplings=dict(self.couplings), shift=self.shift)


def shift_diagonal(H, mu):
    """H - mu*I.  Shares the origin's payload; the shift is applied on device.

    The reference materialises shifted leaf diagonal blocks
    (`compress.py:130-143`) that its engine never reads; here the shifted
    object only records `shift` and links the origin.
    """
    org = H.origin()
    return RankStructuredMatrix(
        fmt=H.fmt, tree=H.tree, structure=H.structure, eps=H.eps,
        leaf_diag=org.leaf_diag, leaf_offdiag=org.leaf_offdiag, bases=org.bases,
        couplings=org.couplings, shift=H.shift + mu, _origin=org)


# ---------------------------------------------------------------- construction
def _far_rows(kernel, tree, st, i):
    L = tree.depth
    I = tree.indices(L, i)
    blocks = [kernel.block(I, tree.indices(L, j)) for j in construction_partners(tree, st, L, i)]
    return np.hstack(blocks) if blocks else np.zeros((len(I), 0))


def _transfer_split(kernel, tree, st, level, i, eps, expanded):
    (lc, c1), (_, c2) = tree.children(level, i)
    e1, e2 = expanded[(lc, c1)], expanded[(lc, c2)]
    I1, I2 = tree.indices(lc, c1), tree.indices(lc, c2)
    slabs = []
    for j in construction_partners(tree, st, level, i):
        J = tree.indices(level, j)
        for s0 in range(0, len(J), COLUMN_SLAB):
            Js = J[s0:s0 + COLUMN_SLAB]
            slabs.append(np.vstack([e1.T @ kernel.block(I1, Js), e2.T @ kernel.block(I2, Js)]))
    Z = np.hstack(slabs) if slabs else np.zeros((e1.shape[1] + e2.shape[1], 0))
    return rrqr_truncated(Z, eps)


def expanded_basis(tree, bases, level, i, memo):
    """Leaf-coordinate skeleton basis of (level, i) through the transfer chain."""
    key = (level, i)
    if key not in memo:
        bs = bases[key]
        if tree.is_leaf_level(level):
            memo[key] = bs.U_S
        else:
            (lc, c1), (_, c2) = tree.children(level, i)
            e1 = expanded_basis(tree, bases, lc, c1, memo)
            e2 = expanded_basis(tree, bases, lc, c2, memo)
            r1 = e1.shape[1]
            memo[key] = np.vstack([e1 @ bs.U_S[:r1], e2 @ bs.U_S[r1:]])
    return memo[key]


def _coupling(kernel, tree, level, i, j, ei, ej):
    I, J = tree.indices(level, i), tree.indices(level, j)
    acc = np.zeros((len(I), ej.shape[1]))
    for s0 in range(0, len(J), COLUMN_SLAB):
        acc += kernel.block(I, J[s0:s0 + COLUMN_SLAB]) @ ej[s0:s0 + COLUMN_SLAB]
    return ei.T @ acc


def construct(kernel, tree, structure, eps):
    """Dense-sampling H2 / HSS / BLR2 construction at relative tolerance eps."""
    if eps <= 0:
        raise ConfigError("eps must be positive")
    if structure.kind == "flat":
        fmt = "blr2"
    elif structure.kind == "weak":
        fmt = "hss" if len(structure.lowrank_levels()) > 1 else "blr2"
    else:
        fmt = "h2"
    L = tree.depth
    leaf_diag = {}
    for i in range(tree.num_clusters(L)):
        I = tree.indices(L, i)
        leaf_diag[i] = kernel.block(I, I) if len(I) else np.zeros((0, 0))
    leaf_offdiag = {(i, j): kernel.block(tree.indices(L, i), tree.indices(L, j))
                    for i, j in structure.dense}
    bases = {}
    if L > 0:
        for i in range(tree.num_clusters(L)):
            bases[(L, i)] = rrqr_truncated(_far_rows(kernel, tree, structure, i), eps)
        if structure.kind != "flat":
            expanded = {(L, i): bases[(L, i)].U_S for i in range(tree.num_clusters(L))}
            memo = {}
            for level in range(L - 1, 0, -1):
                for i in range(tree.num_clusters(level)):
                    bases[(level, i)] = _transfer_split(kernel, tree, structure, level, i, eps,
                                                        expanded)
                    expanded[(level, i)] = expanded_basis(tree, bases, level, i, memo)
    couplings = {}
    memo = {}
    for level in structure.lowrank_levels():
        for i, j in structure.lowrank_at(level):
            ei = expanded_basis(tree, bases, level, i, memo)
            ej = expanded_basis(tree, bases, level, j, memo)
            couplings[(level, i, j)] = _coupling(kernel, tree, level, i, j, ei, ej)
    return RankStructuredMatrix(fmt=fmt, tree=tree, structure=structure, eps=eps,
                                leaf_diag=leaf_diag, leaf_offdiag=leaf_offdiag, bases=bases,
                                couplings=couplings)


def reconstruct_dense(H, cap=None):
    """Dense realisation including the shift (validation path, n <= cap)."""
    n = H.n
    cap = oracle_cap() if cap is None else cap
    if n > cap:
        raise OracleTooLarge(n, cap)
    tree = H.tree
    org = H.origin()
    L = tree.depth
    A = np.zeros((n, n))
    for i, blk in org.leaf_diag.items():
        lo, hi = tree.index_range(L, i)
        A[lo:hi, lo:hi] = blk
    for (i, j), blk in org.leaf_offdiag.items():
        (a0, a1), (b0, b1) = tree.index_range(L, i), tree.index_range(L, j)
        A[a0:a1, b0:b1] = blk
        A[b0:b1, a0:a1] = blk.T
    memo = {}
    for (level, i, j), S in org.couplings.items():
        ei = expanded_basis(tree, org.bases, level, i, memo)
        ej = expanded_basis(tree, org.bases, level, j, memo)
        (a0, a1), (b0, b1) = tree.index_range(level, i), tree.index_range(level, j)
        blk = ei @ S @ ej.T
        A[a0:a1, b0:b1] = blk
        A[b0:b1, a0:a1] = blk.T
    delta = H.shift - org.shift
    if delta:
        A[np.diag_indices(n)] -= delta
    return A


def gershgorin_interval(A):
    """[min(d - radius), max(d + radius)] from absolute row sums."""
    A = np.asarray(A, dtype=np.float64)
    d = np.diagonal(A)
    rad = np.abs(A).sum(axis=1) - np.abs(d)
    return float((d - rad).min()), float((d + rad).max())


def payload_digest(H):
    """sha256 over the origin payload in a canonical order (bitwise identity of two H).

    Works on this package's matrices and on the reference's `RankStructuredMatrix`
    (same field names), so a fixture can pin a rebuilt H to the reference-built one."""
    import hashlib

    org = H.origin() if hasattr(H, "origin") else H
    h = hashlib.sha256()

    def put(tag, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        h.update(f"{tag}{a.shape}".encode())
        h.update(a.tobytes())

    for i in sorted(org.leaf_diag):
        put(("D", i), org.leaf_diag[i])
    for k in sorted(org.leaf_offdiag):
        put(("O",) + tuple(k), org.leaf_offdiag[k])
    for k in sorted(org.bases):
        bs = org.bases[k]
        put(("R",) + tuple(k), bs.U_R)
        put(("S",) + tuple(k), bs.U_S)
    for k in sorted(org.couplings):
        put(("C",) + tuple(k), org.couplings[k])
    return h.hexdigest()


# ------------------------------------------------------------- payload file IO
def save_payload(path, H, compress=True):
    """Serialise the origin payload of H (tree ranges, structure, blocks) to .npz."""
    org = H.origin()
    tree, st = org.tree, org.structure
    out = {
        "meta": np.array([tree.n, tree.leaf_size, tree.depth], dtype=np.int64),
        "fmt": np.array(org.fmt), "kind": np.array(st.kind),
        "eta_eps": np.array([st.eta, org.eps], dtype=np.float64),
        "ranges": np.array([r for lv in tree.ranges for r in lv], dtype=np.int64),
        "dense": np.array(st.dense, dtype=np.int64).reshape(-1, 2),
        "lowrank": np.array([(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]],
                            dtype=np.int64).reshape(-1, 3),
        "deferred": np.array([(l, i, j) for l in sorted(st.deferred) for i, j in st.deferred[l]],
                             dtype=np.int64).reshape(-1, 3),
    }
    for i, blk in org.leaf_diag.items():
        out[f"D_{i}"] = blk
    for (i, j), blk in org.leaf_offdiag.items():
        out[f"O_{i}_{j}"] = blk
    for (l, i), bs in org.bases.items():
        out[f"B_{l}_{i}"] = bs.square()
        out[f"r_{l}_{i}"] = np.array(bs.rank)
    for (l, i, j), blk in org.couplings.items():
        out[f"C_{l}_{i}_{j}"] = blk
    (np.savez_compressed if compress else np.savez)(path, **out)


def load_payload(path):
    """Inverse of `save_payload` (boxes are not stored: the engine never needs them)."""
    from .cluster import BlockStructure, ClusterTree

    z = np.load(path, allow_pickle=False)
    n, leaf, depth = (int(v) for v in z["meta"])
    flat = [tuple(int(x) for x in r) for r in z["ranges"]]
    ranges, pos = [], 0
    for level in range(depth + 1):
        ranges.append(flat[pos:pos + (1 << level)])
        pos += 1 << level
    tree = ClusterTree(n=n, leaf_size=leaf, depth=depth, degenerate=depth == 0, ranges=ranges,
                       boxes=[[None] * len(lv) for lv in ranges])
    eta, eps = (float(v) for v in z["eta_eps"])
    st = BlockStructure(kind=str(z["kind"]), eta=eta)
    st.dense = [(int(i), int(j)) for i, j in z["dense"]]
    for l, i, j in z["lowrank"]:
        st.lowrank.setdefault(int(l), []).append((int(i), int(j)))
    for l, i, j in z["deferred"]:
        st.deferred.setdefault(int(l), []).append((int(i), int(j)))
    leaf_diag, offd, bases, coup = {}, {}, {}, {}
    for key in z.files:
        parts = key.split("_")
        if parts[0] == "D":
            leaf_diag[int(parts[1])] = z[key]
        elif parts[0] == "O":
            offd[(int(parts[1]), int(parts[2]))] = z[key]
        elif parts[0] == "B":
            l, i = int(parts[1]), int(parts[2])
            Q = z[key]
            r = int(z[f"r_{l}_{i}"])
            m = Q.shape[0]
            bases[(l, i)] = BasisSplit(U_S=Q[:, m - r:].copy(), U_R=Q[:, :m - r].copy())
        elif parts[0] == "C":
            coup[(int(parts[1]), int(parts[2]), int(parts[3]))] = z[key]
    leaf_diag = dict(sorted(leaf_diag.items()))
    return RankStructuredMatrix(fmt=str(z["fmt"]), tree=tree, structure=st, eps=eps,
                                leaf_diag=leaf_diag, leaf_offdiag=offd, bases=bases,
                                couplings=coup)
