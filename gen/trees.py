"""PlenOctree array construction (input format only; no rendering arithmetic).

Encoding (reading Q1/Q2):

* ``child[n_nodes][8]`` uint32, entry = ``tag << 30 | index``;
  tag 0 = empty, 1 = internal node index, 2 = leaf index.  Node 0 is the root.
* octant = 4*bx + 2*by + bz, bx = 1 for the upper half in x (C order [x][y][z]).
* leaves are numbered in depth-first (Morton) order, so every subtree owns a
  contiguous leaf-index range; internal nodes are numbered in pre-order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TAG_EMPTY, TAG_INTERNAL, TAG_LEAF = 0, 1, 2
IDX_MASK = (1 << 30) - 1


@dataclass
class Tree:
    """Host-side PlenOctree in the C-ABI layout (include/plenoct.h, po_tree_create)."""
    depth: int                      # D: leaf grid is 2^D per axis
    bbox_min: np.ndarray            # float32[3]
    edge: float                     # cube edge (world units)
    sh_degree: int                  # l_max; B = (l_max+1)^2
    child: np.ndarray               # uint32[n_nodes][8]
    sigma: np.ndarray               # float32[n_leaves]  (sigma-tilde, pre-ReLU)
    sh: np.ndarray                  # float32[n_leaves][B][3]
    leaf_level: np.ndarray = field(default=None)   # int32[n_leaves] depth of each leaf
    leaf_cell: np.ndarray = field(default=None)    # int64[n_leaves][3] cell coords at leaf_level

    @property
    def n_nodes(self) -> int:
        return int(self.child.shape[0])

    @property
    def n_leaves(self) -> int:
        return int(self.sigma.shape[0])

    @property
    def basis_dim(self) -> int:
        return (self.sh_degree + 1) ** 2


def _part1by2(v: np.ndarray) -> np.ndarray:
    """Spread the low 21 bits of v so that bit i moves to bit 3i."""
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton(cells: np.ndarray) -> np.ndarray:
    """Morton code with x as the most significant bit of each 3-bit group (octant = 4x+2y+z)."""
    cells = np.asarray(cells, dtype=np.int64)
    return (_part1by2(cells[:, 0]) << np.uint64(2)) | (_part1by2(cells[:, 1]) << np.uint64(1)) | _part1by2(cells[:, 2])


def build_from_leaf_cells(cells: np.ndarray, depth: int):
    """Build the child table for a set of leaf cells that all sit at ``depth``.

    Returns ``(child, order)``: ``order`` permutes the input cells into leaf-index
    (depth-first) order.  Internal nodes are exactly the ancestors of the leaves.
    """
    cells = np.asarray(cells, dtype=np.int64)
    n = cells.shape[0]
    if n == 0:
        return np.zeros((1, 8), dtype=np.uint32), np.zeros(0, dtype=np.int64)
    code = morton(cells)
    order = np.argsort(code, kind="stable")
    code = code[order]
    if np.any(code[1:] == code[:-1]):
        raise ValueError("duplicate leaf cells")
    D = depth
    # internal node prefixes per level L = 0..D-1
    prefixes = [np.unique(code >> np.uint64(3 * (D - L))) for L in range(D)]
    # pre-order numbering: sort by (first descendant code, level)
    keys = np.concatenate([p << np.uint64(3 * (D - L)) for L, p in enumerate(prefixes)])
    levels = np.concatenate([np.full(p.shape[0], L, dtype=np.int64) for L, p in enumerate(prefixes)])
    pre = np.lexsort((levels, keys))
    node_id = np.empty(pre.shape[0], dtype=np.int64)
    node_id[pre] = np.arange(pre.shape[0])
    offs = np.cumsum([0] + [p.shape[0] for p in prefixes])
    n_nodes = int(offs[-1])
    child = np.zeros((n_nodes, 8), dtype=np.uint32)
    for L in range(D):
        parents = prefixes[L]
        pid = node_id[offs[L]:offs[L + 1]]
        for o in range(8):
            want = parents * np.uint64(8) + np.uint64(o)
            if L + 1 < D:
                tab = prefixes[L + 1]
                cid_base = node_id[offs[L + 1]:offs[L + 2]]
                tag = TAG_INTERNAL
            else:
                tab = code
                cid_base = np.arange(n, dtype=np.int64)
                tag = TAG_LEAF
            pos = np.searchsorted(tab, want)
            pos_c = np.minimum(pos, tab.shape[0] - 1)
            hit = tab[pos_c] == want
            vals = (np.uint64(tag) << np.uint64(30)) | cid_base[pos_c].astype(np.uint64)
            child[pid[hit], o] = vals[hit].astype(np.uint32)
    return child, order


def uniform_tree(depth: int):
    """All 8^depth cells of a full octree are leaves. Returns (child, cells in leaf order)."""
    r = np.arange(1 << depth, dtype=np.int64)
    cells = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    child, order = build_from_leaf_cells(cells, depth)
    return child, cells[order]


def random_tree(rng: np.random.Generator, depth: int, p_split: float = 0.55, p_leaf: float = 0.6):
    """Random mixed-depth octree for tiny parity cases.

    Every slot of a node at level L < depth is split into an internal node with
    probability p_split (if L+1 < depth), else it is a leaf with probability
    p_leaf, else empty.  Returns (child, leaf_level, leaf_cell) in leaf order
    (depth-first, octant order).
    """
    child_rows = []
    leaf_level, leaf_cell = [], []

    def make(level, cell):
        nid = len(child_rows)
        child_rows.append([0] * 8)
        for o in range(8):
            c = (cell[0] * 2 + (o >> 2), cell[1] * 2 + ((o >> 1) & 1), cell[2] * 2 + (o & 1))
            u = rng.random()
            if level + 1 < depth and u < p_split:
                cid = make(level + 1, c)
                child_rows[nid][o] = (TAG_INTERNAL << 30) | cid
            elif rng.random() < p_leaf:
                lid = len(leaf_level)
                leaf_level.append(level + 1)
                leaf_cell.append(c)
                child_rows[nid][o] = (TAG_LEAF << 30) | lid
        return nid

    make(0, (0, 0, 0))
    child = np.array(child_rows, dtype=np.uint32).reshape(-1, 8)
    return child, np.array(leaf_level, dtype=np.int32), np.array(leaf_cell, dtype=np.int64).reshape(-1, 3)


def tree_leaf_boxes(child: np.ndarray, depth: int):
    """Walk the child table; return per-leaf (level, cell) arrays (for host-side checks)."""
    n_leaves = 0
    for row in child:
        n_leaves += int(np.sum((row >> 30) == TAG_LEAF))
    lev = np.full(n_leaves, -1, dtype=np.int32)
    cel = np.zeros((n_leaves, 3), dtype=np.int64)
    stack = [(0, 0, (0, 0, 0))]
    while stack:
        nid, L, c = stack.pop()
        for o in range(8):
            e = int(child[nid, o])
            tag, idx = e >> 30, e & IDX_MASK
            cc = (c[0] * 2 + (o >> 2), c[1] * 2 + ((o >> 1) & 1), c[2] * 2 + (o & 1))
            if tag == TAG_INTERNAL:
                stack.append((idx, L + 1, cc))
            elif tag == TAG_LEAF:
                lev[idx] = L + 1
                cel[idx] = cc
    return lev, cel
