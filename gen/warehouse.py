"""Synthetic warehouse graphs, SKU placements and Zipf order streams.

The paper never defines its aisle/location graph (§4.7 only gives
V=9,716 / E=26,999 for one test graph; §3 labels stops on a
flattened 10x10 grid). The generators below are the documented design choice
of SURVEY.md §8(d) "Synthetic inputs" (reading A1 in DESIGN.md):

* ``aisle(A, L, C, ...)`` - block-stacking aisle grid with cross-aisles.
* ``lattice(nx, ny, nz, ...)`` - the paper's §5 geometry 100x100x10
  (§5), 8-neighbour in-plane + vertical arcs.
* ``place_skus`` - 89 % fill (§4, §5), clustered
  (popular SKUs near the depot, the ABC rationale of PAPER.md:77-80) or a
  seeded shuffle.
* ``zipf_orders`` - order lines ~ Zipf(s) over SKU popularity ranks, distinct
  SKUs within an order, picks per order uniform in [lo, hi].

Nothing here computes a distance, a route or a cluster: the clustered
placement key is the plain coordinate offset from the depot, not a graph
distance.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

I32 = "i32"
F32 = "f32"


@dataclass
class Graph:
    name: str
    V: int
    src: np.ndarray          # int32 [E] arc tails, file (COO) order
    dst: np.ndarray          # int32 [E] arc heads
    w: np.ndarray            # int32 or float32 [E]
    wtype: str               # "i32" | "f32"
    xy: np.ndarray           # int32 [V, 2] integer planar coordinates
    z: np.ndarray            # int32 [V] level (0 for aisle graphs)
    locations: np.ndarray    # int32 node ids that can hold a SKU
    depot_xyz: tuple = (0, 0, 0)

    @property
    def E(self) -> int:
        return int(self.src.shape[0])


@dataclass
class Orders:
    order_ptr: np.ndarray    # int64 [B+1]
    order_nodes: np.ndarray  # int32 [L] location node of each order line
    order_skus: np.ndarray = field(default=None)  # int32 [L] SKU rank of each line

    @property
    def B(self) -> int:
        return int(self.order_ptr.shape[0] - 1)


def _arcs_from_edges(eu, ev, ew):
    """Undirected edge list -> interleaved arcs (u->v, v->u) sharing a weight."""
    eu = np.asarray(eu, dtype=np.int64)
    ev = np.asarray(ev, dtype=np.int64)
    src = np.empty(2 * eu.size, dtype=np.int32)
    dst = np.empty(2 * eu.size, dtype=np.int32)
    src[0::2], dst[0::2] = eu, ev
    src[1::2], dst[1::2] = ev, eu
    w = np.repeat(np.asarray(ew), 2)
    return src, dst, w


def _weights(kind_idx, base_i32, base_f32, wtype, jitter_seed):
    """Per-undirected-edge weights: int base, or fp32 base x U[0.95,1.05)."""
    kind_idx = np.asarray(kind_idx, dtype=np.int64)
    if wtype == I32:
        return np.asarray(base_i32, dtype=np.int32)[kind_idx]
    if wtype != F32:
        raise ValueError(wtype)
    rng = np.random.default_rng(jitter_seed)
    jit = rng.uniform(0.95, 1.05, size=kind_idx.size)
    w = (np.asarray(base_f32, dtype=np.float64)[kind_idx] * jit).astype(np.float32)
    return w


def aisle(A: int, L: int, C: int, ws=1, wa=3, wd=2, wtype: str = I32,
          jitter_seed: int = 0, fws=0.9, fwa=2.7, fwd=5.0) -> Graph:
    """Aisle grid: A aisles x L slots, C cross-aisles (front, back, interior).

    Node ids: slot(a, l) = a*L + l; cross(c, a) = A*L + c*A + a; depot last.
    Block b of an aisle holds slots [b*L//(C-1), (b+1)*L//(C-1)). Undirected
    edges: cross(b,a)-first slot, consecutive slots, last slot-cross(b+1,a)
    (weight ws); cross(c,a)-cross(c,a+1) (wa); depot-cross(0,0) (wd).
    """
    if A < 1 or C < 2 or L < C - 1:
        raise ValueError("aisle needs A>=1, C>=2, L>=C-1")
    slot = lambda a, l: a * L + l  # noqa: E731
    cross = lambda c, a: A * L + c * A + a  # noqa: E731
    depot = A * L + C * A
    V = depot + 1
    eu, ev, kind = [], [], []
    for a in range(A):
        for b in range(C - 1):
            lo, hi = (b * L) // (C - 1), ((b + 1) * L) // (C - 1)
            eu.append(cross(b, a)); ev.append(slot(a, lo)); kind.append(0)
            for l in range(lo, hi - 1):
                eu.append(slot(a, l)); ev.append(slot(a, l + 1)); kind.append(0)
            eu.append(slot(a, hi - 1)); ev.append(cross(b + 1, a)); kind.append(0)
    for c in range(C):
        for a in range(A - 1):
            eu.append(cross(c, a)); ev.append(cross(c, a + 1)); kind.append(1)
    eu.append(depot); ev.append(cross(0, 0)); kind.append(2)
    w = _weights(kind, [ws, wa, wd], [fws, fwa, fwd], wtype, jitter_seed)
    src, dst, warc = _arcs_from_edges(eu, ev, w)
    xy = np.zeros((V, 2), dtype=np.int32)
    for a in range(A):
        for b in range(C - 1):
            lo, hi = (b * L) // (C - 1), ((b + 1) * L) // (C - 1)
            for l in range(lo, hi):
                xy[slot(a, l)] = (2 * a, l + b + 1)
        for c in range(C):
            xy[cross(c, a)] = (2 * a, (c * L) // (C - 1) + c)
    xy[depot] = (0, -1)
    return Graph(name=f"aisle({A},{L},{C})", V=V, src=src, dst=dst, w=warc,
                 wtype=wtype, xy=xy, z=np.zeros(V, dtype=np.int32),
                 locations=np.arange(A * L, dtype=np.int32), depot_xyz=(0, -1, 0))


def lattice(nx: int = 100, ny: int = 100, nz: int = 10, wtype: str = I32,
            jitter_seed: int = 0) -> Graph:
    """3-D rack lattice (§5 geometry): id = ((j*nx)+i)*nz + k.

    In-plane 8-neighbour arcs at every level (orthogonal 10 / diagonal 14,
    fp32 1.0 / 1.41421354), vertical +-1 arcs (5, fp32 0.35).
    """
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    nid = lambda i, j, k: ((j * nx) + i) * nz + k  # noqa: E731
    parts_u, parts_v, parts_k = [], [], []

    def add(mask, di, dj, dk, kind):
        i, j, k = I[mask], J[mask], K[mask]
        parts_u.append(nid(i, j, k).ravel())
        parts_v.append(nid(i + di, j + dj, k + dk).ravel())
        parts_k.append(np.full(i.size, kind, dtype=np.int64))

    add(I < nx - 1, 1, 0, 0, 0)                        # orthogonal +i
    add(J < ny - 1, 0, 1, 0, 0)                        # orthogonal +j
    add((I < nx - 1) & (J < ny - 1), 1, 1, 0, 1)       # diagonal (+i,+j)
    add((I > 0) & (J < ny - 1), -1, 1, 0, 1)           # diagonal (-i,+j)
    add(K < nz - 1, 0, 0, 1, 2)                        # vertical
    eu = np.concatenate(parts_u)
    ev = np.concatenate(parts_v)
    kind = np.concatenate(parts_k)
    order = np.lexsort((ev, eu))                       # edges sorted by (u, v)
    eu, ev, kind = eu[order], ev[order], kind[order]
    w = _weights(kind, [10, 14, 5], [1.0, 1.41421354, 0.35], wtype, jitter_seed)
    src, dst, warc = _arcs_from_edges(eu, ev, w)
    V = nx * ny * nz
    ids = np.arange(V)
    k = ids % nz
    i = (ids // nz) % nx
    j = ids // (nz * nx)
    xy = np.stack([i, j], axis=1).astype(np.int32)
    return Graph(name=f"lattice({nx},{ny},{nz})", V=V, src=src, dst=dst, w=warc,
                 wtype=wtype, xy=xy, z=k.astype(np.int32),
                 locations=np.arange(V, dtype=np.int32), depot_xyz=(0, 0, 0))


def place_skus(g: Graph, clustered: bool, seed: int, fill_pct: int = 89) -> np.ndarray:
    """SKU popularity rank r -> location node. 89 % fill.

    clustered: ranks go to locations sorted by (|x-xd|+|y-yd|+z, node id), the
    coordinate offset from the depot (ABC/class-based storage);
    unclustered: a seeded shuffle of the locations.
    """
    locs = g.locations
    n_sku = (fill_pct * locs.size) // 100
    if clustered:
        xd, yd, zd = g.depot_xyz
        key = (np.abs(g.xy[locs, 0] - xd) + np.abs(g.xy[locs, 1] - yd)
               + np.abs(g.z[locs] - zd))
        order = np.lexsort((locs, key))
        return locs[order[:n_sku]].astype(np.int32)
    rng = np.random.default_rng(seed)
    return locs[rng.permutation(locs.size)[:n_sku]].astype(np.int32)


def zipf_orders(sku_node: np.ndarray, B: int, n_lo: int, n_hi: int, s: float,
                seed: int) -> Orders:
    """B orders; picks ~ U{n_lo..n_hi}; lines ~ Zipf(s) over SKU ranks (s=0:
    uniform); duplicates within an order are redrawn until all distinct."""
    n_sku = sku_node.size
    if n_hi > n_sku:
        raise ValueError("more picks than SKUs")
    rng = np.random.default_rng(seed)
    picks = rng.integers(n_lo, n_hi + 1, size=B)
    ptr = np.zeros(B + 1, dtype=np.int64)
    np.cumsum(picks, out=ptr[1:])
    total = int(ptr[-1])
    p = 1.0 / np.power(np.arange(1, n_sku + 1, dtype=np.float64), s)
    p /= p.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0

    def draw(k):
        return np.searchsorted(cdf, rng.random(k), side="right").astype(np.int64)

    lines = draw(total)
    owner = np.repeat(np.arange(B, dtype=np.int64), picks)
    while True:
        o = np.lexsort((np.arange(total), lines, owner))
        dup = np.zeros(total, dtype=bool)
        same = (owner[o][1:] == owner[o][:-1]) & (lines[o][1:] == lines[o][:-1])
        dup[o[1:][same]] = True
        idx = np.nonzero(dup)[0]
        if idx.size == 0:
            break
        lines[idx] = draw(idx.size)
    skus = lines.astype(np.int32)
    return Orders(order_ptr=ptr, order_nodes=sku_node[skus].astype(np.int32),
                  order_skus=skus)


# --------------------------------------------------------------------------
# The five configurations of BASELINE.json "configs".
# config k: placement seed k, order seed 100+k, fp32 jitter seed 1000+k.
# --------------------------------------------------------------------------
CONFIGS = {
    1: dict(graph=("aisle", (4, 10, 4)), B=1, picks=(5, 5), s=0.0, clustered=False, m=1),
    2: dict(graph=("aisle", (10, 18, 2)), B=256, picks=(6, 8), s=0.0, clustered=False, m=1),
    3: dict(graph=("aisle", (50, 100, 5)), B=16384, picks=(6, 8), s=1.0, clustered=False, m=1),
    4: dict(graph=("aisle", (50, 100, 5)), B=4096, picks=(10, 11), s=1.0, clustered=True, m=3),
    5: dict(graph=("lattice", (100, 100, 10)), B=262144, picks=(6, 8), s=1.0, clustered=False, m=1),
}


def make_graph(kind: str, dims, wtype: str = I32, jitter_seed: int = 0) -> Graph:
    if kind == "aisle":
        return aisle(*dims, wtype=wtype, jitter_seed=jitter_seed)
    return lattice(*dims, wtype=wtype, jitter_seed=jitter_seed)


def config(k: int, wtype: str = I32, clustered=None, B=None, graph: Graph = None):
    """Return (graph, orders, meta) for BASELINE.json configs[k-1].

    ``B`` overrides the order count (a prefix-stable sample is NOT implied:
    a different B re-draws the stream). ``clustered`` overrides the layout
    (config 3 is run both ways).
    """
    c = CONFIGS[k]
    if graph is None:
        graph = make_graph(c["graph"][0], c["graph"][1], wtype, jitter_seed=1000 + k)
    cl = c["clustered"] if clustered is None else clustered
    sku_node = place_skus(graph, clustered=cl, seed=k)
    nB = c["B"] if B is None else B
    orders = zipf_orders(sku_node, nB, c["picks"][0], c["picks"][1], c["s"], seed=100 + k)
    meta = dict(config=k, clustered=cl, m=c["m"], wtype=wtype, B=nB,
                graph=graph.name, V=graph.V, E=graph.E)
    return graph, orders, meta
