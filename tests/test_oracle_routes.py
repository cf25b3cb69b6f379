"""Pins of the oracle's route functions (O4-O8) and of the paper's printed
arithmetic: brute force by itertools, an independent Held-Karp, the
hand-computed 3-aisle example, Theorem 3.1 counts (§3),
2,903,040 = 9!*8 (§4.6). CPU only."""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from test_oracle_bf import load_three_aisle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = np.iinfo(np.int32).max


def load_paper_values():
    rec = {}
    for line in open(os.path.join(GOLD, "paper_values.txt")):
        line = line.split("#")[0].split()
        if line:
            rec.setdefault(line[0], []).append([int(x) for x in line[1:]])
    return rec


def lr_cost(D, seq):
    """Left-to-right route cost written independently (numpy scalars)."""
    if len(seq) < 2:
        return D.dtype.type(0)
    c = D[seq[0], seq[1]]
    for a, b in zip(seq[1:-1], seq[2:]):
        if D.dtype == np.int32:
            if c == INF or D[a, b] == INF:
                c = np.int32(INF)
            else:
                c = np.int32(int(c) + int(D[a, b]))
        else:
            c = np.float32(c + D[a, b])
    return c


def brute(D):
    n = D.shape[0]
    best = None
    for r, p in enumerate(itertools.permutations(range(n))):
        c = lr_cost(D, p)
        if best is None or c < best[0]:
            best = (c, r, p)
    return best


def held_karp(D):
    """Independent O(n^2 2^n) open-path DP (§3) with the same
    left-to-right association: best[S][j] = min_i fl(best[S-j][i] + D[i][j])."""
    n = D.shape[0]
    fp = D.dtype == np.float32
    add = (lambda a, b: np.float32(a + b)) if fp else (lambda a, b: a + b)
    best = {}
    for j in range(n):
        best[(1 << j, j)] = D.dtype.type(0) if fp else 0
    for size in range(2, n + 1):
        for S in range(1 << n):
            if bin(S).count("1") != size:
                continue
            for j in range(n):
                if not S >> j & 1:
                    continue
                P = S & ~(1 << j)
                vals = [add(best[(P, i)], D[i, j]) for i in range(n) if P >> i & 1]
                best[(S, j)] = min(vals)
    full = (1 << n) - 1
    return min(best[(full, j)] for j in range(n))


def lex_argmin_int(D):
    """Exact lexicographically smallest optimal open path for int D: suffix DP
    g[S][j] = cost of best path covering S starting at j, then greedy."""
    n = D.shape[0]
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def g(S, j):
        rest = S & ~(1 << j)
        if rest == 0:
            return 0
        return min(int(D[j, k]) + g(rest, k) for k in range(n) if rest >> k & 1)

    full = (1 << n) - 1
    opt = min(g(full, j) for j in range(n))
    seq, S, cost = [], full, 0
    j = min(j for j in range(n) if g(full, j) == opt)
    seq.append(j)
    while S & ~(1 << j):
        rest = S & ~(1 << j)
        k = min(k for k in range(n) if rest >> k & 1 and int(D[j, k]) + g(rest, k) == g(S, j))
        cost += int(D[j, k])
        S, j = rest, k
        seq.append(j)
    return opt, seq


def random_D(rng, n, kind, symmetric=False):
    if kind == "int":
        D = rng.integers(0, 30, (n, n)).astype(np.int32)
    else:
        D = rng.uniform(0, 10, (n, n)).astype(np.float32)
        D[rng.random((n, n)) < 0.1] = np.float32(0.1)  # force some fp32 ties/absorption
    if symmetric:
        D = np.triu(D) + np.triu(D, 1).T
    np.fill_diagonal(D, 0)
    return D


# ---------------------------------------------------------------- O4
def test_route_cost_hand_sums():
    rec = load_three_aisle()
    D = rec["D"]
    assert oracle.route_cost(D, [0, 2, 1, 3, 4]) == 6 + 2 + 6 + 3
    assert oracle.route_cost(D, [4]) == 0
    D2 = D.copy()
    D2[1, 3] = INF
    assert oracle.route_cost(D2, [0, 1, 3]) == INF


def test_route_cost_left_to_right_fp32():
    # legs (0.2, 1.1, 0.2, 3.7): forward 5.2000003 vs reversed 5.1999998
    D = np.zeros((5, 5), dtype=np.float32)
    legs = [0.2, 1.1, 0.2, 3.7]
    for i, x in enumerate(legs):
        D[i, i + 1] = np.float32(x)
        D[i + 1, i] = np.float32(x)
    fwd = oracle.route_cost(D, [0, 1, 2, 3, 4])
    rev = oracle.route_cost(D, [4, 3, 2, 1, 0])
    assert fwd == np.float32(np.float32(np.float32(np.float32(0.2) + np.float32(1.1)) + np.float32(0.2)) + np.float32(3.7))
    assert fwd != rev
    assert float(fwd) == pytest.approx(5.2000003, abs=1e-7)
    assert float(rev) == pytest.approx(5.1999998, abs=1e-7)


# ---------------------------------------------------------------- O5
def test_exact_three_aisle_and_histogram():
    rec = load_three_aisle()
    D = rec["D"]
    cost, rank, seq = oracle.exact_route(D)
    exp_cost, exp_seq, exp_rank, n_opt, max_cost = rec["exact"]
    assert (cost, rank, seq.tolist()) == (exp_cost, exp_rank, exp_seq)
    costs = [lr_cost(D, p) for p in itertools.permutations(range(5))]
    assert costs.count(exp_cost) == n_opt and max(costs) == max_cost
    # every rank range returns the exact minimum of that range
    for lo, hi in [(0, 1), (0, 7), (5, 64), (64, 120)]:
        c, r, s = oracle.exact_route_range(D, lo, hi)
        sub = costs[lo:hi]
        assert c == min(sub) and r == lo + sub.index(min(sub))


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_exact_equals_brute_force(kind):
    rng = np.random.default_rng(31 if kind == "int" else 32)
    for trial in range(60):
        n = int(rng.integers(1, 7))
        D = random_D(rng, n, kind)
        cost, rank, seq = oracle.exact_route(D)
        bc, br, bp = brute(D)
        assert cost.tobytes() == np.asarray(bc, dtype=D.dtype).tobytes()
        assert rank == br and seq.tolist() == list(bp)
        assert oracle.perm_rank(seq) == rank


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_exact_equals_held_karp(kind):
    rng = np.random.default_rng(41 if kind == "int" else 42)
    for trial in range(40 if kind == "int" else 30):
        n = int(rng.integers(2, 8))
        D = random_D(rng, n, kind)
        cost, rank, seq = oracle.exact_route(D)
        assert np.asarray(cost, D.dtype).tobytes() == np.asarray(held_karp(D), D.dtype).tobytes()
        if kind == "int":
            opt, lseq = lex_argmin_int(D)
            assert cost == opt and seq.tolist() == lseq


def test_reversal_invariance_int_symmetric():
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(2, 8))
        D = random_D(rng, n, "int", symmetric=True)
        p = rng.permutation(n)
        assert oracle.route_cost(D, p) == oracle.route_cost(D, p[::-1])
        cost, rank, seq = oracle.exact_route(D)
        assert seq[0] < seq[-1] or n == 1  # lexicographic argmin has first < last


# ---------------------------------------------------------------- O6
def test_chunked_equals_unchunked():
    rng = np.random.default_rng(51)
    for trial in range(30):
        n = int(rng.integers(2, 8))
        kind = "int" if trial % 2 else "fp32"
        D = random_D(rng, n, kind)
        c0, r0, s0 = oracle.exact_route(D)
        chunk = int(rng.integers(1, math.factorial(n) + 2))
        c1, r1, s1, nch = oracle.exact_route_chunked(D, chunk)
        assert (np.asarray(c0).tobytes(), r0, s0.tolist()) == (np.asarray(c1).tobytes(), r1, s1.tolist())
        assert nch == -(-math.factorial(n) // chunk)


def test_paper_capacity_arithmetic():
    pv = load_paper_values()
    cap = pv["capacity"][0][0]
    assert cap == math.factorial(9) * 8  # P658: 2,903,040 = 9! * (9-1)
    assert math.factorial(9) * 8 <= cap < math.factorial(10) * 9
    for n, nch in pv["chunks"]:
        assert -(-math.factorial(n) // cap) == nch
    # SPEC S445: plan_segmentation(10, 4) -> (0,4),(4,4),(8,2)
    assert [(lo, min(4, 10 - lo)) for lo in range(0, 10, 4)] == [(0, 4), (4, 4), (8, 2)]


def test_chunk_count_on_real_chunked_search():
    rng = np.random.default_rng(3)
    D = random_D(rng, 7, "int")
    c, r, s, nch = oracle.exact_route_chunked(D, 1000)
    assert nch == 6  # ceil(5040 / 1000)


# ---------------------------------------------------------------- O7
def test_segmented_three_aisle():
    rec = load_three_aisle()
    D = rec["D"]
    for labels, cost, seq in rec["segmented"]:
        c, s, counts = oracle.segmented_route(D, labels)
        assert (int(c), s.tolist()) == (cost, seq), labels
    c, s, counts = oracle.segmented_route(D, [0] * 5)
    assert (c, s.tolist(), counts) == (17, [0, 2, 1, 3, 4], (120, 2))
    c, s, counts = oracle.segmented_route(D, [0, 1, 2, 3, 4])
    assert (c, s.tolist(), counts) == (17, [0, 2, 1, 3, 4], (5, 3840))


def test_theorem_3_1_counts_paper():
    pv = load_paper_values()
    for row in pv["thm31"]:
        expect, parts = row[0], row[1:]
        red, brute_count = oracle.route_count_reduction(parts)
        assert red == expect
        assert brute_count == math.factorial(sum(parts)) // 2
        # the oracle's directed stitch enumerates exactly twice that many
        m = len(parts)
        if sum(parts) <= 12:
            D = np.zeros((sum(parts), sum(parts)), dtype=np.int32)
            labels = np.repeat(np.arange(m), parts)
            _, _, counts = oracle.segmented_route(D, labels)
            assert counts[0] + counts[1] == 2 * expect


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_segmented_invariants(kind):
    rng = np.random.default_rng(61 if kind == "int" else 62)
    for trial in range(40):
        n = int(rng.integers(1, 8))
        D = random_D(rng, n, kind)
        ec, er, es = oracle.exact_route(D)
        c1, s1, _ = oracle.segmented_route(D, np.zeros(n, dtype=np.int32))
        assert np.asarray(c1).tobytes() == np.asarray(ec).tobytes() and s1.tolist() == es.tolist()
        cs, ss, _ = oracle.segmented_route(D, np.arange(n))
        assert np.asarray(cs).tobytes() == np.asarray(ec).tobytes() and ss.tolist() == es.tolist()
        labels = rng.integers(0, 3, n)
        c, s, _ = oracle.segmented_route(D, labels)
        assert c >= ec
        assert sorted(s.tolist()) == list(range(n))
        assert np.asarray(oracle.route_cost(D, s)).tobytes() == np.asarray(c).tobytes()


# ---------------------------------------------------------------- NEXT-2 Held-Karp exact
@pytest.mark.parametrize("kind", ["int", "int_ties", "fp32"])
def test_held_karp_equals_enumeration(kind):
    """The subset DP returns exactly O5's result (cost bits, lexicographic
    argmin, rank) - including matrices with many equal-cost orders."""
    rng = np.random.default_rng(81)
    for trial in range(60):
        n = int(rng.integers(1, 10))
        if kind == "int_ties":
            D = rng.integers(0, 3, (n, n)).astype(np.int32)
            np.fill_diagonal(D, 0)
        else:
            D = random_D(rng, n, kind)
        ec, er, es = oracle.exact_route(D)
        hc, hr, hs = oracle.held_karp_route(D)
        assert np.asarray(hc).tobytes() == np.asarray(ec).tobytes()
        assert hs.tolist() == es.tolist() and hr == er


def load_hk_absorption():
    mats, cur = {}, None
    for line in open(os.path.join(GOLD, "hk_absorption.txt")):
        line = line.split("#")[0].split()
        if not line:
            continue
        if line[0] == "matrix":
            cur = line[1]
            mats[cur] = []
        else:
            mats[cur].append([np.float32(x) for x in line])
    return {k: np.array(v, np.float32) for k, v in mats.items()}


def absorption_D(rng, n):
    """fp32 matrices built to make rounding ties: n-1 "near" stops joined by
    small legs (0.5 .. 3) and one "far" stop whose legs are ~1e8 (ulp 8),
    so every order pays one big leg that absorbs the small prefix sums
    before it (reading A16: fl(c + d) is monotone but not strictly)."""
    small = np.array([0.5, 1, 1.5, 2, 3], np.float32)
    D = rng.choice(small, (n, n)).astype(np.float32)
    far = int(rng.integers(0, n))
    D[far, :] = np.float32(1e8) + rng.integers(0, 4, n).astype(np.float32) * 8
    D[:, far] = np.float32(1e8) + rng.integers(0, 4, n).astype(np.float32) * 8
    np.fill_diagonal(D, 0)
    return D


def cheapest_prefix_dp_argmin(D):
    """The round-1 DP (kept for the test only): per state the cheapest
    prefix, ties -> lexicographically smaller prefix. Not O5 for fp32."""
    n = D.shape[0]
    best = {(1 << j, j): (np.float32(0), (j,)) for j in range(n)}
    for size in range(2, n + 1):
        for S in range(1 << n):
            if bin(S).count("1") != size:
                continue
            for j in range(n):
                if not S >> j & 1:
                    continue
                P = S & ~(1 << j)
                cands = [(np.float32(best[(P, i)][0] + D[i, j]), best[(P, i)][1] + (j,)) for i in range(n) if P >> i & 1]
                best[(S, j)] = min(cands, key=lambda x: (x[0], x[1]))
    full = (1 << n) - 1
    return min((best[(full, j)] for j in range(n)), key=lambda x: (x[0], x[1]))[1]


def test_held_karp_fp32_absorption_reproducers():
    """The round-1 counterexamples (tests/golden/hk_absorption.txt and a real
    C3 fp32 order): the subset DP must return O5's lexicographically smallest
    optimum, recomputed here by itertools brute force."""
    for name, D in load_hk_absorption().items():
        bc, br, bs = brute(D)
        hc, hr, hs = oracle.held_karp_route(D)
        assert np.float32(hc).tobytes() == np.float32(bc).tobytes(), name
        assert hs.tolist() == list(bs) and hr == br == 0, name
    g, _, _ = gen.config(3, wtype="f32")
    stops = np.array([40, 1544, 1568, 2145, 2441, 2455, 3461, 3876, 4878], np.int32)
    D = oracle.bf_many(g, stops)[:, stops]
    bc, br, bs = brute(D)
    hc, hr, hs = oracle.held_karp_route(D)
    assert np.float32(hc).tobytes() == np.float32(bc).tobytes()
    assert hs.tolist() == list(bs) and hr == br


def test_held_karp_fp32_absorption_random_vs_brute():
    """Absorption-heavy fp32 matrices, n = 4..7: (cost, order, rank) equal the
    itertools brute force; at least some instances have several optimal
    orders whose prefixes differ in cost, so the round-1 DP that kept one
    cheapest prefix per state returns another order on them."""
    rng = np.random.default_rng(83)
    hard = 0   # instances the round-1 DP (cheapest prefix per state) got wrong
    for trial in range(150):
        n = int(rng.integers(4, 8))
        D = absorption_D(rng, n)
        bc, br, bs = brute(D)
        hc, hr, hs = oracle.held_karp_route(D)
        assert np.float32(hc).tobytes() == np.float32(bc).tobytes(), trial
        assert hs.tolist() == list(bs) and hr == br, trial
        hard += list(cheapest_prefix_dp_argmin(D)) != list(bs)
    assert hard >= 5


def test_held_karp_large_vs_independent_dp():
    """n = 12..13 (beyond cheap enumeration): cost equals the tests' own
    Held-Karp; the int order equals the independent suffix-DP lexicographic
    argmin; the worked example gives 17, (0,2,1,3,4), rank 6."""
    rng = np.random.default_rng(82)
    for n, kind in ((12, "int"), (13, "int"), (12, "fp32")):
        D = random_D(rng, n, kind)
        hc, hr, hs = oracle.held_karp_route(D)
        assert np.asarray(hc).tobytes() == np.asarray(held_karp(D)).tobytes()
        if kind == "int":
            c2, s2 = lex_argmin_int(D)
            assert int(hc) == c2 and hs.tolist() == list(s2)
    D = load_three_aisle()["D"]
    hc, hr, hs = oracle.held_karp_route(D)
    assert int(hc) == 17 and hs.tolist() == [0, 2, 1, 3, 4] and hr == 6


# ---------------------------------------------------------------- NEXT-1 boundary pairs
def _contiguous_best(D, labels):
    """Brute force over ALL n! orders keeping those in which every segment's
    stops are consecutive: (min left-to-right cost, lexicographically
    smallest such order). For int weights this is what the boundary-pair
    stitch must return (reading R1)."""
    n = D.shape[0]
    best = None
    for p in itertools.permutations(range(n)):
        seen, prev, ok = set(), None, True
        for x in p:
            lab = labels[x]
            if lab != prev:
                if lab in seen:
                    ok = False
                    break
                seen.add(lab)
                prev = lab
        if not ok:
            continue
        c = lr_cost(D, p)
        if best is None or c < best[0]:   # permutations() is lexicographic: first wins ties
            best = (c, p)
    return best


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_pairs_reduces_to_exact(kind):
    """One segment, or all singletons: the boundary-pair stitch is the exact
    route (cost and lexicographic argmin)."""
    rng = np.random.default_rng(71 if kind == "int" else 72)
    for trial in range(30):
        n = int(rng.integers(1, 7))   # <= 6 segments (WR_MAX_SEGMENTS)
        D = random_D(rng, n, kind)
        ec, er, es = oracle.exact_route(D)
        for labels in (np.zeros(n, dtype=np.int32), np.arange(n, dtype=np.int32)):
            c, s, _ = oracle.segmented_pairs_route(D, labels)
            assert np.asarray(c).tobytes() == np.asarray(ec).tobytes() and s.tolist() == es.tolist()


def test_pairs_equals_contiguous_brute_force_and_dominates():
    """int: the boundary-pair result is the best segment-contiguous order
    (independent brute force), never worse than the paper's fixed-route
    stitch (O7), strictly better on some instances; counts follow the
    definition (sum n_j! segment orders, m! * prod pairs candidates)."""
    rng = np.random.default_rng(73)
    strictly = 0
    for trial in range(120):
        n = int(rng.integers(2, 8))
        D = random_D(rng, n, "int")
        labels = rng.integers(0, 3, n).astype(np.int32)
        c, s, counts = oracle.segmented_pairs_route(D, labels)
        bc, bp = _contiguous_best(D, labels)
        assert int(c) == int(bc) and tuple(s.tolist()) == tuple(bp)
        oc, _, _ = oracle.segmented_route(D, labels)
        assert int(c) <= int(oc)
        strictly += int(c) < int(oc)
        segs = [int((labels == l).sum()) for l in np.unique(labels)]
        assert counts[0] == sum(math.factorial(k) for k in segs)
        pairs = math.prod(k * (k - 1) if k >= 2 else 1 for k in segs)
        assert counts[1] == math.factorial(len(segs)) * pairs
    assert strictly > 0


def test_pairs_three_aisle_labelings():
    """Worked example (tests/golden/three_aisle.txt): segments of <= 2 stops
    give the same stitch as O7 (both orientations are all endpoint pairs):
    17 / 21 / 22 as in P3."""
    D = load_three_aisle()["D"]
    for labels, cost in (([0, 1, 1, 2, 2], 17), ([0, 0, 1, 1, 2], 21), ([0, 1, 2, 0, 1], 22)):
        c, s, _ = oracle.segmented_pairs_route(D, np.array(labels, np.int32))
        assert int(c) == cost


# ---------------------------------------------------------------- O8
def test_kmeans_separated_clusters():
    xy = np.array([[0, 0], [100, 100], [1, 0], [0, 1], [200, 0], [101, 99], [201, 1]])
    # farthest-point init: c0 = point 0; the farthest from it is (201,1)
    # (40402 > 40000 > 20000) -> cluster 1; then (100,100) -> cluster 2
    assert oracle.kmeans(xy, 3).tolist() == [0, 2, 0, 0, 1, 2, 1]
    assert oracle.kmeans(xy, 1).tolist() == [0] * 7
    assert oracle.kmeans(xy[:2], 3).tolist() == [0, 1]


def test_kmeans_is_lloyd_fixpoint():
    """Independent check with exact rationals: on convergence every point sits
    at a nearest centroid of the final partition (ties -> lower index)."""
    rng = np.random.default_rng(71)
    for trial in range(100):
        n = int(rng.integers(1, 13))
        K = int(rng.integers(1, 4))
        xy = rng.integers(0, 40, (n, 2))
        lab = oracle.kmeans(xy, K)
        Kc = min(K, n)
        assert lab.min() >= 0 and lab.max() < Kc
        cents = {}
        for k in range(Kc):
            pts = xy[lab == k]
            if len(pts):
                cents[k] = (Fraction(int(pts[:, 0].sum()), len(pts)), Fraction(int(pts[:, 1].sum()), len(pts)))
        for p in range(n):
            d = {k: (xy[p, 0] - c[0]) ** 2 + (xy[p, 1] - c[1]) ** 2 for k, c in cents.items()}
            best = min(d.values())
            # the point's own cluster is at minimal distance, and no nonempty
            # lower-index cluster ties with it (a fixpoint of the tie rule)
            assert d[lab[p]] == best
            assert all(not (k < lab[p] and d[k] == best) for k in d)


def test_order_stops_vs_numpy():
    rng = np.random.default_rng(81)
    for _ in range(50):
        nodes = rng.integers(0, 20, int(rng.integers(1, 15)))
        assert oracle.order_stops(nodes).tolist() == np.unique(nodes).tolist()


# ------------------------------------------------------- composed pipeline
def test_route_orders_composition_c2():
    g, orders, meta = gen.config(2)
    res = oracle.route_orders(g, orders, m=1)
    assert res["rc"] == 0
    for o in range(0, orders.B, 37):
        nodes = orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]]
        stops = np.unique(nodes)
        rows = oracle.bf_many(g, stops)
        D = rows[:, stops]
        c, r, s = oracle.exact_route(D)
        assert res["cost"][o] == c and res["rank"][o] == r
        assert res["seq"][o, :len(stops)].tolist() == stops[s].tolist()


# ------------------------------------------------ NEXT-4 closed tour (R4)
def lr_closed(D, din, dout, seq):
    """Closed tour depot -> seq -> depot written independently: the first
    leg, then each stop leg, then the return leg, left to right."""
    fp = D.dtype == np.float32
    c = din[seq[0]]
    legs = [D[a, b] for a, b in zip(seq[:-1], seq[1:])] + [dout[seq[-1]]]
    for x in legs:
        if fp:
            c = np.float32(c + x)
        else:
            c = np.int32(INF) if (c == INF or x == INF) else np.int32(int(c) + int(x))
    return c


def brute_closed(D, din, dout):
    best, nopt = None, 0
    for r, p in enumerate(itertools.permutations(range(D.shape[0]))):
        c = lr_closed(D, din, dout, p)
        if best is None or c < best[0]:
            best, nopt = (c, r, p), 1
        elif c == best[0]:
            nopt += 1
    return best, nopt


def legs_for(rng, n, kind):
    if kind == "int":
        return rng.integers(0, 30, n).astype(np.int32), rng.integers(0, 30, n).astype(np.int32)
    return rng.uniform(0, 10, n).astype(np.float32), rng.uniform(0, 10, n).astype(np.float32)


def test_closed_three_aisle_worked_example():
    rec = load_three_aisle()
    depot, din, cost, seq, rank, nopt = rec["closed"]
    g = gen.aisle(3, 4, 2, ws=1, wa=3, wd=2)
    picks = rec["picks"]
    assert oracle.bf(g, depot)[picks].tolist() == din                 # the legs, by BF
    assert [int(oracle.bf(g, p)[depot]) for p in picks] == din        # undirected: dout = din
    D = rec["D"]
    c, r, s = oracle.exact_closed_route(D, din, din)
    assert (int(c), r, s.tolist()) == (cost, rank, seq)
    (bc, br, bp), bn = brute_closed(D, np.array(din, np.int32), np.array(din, np.int32))
    assert (int(bc), br, list(bp), bn) == (cost, rank, seq, nopt)
    assert oracle.closed_route_cost(D, din, din, [0, 2, 1, 3, 4]) == 34   # the open optimum, closed
    hc, hr, hs = oracle.held_karp_closed_route(D, din, din)
    assert (int(hc), hr, hs.tolist()) == (cost, rank, seq)


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_closed_exact_and_held_karp_equal_brute_force(kind):
    rng = np.random.default_rng(404 if kind == "int" else 405)
    for trial in range(60):
        n = int(rng.integers(1, 7))
        D = random_D(rng, n, kind)
        din, dout = legs_for(rng, n, kind)
        (bc, br, bp), _ = brute_closed(D, din, dout)
        c, r, s = oracle.exact_closed_route(D, din, dout)
        assert c.tobytes() == np.asarray(bc).tobytes() and r == br and tuple(s) == bp, trial
        hc, hr, hs = oracle.held_karp_closed_route(D, din, dout)
        assert hc.tobytes() == c.tobytes() and hr == r and tuple(hs) == tuple(s), trial


def test_closed_held_karp_fp32_absorption_vs_brute():
    """Rounding ties with a far stop (reading A16) and far depot legs."""
    rng = np.random.default_rng(406)
    for trial in range(40):
        n = int(rng.integers(3, 8))
        D = absorption_D(rng, n)
        din = (np.float32(1e8) + rng.integers(0, 4, n) * 8).astype(np.float32)
        dout = rng.choice(np.array([0.5, 1, 2], np.float32), n).astype(np.float32)
        (bc, br, bp), _ = brute_closed(D, din, dout)
        hc, hr, hs = oracle.held_karp_closed_route(D, din, dout)
        assert hc.tobytes() == np.asarray(bc).tobytes() and hr == br and tuple(hs) == bp, trial


def test_closed_with_zero_legs_is_the_open_route():
    """Zero depot legs reduce every closed function to its open counterpart
    bit for bit (fl(0 + c) = c, fl(c + 0) = c): exact, Held-Karp, O7 and the
    pair stitch."""
    rng = np.random.default_rng(407)
    for kind in ("int", "fp32"):
        for trial in range(25):
            n = int(rng.integers(2, 8))
            D = random_D(rng, n, kind)
            z = np.zeros(n, D.dtype)
            a, b = oracle.exact_closed_route(D, z, z), oracle.exact_route(D)
            assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1] and np.array_equal(a[2], b[2])
            h = oracle.held_karp_closed_route(D, z, z)
            assert h[0].tobytes() == b[0].tobytes() and h[1] == b[1]
            labels = rng.integers(0, 3, n).astype(np.int32)
            sc, ss, sn = oracle.segmented_closed_route(D, z, z, labels)
            oc, os_, on = oracle.segmented_route(D, labels)
            assert sc.tobytes() == np.asarray(oc).tobytes() and np.array_equal(ss, os_) and sn == on
            pc, ps, pn = oracle.segmented_pairs_closed_route(D, z, z, labels)
            qc, qs, qn = oracle.segmented_pairs_route(D, labels)
            assert pc.tobytes() == np.asarray(qc).tobytes() and np.array_equal(ps, qs) and pn == qn


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_closed_segmented_invariants(kind):
    """O7 / pair stitch of a closed tour (segments routed open, the stitch
    costs the closed tour): all-singleton labelings equal the exact closed
    tour; one segment gives the better orientation of the open O5 route,
    closed; any labeling costs >= the exact closed tour; the pair stitch
    never costs more than O7 for int weights; an int instance equals brute
    force over all segment-contiguous closed orders (the pair stitch's
    definition)."""
    rng = np.random.default_rng(408 if kind == "int" else 409)
    for trial in range(25):
        n = int(rng.integers(2, 8))
        D = random_D(rng, n, kind)
        din, dout = legs_for(rng, n, kind)
        ec, er, es = oracle.exact_closed_route(D, din, dout)
        c, s, _ = oracle.segmented_closed_route(D, din, dout, np.arange(n, dtype=np.int32))
        assert c.tobytes() == ec.tobytes() and np.array_equal(s, es)
        _, _, op = oracle.exact_route(D)
        cands = sorted([(lr_closed(D, din, dout, q), tuple(q)) for q in (list(op), list(op)[::-1])])
        c, s, _ = oracle.segmented_closed_route(D, din, dout, np.zeros(n, np.int32))
        assert c.tobytes() == np.asarray(cands[0][0]).tobytes() and tuple(s) == cands[0][1]
        labels = rng.integers(0, 3, n).astype(np.int32)
        c, s, _ = oracle.segmented_closed_route(D, din, dout, labels)
        assert c >= ec and lr_closed(D, din, dout, s).tobytes() == c.tobytes()
        pc, ps, _ = oracle.segmented_pairs_closed_route(D, din, dout, labels)
        assert lr_closed(D, din, dout, ps).tobytes() == pc.tobytes()
        if kind == "int":
            assert pc <= c
            # brute force over orders whose segments are contiguous
            best = None
            for p in itertools.permutations(range(n)):
                segs = [labels[i] for i in p]
                runs = [k for k in range(n) if k == 0 or segs[k] != segs[k - 1]]
                if len(runs) != len(set(labels.tolist())):
                    continue
                cc = lr_closed(D, din, dout, p)
                if best is None or cc < best[0] or (cc == best[0] and p < best[1]):
                    best = (cc, p)
            assert int(pc) == int(best[0]) and tuple(ps) == best[1]


def test_closed_reversal_invariance_int_symmetric():
    rng = np.random.default_rng(410)
    for _ in range(30):
        n = int(rng.integers(2, 8))
        D = random_D(rng, n, "int", symmetric=True)
        din, _ = legs_for(rng, n, "int")
        c, r, s = oracle.exact_closed_route(D, din, din)
        assert lr_closed(D, din, din, s[::-1]) == c
