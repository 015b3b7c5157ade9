"""Pins for oracle/partition.py (brute force) and oracle/reorder.py (Alg. 1 invariants)."""
import itertools

import numpy as np
import pytest

import gen
from oracle import bittcf as bt
from oracle import partition as op
from oracle import reorder as orr


# ----------------------------------------------------------------------------- partition

@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_bounds(seed, P):
    A = gen.uniform_random(200 + seed * 37, 300, 4000, seed=seed)
    b = op.bounds(A.M, A.rowptr, P)
    W = (A.M + 7) // 8
    assert b[0] == 0 and b[-1] == W and all(x <= y for x, y in zip(b, b[1:]))
    wn = op.window_nnz(A.M, A.rowptr)
    pre = np.concatenate([[0], np.cumsum(wn)])
    nnz = A.nnz
    # independent check of the min{} definition via searchsorted on the exact integer prefix
    for k in range(1, P):
        assert b[k] == int(np.searchsorted(P * pre, k * nnz, side="left"))
    # balance: no part exceeds its share by more than one window
    for k in range(P):
        assert pre[b[k + 1]] - pre[b[k]] <= -(-nnz // P) + wn.max()


# ----------------------------------------------------------------------------- reorder

def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    return gen.csr_from_pairs(iu[keep], ju[keep], n, n, symmetric=True)


def test_modularity_closed_forms():
    # S:153 all-in-one community -> Q = 0; S:154 two disjoint edges as two communities -> 0.5
    for seed in range(50):
        A = _random_graph(int(np.random.default_rng(seed).integers(3, 20)), 0.4, seed)
        adj = orr.affinity_graph(A.M, A.rowptr, A.colidx)
        if sum(len(a) for a in adj) == 0:
            continue
        assert abs(orr.modularity(adj, [0] * A.M)) < 1e-12
    two = gen.csr_from_pairs([0, 2], [1, 3], 4, 4, symmetric=True)
    adj = orr.affinity_graph(4, two.rowptr, two.colidx)
    assert orr.modularity(adj, [0, 0, 1, 1]) == pytest.approx(0.5, abs=1e-15)
    # K2: Q(split) = -0.5, Q(merged) = 0, dQ = 2*(1/2 - 1*1/4) = 0.5
    K2 = gen.csr_from_pairs([0], [1], 2, 2, symmetric=True)
    k2 = orr.affinity_graph(2, K2.rowptr, K2.colidx)
    assert orr.modularity(k2, [0, 1]) == pytest.approx(-0.5) and orr.modularity(k2, [0, 0]) == 0.0
    assert orr.delta_q(1, 1, 1, 2) == pytest.approx(0.5)


@pytest.mark.parametrize("seed", range(12))
def test_delta_q_equals_two_evaluations(seed):
    """dQ(u,v) == Q(after) - Q(before), exhaustively over community pairs, n <= 12."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 13))
    A = _random_graph(n, 0.35, seed)
    adj = orr.affinity_graph(n, A.rowptr, A.colidx)
    m2 = sum(len(a) for a in adj)
    if m2 == 0:
        return
    comm = list(rng.integers(0, 4, size=n))
    for cu, cv in itertools.permutations(sorted(set(comm)), 2):
        w = sum(1 for i in range(n) if comm[i] == cu for j in adj[i] if comm[j] == cv)
        au = sum(len(adj[i]) for i in range(n) if comm[i] == cu)
        av = sum(len(adj[i]) for i in range(n) if comm[i] == cv)
        after = [cu if c == cv else c for c in comm]
        assert orr.delta_q(w, au, av, m2) == pytest.approx(
            orr.modularity(adj, after) - orr.modularity(adj, comm), abs=1e-12)


def test_affinity_graph_symmetrises_and_drops_diag():
    chain = gen.csr_from_pairs([0, 1, 2], [1, 2, 2], 3, 3)   # S:144 chain 0->1->2 (+ a self-loop)
    adj = orr.affinity_graph(3, chain.rowptr, chain.colidx)
    assert [len(a) for a in adj] == [1, 2, 1]
    diag = gen.identity(5)
    assert all(len(a) == 0 for a in orr.affinity_graph(5, diag.rowptr, diag.colidx))


def test_star_merges_into_one_community():
    S = gen.star(4)
    adj = orr.affinity_graph(5, S.rowptr, S.colidx)
    parent, children, roots = orr.dendrogram(adj)
    assert len(roots) == 1


def test_reorder_bijection_determinism_identity_cases():
    for seed in range(20):
        A = _random_graph(60, 0.08, seed)
        p1 = orr.reorder(A.M, A.K, A.rowptr, A.colidx)
        p2 = orr.reorder(A.M, A.K, A.rowptr, A.colidx)
        assert sorted(p1.tolist()) == list(range(60)) and np.array_equal(p1, p2)
    D = gen.identity(9)   # diagonal only -> empty graph -> DFS order = identity
    assert orr.reorder(9, 9, D.rowptr, D.colidx).tolist() == list(range(9))
    R = gen.uniform_random(10, 12, 30, seed=1)   # non-square -> identity (Q14)
    assert orr.reorder(10, 12, R.rowptr, R.colidx).tolist() == list(range(10))


@pytest.mark.parametrize("seed", range(5))
def test_two_cliques_recovered_contiguously(seed):
    """shuffled two-clique fixture -> each clique a contiguous index range."""
    k = 8
    A = gen.two_cliques(k, seed=seed)
    lab = np.random.default_rng(seed).permutation(2 * k)
    clique_of = {int(lab[i]): (0 if i < k else 1) for i in range(2 * k)}
    perm = orr.reorder(A.M, A.K, A.rowptr, A.colidx)
    seq = [clique_of[int(v)] for v in perm]
    assert seq == sorted(seq) or seq == sorted(seq, reverse=True)


def test_dfs_tie_break_walkthrough():
    """the source gets id 0; among candidates tied at one common neighbour
    the DFS-earliest is taken next (vertices 2, 7, 4 tie via vertex 0; 2 chosen)."""
    # source 5 shares neighbour 0 with 2, 7 and 4; a dendrogram with one root 5 whose
    # DFS order is 5, 2, 7, 4, 0, ... is imposed directly.
    n = 8
    adj = [[] for _ in range(n)]
    for a, b in [(5, 0), (2, 0), (7, 0), (4, 0), (1, 3), (6, 3)]:
        adj[a].append(b)
        adj[b].append(a)
    adj = [sorted(a) for a in adj]
    children = [[] for _ in range(n)]
    children[5] = [2, 7, 4, 0, 1, 3, 6]
    perm = orr.ordering(adj, children, [5])
    assert perm[0] == 5 and perm[1] == 2


def test_reordering_raises_mean_nnz_tc_on_sbm():
    """S:572 acceptance 5: MeanNNZTC(reordered) > MeanNNZTC(shuffled) on SBM n=512, 16 blocks, 10 seeds."""
    for seed in range(10):
        A = gen.sbm(512, 16, 0.3, 0.005, seed=seed, shuffle=True)
        perm = orr.reorder(A.M, A.K, A.rowptr, A.colidx)
        rp, ci, _ = bt.permute_rows(A.M, A.rowptr, A.colidx, None, perm)
        before = bt.mean_nnz_tc(bt.encode(A.M, A.K, A.rowptr, A.colidx))
        after = bt.mean_nnz_tc(bt.encode(A.M, A.K, rp, ci))
        assert after > before
