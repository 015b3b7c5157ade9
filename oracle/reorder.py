"""Data-affinity-based reordering, Algorithm 1 (TEST INFRASTRUCTURE ONLY; small graphs).

PAPER.md §3.2, Algorithm 1, Eq. (1).
The reordering is a heuristic: many orderings are valid, so the exact ordering
is "parity unpinned" -- it is pinned only by invariants
(bijection, Q/dQ closed forms, clique contiguity, MeanNNZTC gain).

Readings:
  * graph: pattern(A or A^T) without the diagonal, weight 1 per edge;
  * Eq. (1) is global Q; the merge gain is dQ(u,v) = 2*(w_uv/2m - a_u*a_v/(2m)^2) (Q9);
  * Step I is ONE pass over vertices in ascending degree, ties by id (Alg. 1 l.2-8,
    Q11); argmax-dQ ties go to the smallest community id; merge iff dQ > 0;
  * the dendrogram DFS visits roots in ascending id, each node before its children,
    children in merge order -- the leaf (vertex) sequence;
  * Step II (Alg. 1 l.9-27): the candidate set of "u in DFS that has most common
    nbrs with v" is the next L unvisited vertices in DFS order, neighbour lists
    capped at their first H entries (ascending id); ties by DFS order;
    no candidate with >= 1 common neighbour -> continue with the next DFS vertex.
  * edge_cap (default None = Alg. 1 as printed): the library's reading R6b, where after a
    visit (whose merge decision uses all of its edges) a community carries on only its
    edge_cap = 256 heaviest community edges (ties: smaller id) -- a bound on the coarsening
    work.  The oracle's default is the literal algorithm; ``edge_cap=EDGE_CAP`` reproduces
    the library's bounded variant so tests can check the branch where it triggers
    (tests/test_oracle_partition_reorder.py) and show it is a no-op where no list grows
    past the cap;
  * non-square A -> identity (Q14).
"""
from __future__ import annotations

import numpy as np

CAND_WINDOW = 64   # L
HUB_CAP = 128      # H
EDGE_CAP = 256     # community edges carried up a merge (reading R6b)


def affinity_graph(n: int, rowptr, colidx):
    """Sorted adjacency lists of pattern(A or A^T) minus self-loops."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    keep = rows != colidx
    r, c = rows[keep], colidx[keep]
    keys = np.unique(np.concatenate([r * n + c, c * n + r]))
    src, dst = keys // n, keys % n
    adj = [[] for _ in range(n)]
    for s, d in zip(src.tolist(), dst.tolist()):
        adj[s].append(d)
    return adj


def modularity(adj, comm) -> float:
    """Eq. (1) as the global Q = (1/2m) sum_{i,j} (A_ij - k_i k_j / 2m) delta(s_i, s_j)."""
    n = len(adj)
    k = [len(a) for a in adj]
    m2 = sum(k)
    if m2 == 0:
        raise ValueError("empty graph")
    q = 0.0
    for i in range(n):
        nb = set(adj[i])
        for j in range(n):
            if comm[i] == comm[j]:
                q += (1.0 if j in nb else 0.0) - k[i] * k[j] / m2
    return q / m2


def delta_q(w_uv: float, a_u: float, a_v: float, m2: float) -> float:
    """Merge gain of joining communities u and v."""
    return 2.0 * (w_uv / m2 - a_u * a_v / (m2 * m2))


def dendrogram(adj, edge_cap: int | None = None, stats: dict | None = None):
    """Alg. 1 Step I (l.1-8): returns (parent, children, roots) of the merge forest.

    edge_cap: None = literal Alg. 1; an int = reading R6b (see the module docstring).
    stats (optional dict): receives "truncations" = how many visits truncated a list."""
    n = len(adj)
    deg = [len(a) for a in adj]
    m2 = float(sum(deg))
    parent = list(range(n))
    a = [float(d) for d in deg]
    children = [[] for _ in range(n)]
    edges = [dict((x, 1) for x in adj[v]) for v in range(n)]

    def find(x):
        root = x
        while parent[root] != root:
            root = parent[root]
        while parent[x] != root:
            parent[x], x = root, parent[x]
        return root

    for v in sorted(range(n), key=lambda u: (deg[u], u)):   # l.2 ascending degree
        if deg[v] == 0 or m2 == 0:
            continue
        acc = {}
        for x, w in edges[v].items():
            r = find(x)
            if r != v:
                acc[r] = acc.get(r, 0) + w
        best, best_dq = -1, 0.0
        for r in sorted(acc):                                # l.4 argmax dQ, smallest id on ties
            dq = delta_q(acc[r], a[r], a[v], m2)
            if best < 0 or dq > best_dq:
                best, best_dq = r, dq
        if edge_cap is not None and len(acc) > edge_cap:     # reading R6b (not in Alg. 1)
            keep = sorted(acc.items(), key=lambda kv: (-kv[1], kv[0]))[:edge_cap]
            acc = dict(keep)
            if stats is not None:
                stats["truncations"] = stats.get("truncations", 0) + 1
        edges[v] = acc
        if best >= 0 and best_dq > 0.0:                      # l.5-7 merge v into u
            u = best
            parent[v] = u
            a[u] += a[v]
            eu = edges[u]
            for x, w in acc.items():
                eu[x] = eu.get(x, 0) + w
            edges[v] = {}
            children[u].append(v)
    roots = [v for v in range(n) if parent[v] == v]
    return parent, children, roots


def dfs_sequence(children, roots):
    seq = []
    for r in roots:
        stack = [r]
        while stack:
            x = stack.pop()
            seq.append(x)
            stack.extend(reversed(children[x]))
    return seq


def ordering(adj, children, roots, L: int = CAND_WINDOW, H: int = HUB_CAP):
    """Alg. 1 Step II (l.9-27): returns perm new -> old."""
    n = len(adj)
    seq = dfs_sequence(children, roots)
    capped = [a[:H] for a in adj]
    visited = [False] * n
    perm = []
    alive = list(seq)  # unvisited vertices in DFS order (small graphs: a plain list)

    def assign(x):
        visited[x] = True
        perm.append(x)
        alive.remove(x)

    for v in seq:
        if visited[v]:
            continue
        assign(v)                                            # l.15-17
        while alive:                                         # l.18 while-loop
            nv = set(capped[v])
            best, best_c = -1, 0
            for u in alive[:L]:
                c = sum(1 for x in capped[u] if x in nv)
                if c > best_c:
                    best, best_c = u, c
            if best < 0:
                break
            assign(best)                                     # l.22-24
            v = best                                         # l.25
    return np.asarray(perm, dtype=np.int64)


def dendrogram_rounds(adj, round_size: int):
    """Reading R21, Step I: Alg. 1's merge rule (l.2-8) applied in rounds of ``round_size``
    vertices in ascending (degree, id) order.  Each vertex of a round decides from the state at
    the round's start, counting only its own edges towards each neighbouring community; the
    merges (dQ > 0, ties by smallest community id) are applied in round order, a target that
    joined another community meanwhile standing for that community's root (skipped if it is
    the deciding vertex itself)."""
    n = len(adj)
    deg = [len(x) for x in adj]
    m2 = float(sum(deg))
    parent = list(range(n))
    a = [float(d) for d in deg]
    children = [[] for _ in range(n)]

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x

    order = sorted(range(n), key=lambda u: (deg[u], u))
    for r0 in range(0, n, round_size):
        batch = order[r0:r0 + round_size]
        props = []
        for v in batch:                                       # decisions: state at round start
            best = None
            if deg[v] > 0 and m2 > 0:
                w = {}
                for x in adj[v]:
                    r = find(x)
                    if r != v:
                        w[r] = w.get(r, 0) + 1
                best_dq = 0.0
                for r in sorted(w):
                    dq = delta_q(w[r], a[r], a[v], m2)
                    if best is None or dq > best_dq:
                        best, best_dq = r, dq
                if best is not None and not best_dq > 0.0:
                    best = None
            props.append(best)
        for v, r in zip(batch, props):                        # merges: round order
            if r is None:
                continue
            u = find(r)
            if u == v:
                continue
            parent[v] = u
            a[u] += a[v]
            children[u].append(v)
    roots = [v for v in range(n) if parent[v] == v]
    return parent, children, roots


def ordering_segments(adj, children, roots, segments: int, L: int, H: int = HUB_CAP):
    """Reading R21, Step II: the DFS leaf sequence cut into ``segments`` contiguous pieces of
    ceil(n/segments) vertices; the greedy chaining of ``ordering`` runs in each piece alone."""
    n = len(adj)
    seq = dfs_sequence(children, roots)
    size = -(-n // segments) if n else 0
    capped = [x[:H] for x in adj]
    perm = []
    for s0 in range(0, n, max(size, 1)):
        alive = list(seq[s0:s0 + size])
        visited = set()
        for v in list(alive):
            if v in visited:
                continue
            visited.add(v)
            perm.append(v)
            alive.remove(v)
            while alive:
                nv = set(capped[v])
                best, best_c = -1, 0
                for u in alive[:L]:
                    c = sum(1 for x in capped[u] if x in nv)
                    if c > best_c:
                        best, best_c = u, c
                if best < 0:
                    break
                visited.add(best)
                perm.append(best)
                alive.remove(best)
                v = best
    return np.asarray(perm, dtype=np.int64)


def reorder_parallel(M: int, K: int, rowptr, colidx, round_size: int, segments: int, L: int = 8,
                     H: int = HUB_CAP):
    """Reading R21 end to end (the library's variant for graphs above 8M vertices)."""
    if M != K:
        return np.arange(M, dtype=np.int64)
    adj = affinity_graph(M, rowptr, colidx)
    _, children, roots = dendrogram_rounds(adj, round_size)
    return ordering_segments(adj, children, roots, segments, L, H)


def reorder(M: int, K: int, rowptr, colidx, L: int = CAND_WINDOW, H: int = HUB_CAP,
            edge_cap: int | None = None, stats: dict | None = None):
    """Algorithm 1 end to end: perm new->old (identity when M != K, Q14).
    edge_cap=EDGE_CAP gives the library's reading R6b; None (default) the literal Alg. 1."""
    if M != K:
        return np.arange(M, dtype=np.int64)
    adj = affinity_graph(M, rowptr, colidx)
    _, children, roots = dendrogram(adj, edge_cap, stats)
    return ordering(adj, children, roots, L, H)
