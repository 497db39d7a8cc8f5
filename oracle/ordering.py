"""Exact greedy minimum-degree ordering (oracle).

Restates ``amd_order`` (reference src/gridnlp/sparse/amd.py:18-54): at each
step the live vertex with the smallest key ``(degree, initial_degree,
index)`` is eliminated and its neighbours are joined into a clique
(amd.py:49-53).  The reference finds the minimum with an O(n) scan per
step (amd.py:33-42); here a lazy binary heap over the same key gives the
same vertex at every step (ties are resolved by the index component, which
the scan resolves identically because it keeps the first strict minimum).
"""
from __future__ import annotations

import heapq

import numpy as np


def adjacency_from_lower(n, rows, cols):
    """Neighbour sets of the symmetric pattern, diagonal dropped (amd.py:21-26)."""
    adj = [set() for _ in range(n)]
    for i, j in zip(np.asarray(rows).tolist(), np.asarray(cols).tolist()):
        if i != j:
            adj[i].add(j)
            adj[j].add(i)
    return adj


def min_degree_order(n, rows, cols) -> np.ndarray:
    """perm[k] = original index eliminated at step k (amd.py:19)."""
    adj = adjacency_from_lower(n, rows, cols)
    deg = [len(a) for a in adj]
    deg0 = list(deg)
    alive = [True] * n
    heap = [(deg[v], deg0[v], v) for v in range(n)]
    heapq.heapify(heap)
    perm = np.empty(n, dtype=np.int64)
    for k in range(n):
        while True:
            d, d0, v = heapq.heappop(heap)
            if alive[v] and d == deg[v]:
                break
        perm[k] = v
        alive[v] = False
        nb = adj[v]
        for u in nb:                      # clique formation, amd.py:49-53
            au = adj[u]
            au.discard(v)
            au |= nb
            au.discard(u)
        for u in nb:
            if len(adj[u]) != deg[u]:
                deg[u] = len(adj[u])
                heapq.heappush(heap, (deg[u], deg0[u], u))
        adj[v] = set()
    return perm
