"""Seeded instance generators -- drop-in for ``parcut.generate``.

Same instances as generate.py:8-62 (the COO comes from instances.py and is
canonicalised on the GPU by WeightedGraph).
"""

from .graph import WeightedGraph
from .instances import grid_coo, random_coo


def random_graph(num_nodes, edge_probability, seed=0):
    """Erdos-Renyi graph with N(0,1) costs (generate.py:8-25)."""
    n, u, v, c = random_coo(num_nodes, edge_probability, seed)
    return WeightedGraph(n, u, v, c)


def grid_graph(height, width, stride=0, seed=0):
    """4-connected grid plus optional coarse lattice edges (generate.py:28-62)."""
    n, u, v, c = grid_coo(height, width, stride, seed)
    return WeightedGraph(n, u, v, c)
