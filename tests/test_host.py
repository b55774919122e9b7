"""Host-side checks that need no GPU: the C ABI library loads and exports
every entry point declared in include/rama_b200.h; config validation and
the public API surface mirror the reference (parcut/__init__.py:58-104,
solver.py:27-62)."""

import ctypes
import os
import re

import pytest

import paper_2109_01838_b200 as P
from paper_2109_01838_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rama_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t|uint64_t)\s+(rama_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    path = _build.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    # the Python binding covers exactly the header
    assert sorted(_lib.EXPORTED) == syms


def test_version_and_error_without_device():
    lib = _lib.load()
    assert lib.rama_version() >= 10000
    assert lib.rama_last_error() is not None


def test_abi_struct_layout():
    assert ctypes.sizeof(_lib.RamaCfg) == 32
    assert ctypes.sizeof(_lib.RamaRound) == 64


def test_public_names_match_reference_hot_path():
    hot = ["ContractionMapping", "ContractionResult", "connected_components", "contract", "contract_graph",
           "contraction_step", "gaec_exhaustive", "select_matching", "select_max_edge",
           "select_spanning_forest_no_conflicts", "MC_TRIANGLE", "ConflictedCycle", "DualState", "Triplet",
           "lower_bound", "message_passing_iteration", "mp_edge_to_triplets", "mp_triplets_to_edges",
           "reparametrized_edge_costs", "reparametrized_graph", "separate_conflicted_cycles",
           "triangle_min_marginal", "triangulate", "grid_graph", "random_graph", "ParseError", "SparseAdjacency",
           "WeightedGraph", "build_adjacency", "canonical_labels", "clustering_cost", "parse_instance",
           "serialize_instance", "MODES", "RoundRecord", "Solution", "SolverConfig", "dual_bound", "solve"]
    for name in hot:
        assert hasattr(P, name), name


def test_config_validation_matches_reference():  # test_solver.py:221-246
    assert P.SolverConfig(mode="PD").resolved_cycle_length() == 5
    assert P.SolverConfig(mode="PD+").resolved_cycle_length() == 7
    assert P.SolverConfig(mode="PD+", max_cycle_length=4).resolved_cycle_length() == 4
    bad = [dict(mode="QP"), dict(mode="D", mp_iterations=0), dict(max_cycle_length=2),
           dict(matching_switch_fraction=0.0), dict(matching_switch_fraction=1.5), dict(max_rounds=0),
           dict(mode="D", separation_rounds=0)]
    for kw in bad:
        with pytest.raises(ValueError):
            P.SolverConfig(**kw).validate()
    P.SolverConfig(mode="P", matching_switch_fraction=1.0).validate()


def test_cfg_marshalling():
    c = P.SolverConfig(mode="PD+", mp_iterations=3, max_rounds=7).to_c()
    assert (c.mode, c.mp_iterations, c.max_cycle_length, c.max_rounds) == (2, 3, 7, 7)


def test_dual_bound_requires_mode_d():
    with pytest.raises(ValueError):
        P.dual_bound(None, P.SolverConfig(mode="PD"))


def test_canonical_labels_and_parse_host():  # graph.py:148-157, test_graph.py
    assert P.canonical_labels([5, 5, 2, 7, 2]).tolist() == [0, 0, 1, 2, 1]
    with pytest.raises(P.ParseError, match="line 1"):
        P.parse_instance("0 1 2.5\n")
    with pytest.raises(P.ParseError, match="line 2"):
        P.parse_instance("MULTICUT\n0 0 1.0\n")


def test_gaec_mode_warns_on_large_graphs():
    """Mode GAEC is exact but joins one edge per round:
    large inputs get a RuntimeWarning before any work, small ones do not."""
    import warnings

    from paper_2109_01838_b200 import solver as S

    cfg = S.SolverConfig(mode="GAEC")
    with pytest.warns(RuntimeWarning, match="one edge per round"):
        S._warn_gaec(cfg, S.GAEC_WARN_NODES + 1)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        S._warn_gaec(cfg, 1000)
        S._warn_gaec(S.SolverConfig(mode="PD"), 10 ** 7)
