"""CPU-only checks: the C-ABI library loads and exports everything
include/fqaoa.h declares, the host-side planner, and the host mirror of the
reference API (validation, encodings, error contract).  No kernel launches."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2309_04841_b200 import _lib
from paper_2309_04841_b200.mixers import SU2, Mixer, complete_edges, ring_edges
from paper_2309_04841_b200.problems import Graph, labs_terms, maxcut_terms, portfolio_terms, triangle_graph
from paper_2309_04841_b200.qaoa import QaoaParams
from paper_2309_04841_b200.terms import (CompactRangeError, Term, TermPolynomial, _dyadic, compact_costs,
                                         load_terms, save_terms, term_arrays)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "fqaoa.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), f"libfqaoa.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTED), "ctypes signature table out of sync with fqaoa.h"


def test_library_is_sm100a():
    path = _lib.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_version_and_error_plumbing_without_gpu():
    lib = _lib.load()
    assert lib.fq_version() == 1
    # argument validation happens before any CUDA call
    st = lib.fq_su2_on_pairs(None, 3, 1.0, 0.0, 0.0, 0.0, 0, None)
    assert st == _lib.FQ_ERR_ARG
    assert b"bad buffer" in lib.fq_last_error()
    with pytest.raises(ValueError, match="p_lo < p_hi"):
        _lib.check(lib.fq_xy_on_pairs(ctypes.c_void_p(16), 16, 1.0, 0.0, 2, 1, None), "xy")


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.device()
    from paper_2309_04841_b200 import QaoaSimulator

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        QaoaSimulator(terms=labs_terms(4))
    from paper_2309_04841_b200 import _kernels

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _kernels.warm_up()


def _plan(n, p, state_kind=0):
    layers = (_lib.FqLayer * p)(*[_lib.FqLayer(0.1, 0.2, 1, 0, n) for _ in range(p)])
    return _lib.load().fq_plan_x_passes(n, p, layers, state_kind)


def test_pass_planner_counts():
    # 3 qubit groups at n = 26 (7 + 12 + 7) -> 1 + 2p fused passes
    assert _plan(26, 10) == 21
    assert _plan(26, 1) == 3
    # n = 13..22: two groups -> p + 1 passes (n = 22: the state stays in L2, so a
    # 10-target group with 4-amplitude runs costs nothing extra)
    assert _plan(16, 4) == 5
    assert _plan(22, 10) == 11
    # complex64 halves the bytes per amplitude: n = 23 is still L2-resident
    assert _plan(23, 10, _lib.STATE_C64) == 11
    assert _plan(23, 10) == 21
    # n = 34 local 31: 12 + 19 high targets; chunks of <= 10 would leave runs of
    # 4-8 amplitudes (64-128 B), so the cost model takes 3 high chunks of 6-7
    # targets (runs of >= 32 amplitudes) -> 4 groups, 1 + 3p passes
    assert _plan(31, 10) == 31
    assert _plan(31, 10, _lib.STATE_C64) == 31
    assert _plan(12, 4) == 1  # resident


def _plan_sharded(nl, k, p):
    import ctypes

    layers = (_lib.FqLayer * p)(*[_lib.FqLayer(0.1, 0.2, 1, 0, nl + k) for _ in range(p)])
    gp = ctypes.c_int()
    total = _lib.load().fq_plan_sharded_passes(nl, k, p, layers, ctypes.byref(gp))
    return total, gp.value


def test_sharded_planner_counts():
    # weak scaling at 2^26 amplitudes per GPU (n = 27..29 on 2..8 GPUs): the same
    # 3 groups as one GPU, the global qubits inside the group that is a fusion
    # point every other layer -> 1 + 2p passes of which p/2 span the shards
    for k in (1, 2, 3):
        assert _plan_sharded(26, k, 10) == (21, 5)
    # n = 34 on 8 GPUs (n_local 31): 4 groups -> 1 + 3p passes, 5 spanning
    assert _plan_sharded(31, 3, 10) == (31, 5)
    assert _plan_sharded(31, 3, 1) == (4, 1)
    assert _plan_sharded(11, 1, 2) == (-1, 0)  # shards need >= 12 local qubits


# ------------------------------------------------------------------ host mirror of the reference
def test_term_validation():
    assert Term(1.0, (3, 1)).support == (1, 3)
    with pytest.raises(ValueError, match="duplicate"):
        Term(1.0, (1, 1))
    with pytest.raises(ValueError, match="negative"):
        Term(1.0, (-1,))
    with pytest.raises(ValueError, match="does not fit"):
        TermPolynomial(2, (Term(1.0, (2,)),))
    assert Term(1.0, (0, 3)).mask == 9


def test_labs_and_maxcut_match_oracle_generators():
    for n in (2, 3, 7, 12, 26):
        ours = [(t.weight, t.support) for t in labs_terms(n).terms]
        assert ours == O.labs_terms(n)
    assert len(labs_terms(26).terms) == 1378
    assert len(labs_terms(34).terms) == 3128
    tri = maxcut_terms(triangle_graph())
    assert [(t.weight, t.support) for t in tri.terms] == [(0.5, (0, 1)), (0.5, (0, 2)), (0.5, (1, 2)), (-1.5, ())]


def test_dyadic_detection():
    iw, s, tot = _dyadic(np.array([2.0, 1.0, -3.0]))
    assert s == 0 and list(iw) == [2, 1, -3] and tot == 6
    iw, s, tot = _dyadic(np.array([0.5, 0.5, -1.5]))
    assert s == 1 and list(iw) == [1, 1, -3]
    iw, s, tot = _dyadic(np.array([0.1]))
    assert iw is None
    ta = term_arrays(portfolio_terms(8))
    assert ta.iweights is None  # float weights -> sequential f64 kernel


def test_compact_costs_host_format(golden):
    for name in ("labs12", "labs14", "cubic12"):
        cc = compact_costs(golden[f"diag/{name}"])
        np.testing.assert_array_equal(cc.values, golden[f"compact/{name}/values"])
        assert (cc.scale, cc.offset) == tuple(golden[f"compact/{name}/scale_offset"])
        np.testing.assert_array_equal(cc.decode(), golden[f"diag/{name}"])
    with pytest.raises(CompactRangeError):
        compact_costs(np.array([0.0, 1.0, np.pi, 70000.0]))


def test_terms_json_round_trip(tmp_path):
    poly = labs_terms(6)
    p = tmp_path / "t.json"
    save_terms(poly, str(p))
    assert load_terms(str(p)) == poly


def test_params_and_mixers():
    with pytest.raises(ValueError, match="gammas"):
        QaoaParams((0.1,), (0.1, 0.2))
    assert QaoaParams.from_flat(QaoaParams((0.1, 0.2), (0.3, 0.4)).to_flat()) == QaoaParams((0.1, 0.2), (0.3, 0.4))
    with pytest.raises(ValueError, match="odd"):
        QaoaParams.from_flat([1.0, 2.0, 3.0])
    assert ring_edges(5) == [(0, 1), (2, 3), (1, 2), (3, 4), (4, 0)]
    assert complete_edges(3) == [(0, 1), (0, 2), (1, 2)]
    with pytest.raises(ValueError, match="unknown"):
        Mixer("zz")
    with pytest.raises(ValueError, match="factory"):
        Mixer("custom")
    assert Mixer.parse("xy-ring").preserves_hamming_weight
    with pytest.raises(ValueError, match="special unitary"):
        SU2(1.0, 1.0)
    np.testing.assert_allclose(SU2.rx(0.3).matrix(), [[np.cos(0.3), -1j * np.sin(0.3)],
                                                      [-1j * np.sin(0.3), np.cos(0.3)]])


def test_graph_validation():
    with pytest.raises(ValueError, match="duplicate"):
        Graph.from_edges(3, [(0, 1), (1, 0)])
    with pytest.raises(ValueError, match="self-loop"):
        Graph.from_edges(3, [(1, 1)])
    edges = [tuple(map(int, l.split())) for l in open(os.path.join(ROOT, "tests", "golden", "maxcut26.edges"))
             if not l.startswith("#")]
    g = Graph.from_edges(26, edges)
    assert len(g.edges) == 39 and len(maxcut_terms(g).terms) == 40


def test_xy_planner_and_host_program_without_gpu():
    """The tiled-XY scheduler and the whole host side of fq_qaoa_evolve run on
    CPU up to the first launch (which must fail cleanly: no device)."""
    import ctypes

    lib = _lib.load()
    assert lib.fq_plan_xy_passes(12, 1, None) == 1  # on chip
    assert lib.fq_plan_xy_passes(26, 1, None) <= 5  # ring: 26 gates in a handful of passes
    rounds = ctypes.c_int()
    assert lib.fq_plan_xy_passes(26, 2, ctypes.byref(rounds)) <= 40  # complete: 325 gates
    assert rounds.value <= 160  # 153 measured: 325 gates, incl. the load/store re-layout rounds
    for n in (13, 20, 26):
        for mixer in (1, 2):
            lay = (_lib.FqLayer * 2)(_lib.FqLayer(0.1, 0.2, 1, 0, n), _lib.FqLayer(0.3, 0.4, 1, 0, n))
            d = _lib.FqEvolveDesc()
            d.psi, d.n, d.cost_kind, d.costs, d.mixer = 0x1000, n, 0, 0x2000, mixer
            d.n_layers, d.layers, d.scratch = 2, lay, 0x3000
            assert lib.fq_qaoa_evolve(ctypes.byref(d), None) == _lib.FQ_ERR_CUDA


def test_sharded_cost_consensus():
    from paper_2309_04841_b200.distributed import cost_consensus

    # two uint16 shards on one scale: common origin = global minimum, levels = union range
    a = (True, True, 0.5, -3.0, 10.0)
    b = (True, True, 0.5, -1.0, 20.0)
    assert cost_consensus([a, b], b) == (_lib.COST_U16, -3.0, 47, 4)
    assert cost_consensus([a, b], a) == (_lib.COST_U16, -3.0, 47, 0)
    # scales disagree -> float64 everywhere (kept)
    c = (True, True, 1.0, 0.0, 5.0)
    assert cost_consensus([a, c], a)[0] == _lib.COST_F64
    # union range beyond 16 bits -> float64
    d = (True, True, 1.0, 0.0, 40000.0)
    e = (True, True, 1.0, -40000.0, 0.0)
    assert cost_consensus([d, e], d)[0] == _lib.COST_F64
    # a shard without uint16 levels and another without float64: no common encoding
    with pytest.raises(MemoryError):
        cost_consensus([(False, True, 1.0, 0.0, 0.0), (True, False, 1.0, 0.0, 3.0)], a)


def test_planner_shapes_host_only():
    """The X-mixer planner runs on the host (no device): LABS n = 26 takes three
    groups [7 high, 12 low, 7 high] and 1 + 2p passes with p - 1 fused two-layer
    passes; n >= 31 takes four groups (1 + 3p); forced shapes (plan / plan_tmax)
    change the grouping.  tests/test_gpu_plans.py runs every forced shape."""
    from paper_2309_04841_b200 import _lib

    d26 = _lib.describe_x_plan(26, 10)
    groups = d26.split(" ")[0][len("groups="):].split(";")
    assert [len(g.split("/")[0].split(",")) for g in groups] == [7, 12, 7]
    passes = d26.split("passes=")[1].split(",")
    assert len(passes) == 21 and sum(p.endswith("f") for p in passes) == 9
    d34 = _lib.describe_x_plan(34, 10)
    assert len(d34.split(" ")[0].split(";")) == 4 and len(d34.split("passes=")[1].split(",")) == 31
    try:
        _lib.call("fq_set_option", b"plan", 0)
        _lib.call("fq_set_option", b"plan_tmax", 4)
        forced = _lib.describe_x_plan(26, 10)
        assert forced != d26
        assert all(len(g.split("/")[0].split(",")) <= 12 for g in forced.split(" ")[0][7:].split(";"))
    finally:
        _lib.call("fq_set_option", b"plan", -1)
        _lib.call("fq_set_option", b"plan_tmax", 0)
    assert _lib.describe_x_plan(26, 10) == d26
    # sharded register (k global qubits): the global qubits share one group
    d = _lib.describe_x_plan(34, 4, k=3)
    assert any({"31", "32", "33"} <= set(g.split("/")[0].split(",")) for g in d.split(" ")[0][7:].split(";"))


def test_round2_options_and_n30_plan_host_only():
    """Run-time options of this round's kernel paths are accepted with their ranges
    (lane butterflies, cost L2 policy, shared cost tile) and rejected outside them;
    LABS n = 30 plans three groups with 9-target high groups (the lane-butterfly
    shape, K_LANE3) and 21 passes for p = 10."""
    from paper_2309_04841_b200 import _lib

    for name, good, bad in ((b"lane3", (0, 1), 2), (b"cost_l2", (-1, 0, 1), 2), (b"cost_stage", (0, 1), -1)):
        for v in good:
            _lib.call("fq_set_option", name, v)
        with pytest.raises(ValueError):
            _lib.call("fq_set_option", name, bad)
    _lib.call("fq_set_option", b"lane3", 1)
    _lib.call("fq_set_option", b"cost_l2", -1)
    _lib.call("fq_set_option", b"cost_stage", 1)
    d30 = _lib.describe_x_plan(30, 10)
    groups = d30.split(" ")[0][len("groups="):].split(";")
    assert sorted(len(g.split("/")[0].split(",")) for g in groups) == [9, 9, 12]
    assert len(d30.split("passes=")[1].split(",")) == 21


def test_fq_options_env_applied_at_load():
    """FQ_OPTIONS="name=value,..." is applied when the library is loaded (A/B runs of
    the suite under a kernel variant) and a bad entry fails loudly."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = "from paper_2309_04841_b200 import _lib; _lib.load(); print('loaded')"
    env = dict(os.environ, FQ_OPTIONS="lane3=0,cost_stage=0")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "loaded" in out.stdout, out.stderr
    env = dict(os.environ, FQ_OPTIONS="no_such_option=1")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert out.returncode != 0 and "FQ_OPTIONS" in out.stderr
