"""Cost-model balancing (north_star "predicted atom/edge cost").

The reference balances on atom counts (S/scheduler.cpp:62-158) and has a cost
model only in its simulator (H/simulator.hpp:22-27, S/simulator.cpp:19-59).
lamm_plan_cost runs the same plan with a predicted per-sample cost as the key:
  * with the pure-atoms model it is the reference's plan bit for bit (checked
    against oracle/_ref in every mode);
  * with an edge-aware model its greedy assignment equals an independent Python
    restatement of greedy_assign over the cost key;
  * the fit recovers a known linear cost model.
"""
import numpy as np
import pytest

from oracle import ref_available


@pytest.fixture(scope="module")
def pk():
    import paper_2505_22208_b200 as pk
    return pk


def _greedy(keys, G, B):
    """S/scheduler.cpp:62-89 restated over an arbitrary key (LPT, cap B, ties -> lower worker)."""
    order = sorted(range(len(keys)), key=lambda e: (-keys[e], e))
    load, filled, out = [0.0] * G, [0] * G, [0] * len(keys)
    for e in order:
        pick = min((g for g in range(G) if filled[g] < B), key=lambda g: (load[g], g))
        out[e] = pick
        load[pick] += keys[e]
        filled[pick] += 1
    return out


@pytest.mark.parametrize("mode", ["balanced", "greedy_only", "naive"])
def test_atoms_model_is_the_reference_plan(pk, mode):
    atoms = pk.make_trace("lognormal", 5000, 2, 2000, mode=20.0, sigma=1.0, seed=4)
    a = pk.plan(atoms, 8, 4, 50, seed=9, mode=mode)
    c = pk.plan_cost(atoms, None, pk.CostModel(0.0, 1.0, 0.0), 8, 4, 50, seed=9, mode=mode)
    for k in ("sample", "worker", "atoms", "split", "chunk_rank", "worker_atoms"):
        assert np.array_equal(a[k], c[k]), k
    assert a["n_batches"] == c["n_batches"] and a["dropped"] == c["dropped"]
    if ref_available():
        from oracle import ref
        r = ref().plan(atoms, 8, 4, 50, seed=9, mode=mode)
        assert np.array_equal(r["sample"], c["sample"]) and np.array_equal(r["worker"], c["worker"])


def test_edge_model_matches_python_greedy(pk):
    rng = np.random.default_rng(3)
    n, G, B = 4096, 4, 8
    atoms = rng.integers(5, 300, n)
    edges = (atoms * rng.uniform(10, 40, n)).astype(np.int64)
    cm = pk.CostModel(per_sample=3.0, per_atom=0.5, per_edge=0.02)
    cost = pk.sample_cost(atoms, edges, cm)
    assert np.array_equal(cost, (3.0 + 0.5 * atoms.astype(float)) + 0.02 * edges.astype(float))
    p = pk.plan_cost(atoms, edges, cm, G, B, 16, seed=1, mode="greedy_only")
    per = G * B
    for b in range(p["n_batches"]):
        ids = p["sample"][b * per:(b + 1) * per]
        want = np.array(_greedy(cost[ids].tolist(), G, B))
        got = p["worker"][b * per:(b + 1) * per]
        assert np.array_equal(np.sort(ids[got == 0]), np.sort(ids[want == 0]))
        assert np.array_equal(got, np.sort(got))  # worker-major emission (pack_batch)
        wc = p["worker_cost"][b * G:(b + 1) * G]
        for g in range(G):
            assert wc[g] == pytest.approx(cost[ids[got == g]].sum(), rel=1e-12)
    # the cost plan balances the cost better than the atom plan does
    pa = pk.plan(atoms, G, B, 16, seed=1, mode="greedy_only")
    wa = np.array([cost[pa["sample"][b * per:(b + 1) * per][pa["worker"][b * per:(b + 1) * per] == g]].sum()
                   for b in range(pa["n_batches"]) for g in range(G)]).reshape(-1, G)
    assert p["cost_imbalance_mean"] <= float(np.mean(wa.max(1) / wa.mean(1))) + 1e-12


def test_cost_model_rejects_bad_input(pk):
    with pytest.raises(pk.InputError):
        pk.sample_cost(np.array([3, 4]), None, pk.CostModel(0.0, 1.0, 0.5))  # per_edge without edges
    with pytest.raises(pk.InputError):
        pk.sample_cost(np.array([3, 4]), None, pk.CostModel(-10.0, 1.0, 0.0))  # non-positive cost


def test_fit_recovers_linear_model(pk):
    rng = np.random.default_rng(0)
    atoms = rng.integers(500, 3000, 64)
    edges = atoms * rng.integers(12, 45, 64)
    t = 0.12 + 2e-5 * atoms + 3e-6 * edges
    cm, t0, r2 = pk.fit_cost_model(atoms, edges, t)
    assert t0 == pytest.approx(0.12, rel=1e-6) and cm.per_atom == pytest.approx(2e-5, rel=1e-6)
    assert cm.per_edge == pytest.approx(3e-6, rel=1e-6) and r2 > 0.999999


@pytest.mark.parametrize("mode", ["balanced", "naive"])
def test_simulate_bit_exact_with_reference(pk, mode):
    """simulator::simulate (S/simulator.cpp:19-59) natively: step times, idle,
    realloc events, per-worker idle and totals equal the reference's, bit for bit."""
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle import ref
    atoms = pk.make_trace("lognormal", 20000, 2, 2000, mode=20.0, sigma=1.0, seed=7)
    sch = pk.plan(atoms, 8, 4, 100, seed=3, mode=mode)
    cost = (0.004, 2e-5, 0.003, 0.05)
    got = pk.simulate(sch, *cost)
    G, nb = 8, sch["n_batches"]
    want = ref().simulate(sch["worker_atoms"], nb, G, 32, cost)
    for k in ("step_time", "step_idle", "step_max_atoms", "worker_idle"):
        assert np.array_equal(np.asarray(got[k]).view(np.uint64) if got[k].dtype == np.float64 else got[k],
                              np.asarray(want[k]).view(np.uint64) if want[k].dtype == np.float64 else want[k]), k
    assert np.array_equal(got["step_realloc"], want["step_realloc"])
    assert got["total_s"] == want["totals"][0] and got["throughput_samples_per_s"] == want["totals"][1]
    assert got["realloc_events"] == want["totals"][2] and got["samples"] == want["totals"][3]


def test_simulate_with_predicted_worker_cost(pk):
    rng = np.random.default_rng(1)
    atoms = rng.integers(10, 400, 2048)
    edges = atoms * rng.integers(10, 40, 2048)
    cm = pk.CostModel(0.0, 1e-6, 2e-7)
    p = pk.plan_cost(atoms, edges, cm, 4, 8, 8, seed=2, mode="balanced")
    s = pk.simulate(p, alpha_s=0.0, beta_s_per_atom=1e-9, gamma_s=0.0, delta_s=0.0, worker_cost=p["worker_cost"])
    wc = p["worker_cost"].reshape(-1, 4)
    assert np.allclose(s["step_time"], wc.max(1), rtol=0, atol=0)
    assert s["step_idle"] == pytest.approx((wc.max(1, keepdims=True) - wc).sum(1))
