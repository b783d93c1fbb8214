"""Pin the CPU oracle (oracle/routing_ref.py, oracle/backward_ref.py).

1. Against golden vectors produced by the reference itself
   (tests/golden/make_golden.py -> routing_golden.npz).
2. Against the reference's own hand goldens (reference pkg/tests/test_routing.py).
3. The backward restatement against central finite differences of the oracle
   forward, and against the reference aux_loss_grad_wr.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle import backward_ref as B
from oracle import routing_ref as R

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "routing_golden.npz")


def close(a, b, rtol=1e-12, atol=1e-12):
    np.testing.assert_allclose(np.asarray(a), np.asarray(b), rtol=rtol, atol=atol)


def exact(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.array_equal(a, b)


def params(prefix="params", e=6, gated=True):
    return R.ExpertParams(
        w1=[GOLD[f"{prefix}/w1/{i}"] for i in range(e)],
        w2=[GOLD[f"{prefix}/w2/{i}"] for i in range(e)],
        gate=[GOLD[f"{prefix}/gate/{i}"] for i in range(e)] if gated else None,
    )


def check_decision(prefix, d):
    exact(d.routing_map, GOLD[f"{prefix}/routing_map"])
    exact(d.counts, GOLD[f"{prefix}/counts"])
    exact(d.effective_counts(), GOLD[f"{prefix}/effective_counts"])
    close(d.probs, GOLD[f"{prefix}/probs"])
    close(d.scores, GOLD[f"{prefix}/scores"])
    if f"{prefix}/dropped" in GOLD:
        exact(d.dropped, GOLD[f"{prefix}/dropped"])
    if f"{prefix}/phantom_rows" in GOLD:
        exact(d.phantom_rows, GOLD[f"{prefix}/phantom_rows"])


CASES = {
    "softmax_k2": dict(score="softmax", top_k=2),
    "sigmoid_k3": dict(score="sigmoid", top_k=3),
    "softmax_k2_bias": dict(score="softmax", top_k=2, bias=True),
    "sigmoid_k1_bias": dict(score="sigmoid", top_k=1, bias=True),
}


@pytest.mark.parametrize("name", list(CASES))
def test_route_permute_combine_vs_reference(name):
    kw = dict(CASES[name])
    x, w_r = GOLD["x"], GOLD["w_r"]
    if kw.pop("bias", False):
        kw["selection_bias"] = GOLD["bias"]
    d = R.route(x, w_r, **kw)
    check_decision(f"route/{name}", d)
    close(R.aux_loss(d, 0.01), GOLD[f"aux/{name}"])
    rows, rmap = R.permute(x, d)
    exact(rmap, GOLD[f"permute/{name}/row_id_map"])
    exact(rows, GOLD[f"permute/{name}/rows"])
    exact(R.unpermute_sum(rows, rmap, x.shape[0]), GOLD[f"unpermute/{name}"])
    for tag, p in (("gated", params()), ("plain", params(gated=False))):
        close(R.combine_standard(x, d, p), GOLD[f"combine_standard/{name}/{tag}"], 1e-10, 1e-10)
        close(R.combine_mem_efficient(x, d, p), GOLD[f"combine_mem_efficient/{name}/{tag}"],
              1e-10, 1e-10)


def test_ties_lowest_index():
    d = R.route(np.zeros((3, 5)), np.eye(5), top_k=3)
    check_decision("route/ties", d)


def test_aux_grad_and_bias_update():
    close(R.aux_loss_grad_wr(GOLD["x"], GOLD["w_r"], 2, 0.37), GOLD["aux_grad/k2"])
    close(R.auxfree_bias_update(GOLD["auxfree/counts"], GOLD["bias"], 0.05), GOLD["auxfree/out"])


@pytest.mark.parametrize("pad", [False, True])
@pytest.mark.parametrize("cf", [1.0, 0.5, 1.25])
def test_capacity_vs_reference(cf, pad):
    x = GOLD["x"]
    d = R.route(GOLD["cap/logits"], np.eye(6), top_k=2)
    c = R.apply_capacity(d, cf, pad=pad)
    key = f"cap/cf{cf}_pad{int(pad)}"
    check_decision(key, c)
    rows, rmap = R.permute(x, c)
    exact(rmap, GOLD[f"{key}/row_id_map"])
    exact(rows, GOLD[f"{key}/rows"])
    close(R.moe_output_with_residual(x, c, params()), GOLD[f"{key}/residual_out"], 1e-10, 1e-10)


def test_expert_capacity_values():
    got = [R.expert_capacity(1.0, 128, 2, 8), R.expert_capacity(1.0, 16384, 2, 8),
           R.expert_capacity(1.0, 32768, 8, 128), R.expert_capacity(1.0, 4096, 8, 256),
           R.expert_capacity(0.7, 999, 3, 7)]
    exact(got, GOLD["cap/expert_capacity"])
    assert got[:4] == [32, 4096, 2048, 128]


@pytest.mark.parametrize("mult", [4, 8, 16])
def test_routing_map_pad_vs_reference(mult):
    d = R.route(GOLD["x"], GOLD["w_r"], top_k=2)
    pd = R.routing_map_pad(d, mult)
    check_decision(f"pad/m{mult}", pd)
    exact(R.permute(GOLD["x"], pd)[1], GOLD[f"pad/m{mult}/row_id_map"])


def test_latent_and_shared_vs_reference():
    x, w_r = GOLD["x"], GOLD["w_r"]
    d = R.route(x, w_r, top_k=2)
    experts = params("latent/experts")
    shared = R.ExpertParams(w1=[GOLD["latent/shared/w1"]], w2=[GOLD["latent/shared/w2"]],
                            gate=[GOLD["latent/shared/gate"]])
    close(R.latent_moe_forward(x, GOLD["latent/w_down"], GOLD["latent/w_up"], experts, d, shared),
          GOLD["latent/out"], 1e-10, 1e-10)
    eye = np.eye(x.shape[1])
    close(R.latent_moe_forward(x, eye, eye, params(), d, shared),
          GOLD["latent/identity_shared_out"], 1e-10, 1e-10)


def test_upcycle_vs_reference():
    up, wr0 = R.upcycle(GOLD["upcycle/in_w1"], GOLD["upcycle/in_w2"], 2, 2,
                        dense_gate=GOLD["upcycle/in_gate"])
    for i in range(4):
        exact(up.w1[i], GOLD[f"upcycle/w1/{i}"])
        exact(up.w2[i], GOLD[f"upcycle/w2/{i}"])
        exact(up.gate[i], GOLD[f"upcycle/gate/{i}"])
    exact(wr0, GOLD["upcycle/w_r"])
    with pytest.raises(ValueError, match="divisible"):
        R.upcycle(np.zeros((9, 4)), np.zeros((4, 9)), 2, 2)


def test_a2a_volume_vs_reference():
    for tok, k, hid, ep, want in GOLD["a2a/table"]:
        assert R.a2a_send_volume(int(tok), int(k), int(hid), int(ep), 2) == want
    assert R.a2a_send_volume(4096, 8, 7168, 64, 2) == 462_422_016  # reference test_perf.py:37-38


# ---- the reference's own hand goldens (pkg/tests/test_routing.py) -----------

def from_logits(logits, k, score="softmax"):
    logits = np.asarray(logits, dtype=np.float64)
    return R.route(logits, np.eye(logits.shape[1]), score=score, top_k=k)


def test_hand_goldens():
    d = from_logits([[2.0, 1.0, 0.0, -1.0]], 2)                     # :42-47
    assert set(np.flatnonzero(d.routing_map[0])) == {0, 1}
    assert d.probs[0, 0] == pytest.approx(0.6439, abs=2e-4)
    assert d.probs[0, 1] == pytest.approx(0.2369, abs=2e-4)
    assert np.allclose(from_logits(np.zeros((3, 5)), 5).probs, 0.2)  # :49-52
    s = from_logits(np.random.default_rng(0).normal(size=(7, 6)), 2, "sigmoid").scores
    assert np.allclose(s.sum(1), 1.0)                                # :55-58
    assert list(np.flatnonzero(from_logits([[1.0, 1.0, 1.0]], 2).routing_map[0])) == [0, 1]
    with pytest.raises(ValueError, match="finite"):                  # :66-68
        R.route(np.array([[np.inf, 0.0]]), np.eye(2), top_k=1)
    _, rmap = R.permute(np.arange(6.0).reshape(3, 2), from_logits(np.zeros((3, 2)), 2))
    assert list(rmap) == [0, 1, 2, 0, 1, 2]                           # :189-194
    assert R.expert_capacity(1.0, 128, 2, 8) == 32                   # :261-262
    scores = np.full((4, 4), 0.25)
    routing = np.eye(4, dtype=bool)
    d = R.RoutingDecision(probs=np.where(routing, 0.25, 0), routing_map=routing,
                          counts=routing.sum(0), scores=scores)
    assert R.aux_loss(d, 0.01) == pytest.approx(0.01)                # :82-88
    with pytest.raises(ValueError, match="filler"):                  # :434-437
        R.routing_map_pad(from_logits(np.random.default_rng(21).normal(size=(5, 2)), 1), 128,
                          num_filler_tokens=1)


def test_dropless_conservation_and_equivalence():
    """reference test_acceptance.py:215-239 style: 200 random instances."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        t = int(rng.integers(1, 65))
        e = int(rng.integers(2, 17))
        k = int(rng.integers(1, min(6, e) + 1))
        h, m = int(rng.integers(2, 9)), int(rng.integers(2, 17))
        x = rng.normal(size=(t, h))
        p = R.ExpertParams(w1=[rng.normal(size=(m, h)) for _ in range(e)],
                           w2=[rng.normal(size=(h, m)) for _ in range(e)])
        d = R.route(x, rng.normal(size=(h, e)), top_k=k)
        assert int(d.counts.sum()) == t * k
        a = R.combine_standard(x, d, p)
        b = R.combine_mem_efficient(x, d, p)
        assert np.abs(a - b).max() <= 1e-6 * max(np.abs(a).max(), 1e-30)


# ---- backward restatement pinned by finite differences ----------------------

def _fd_case(seed, score, variant, gated, capacity, bias):
    rng = np.random.default_rng(seed)
    t, h, e, k, m = 6, 5, 4, 2, 7
    x = rng.normal(size=(t, h))
    w_r = rng.normal(size=(h, e))
    p = R.ExpertParams(w1=[rng.normal(size=(m, h)) for _ in range(e)],
                       w2=[rng.normal(size=(h, m)) for _ in range(e)],
                       gate=[rng.normal(size=(m, h)) for _ in range(e)] if gated else None)
    dy = rng.normal(size=(t, h))
    sb = rng.normal(size=e) * 0.01 if bias else None
    kw = dict(score=score, top_k=k, coeff=0.3, variant=variant, capacity=capacity,
              selection_bias=sb)
    return x, w_r, p, dy, kw


@pytest.mark.parametrize("score", ["softmax", "sigmoid"])
@pytest.mark.parametrize("variant", ["standard", "mem_efficient"])
@pytest.mark.parametrize("gated", [True, False])
@pytest.mark.parametrize("capacity", [None, (0.5, True)])
def test_backward_matches_finite_differences(score, variant, gated, capacity):
    x, w_r, p, dy, kw = _fd_case(11, score, variant, gated, capacity, bias=False)
    g = B.moe_forward_backward(x, w_r, p, dy, **kw)
    # freeze the routing decision: selection is piecewise constant
    dec = g["decision"]
    eps = 1e-6

    def L(x_=x, w_r_=w_r, p_=p):
        # recompute probs/scores with the frozen selection
        d = R.route(x_, w_r_, score=score, top_k=2)
        d = R.RoutingDecision(probs=np.where(dec.routing_map, d.scores, 0.0),
                              routing_map=dec.routing_map, counts=dec.counts, scores=d.scores,
                              dropped=dec.dropped, phantom_rows=dec.phantom_rows)
        kk = dict(kw)
        kk.pop("capacity")
        kk.pop("selection_bias")
        return B.loss(x_, w_r_, p_, dy, decision=d, **kk)

    def fd(arr, setter):
        out = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            a1, a2 = arr.copy(), arr.copy()
            a1[i] += eps
            a2[i] -= eps
            out[i] = (setter(a1) - setter(a2)) / (2 * eps)
        return out

    def rel(a, b):
        return np.abs(a - b).max() / max(np.abs(b).max(), 1e-12)

    assert rel(g["dx"], fd(x, lambda a: L(x_=a))) < 1e-6
    assert rel(g["dw_r"], fd(w_r, lambda a: L(w_r_=a))) < 1e-6
    e0 = 1
    w1 = p.w1[e0]

    def with_w1(a):
        return L(p_=R.ExpertParams(w1=[a if i == e0 else w for i, w in enumerate(p.w1)],
                                   w2=p.w2, gate=p.gate))

    assert rel(g["dw1"][e0], fd(w1, with_w1)) < 1e-6

    def with_w2(a):
        return L(p_=R.ExpertParams(w1=p.w1, w2=[a if i == e0 else w for i, w in enumerate(p.w2)],
                                   gate=p.gate))

    assert rel(g["dw2"][e0], fd(p.w2[e0], with_w2)) < 1e-6
    if gated:
        def with_g(a):
            return L(p_=R.ExpertParams(w1=p.w1, w2=p.w2,
                                       gate=[a if i == e0 else w for i, w in enumerate(p.gate)]))

        assert rel(g["dgate"][e0], fd(p.gate[e0], with_g)) < 1e-6


def test_backward_aux_part_matches_reference_grad():
    """With dY = 0 the W_r gradient is exactly the reference aux_loss_grad_wr."""
    x, w_r = GOLD["x"], GOLD["w_r"]
    p = params()
    g = B.moe_forward_backward(x, w_r, p, np.zeros_like(x), score="softmax", top_k=2, coeff=0.37)
    close(g["dw_r"], GOLD["aux_grad/k2"], 1e-10, 1e-12)
