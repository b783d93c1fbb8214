"""The drop-in function API (paper_2603_07685_b200.routing) on the GPU, written like the
reference's own suite (reference pkg/tests/test_routing.py) with the device tolerances
stated: maps / indices / counts bit-exact; float outputs within bf16 tolerance."""
import numpy as np
import pytest
import torch

from oracle import routing_ref as R

pytestmark = pytest.mark.gpu

from paper_2603_07685_b200 import routing as G  # noqa: E402

TOL = 1e-2  # relFro for bf16 storage / fp32 accumulate


@pytest.fixture(autouse=True, scope="module")
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def bf(a):
    """Round to bf16 once and return fp64 (what the oracle is fed)."""
    return torch.as_tensor(np.asarray(a, dtype=np.float64)).to(torch.bfloat16).double().numpy()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def from_logits(logits, k, score="softmax"):
    logits = np.asarray(logits, dtype=np.float64)
    return G.route(logits, np.eye(logits.shape[1]), score=score, top_k=k)


def rparams(rng, e, h, m, gated=False):
    return G.ExpertParams(
        w1=[bf(rng.normal(size=(m, h)) / np.sqrt(h)) for _ in range(e)],
        w2=[bf(rng.normal(size=(h, m)) / np.sqrt(m)) for _ in range(e)],
        gate=[bf(rng.normal(size=(m, h)) / np.sqrt(h)) for _ in range(e)] if gated else None)


def oparams(p):
    return R.ExpertParams(w1=p.w1, w2=p.w2, gate=p.gate)


# -- route (reference test_routing.py:42-77) ------------------------------------

def test_route_softmax_example():
    d = from_logits([[2.0, 1.0, 0.0, -1.0]], k=2)
    assert set(np.nonzero(d.routing_map[0])[0]) == {0, 1}
    assert d.probs[0, 0] == pytest.approx(0.6439, abs=2e-4)
    assert d.probs[0, 1] == pytest.approx(0.2369, abs=2e-4)


def test_route_uniform_sigmoid_ties_nonfinite():
    d = from_logits(np.zeros((3, 5)), k=5)
    assert np.allclose(d.probs, 0.2) and d.routing_map.all()
    d = from_logits(np.random.default_rng(0).normal(size=(7, 6)), k=2, score="sigmoid")
    assert np.allclose(d.scores.sum(axis=1), 1.0, atol=1e-6)
    assert list(np.nonzero(from_logits([[1.0, 1.0, 1.0]], k=2).routing_map[0])[0]) == [0, 1]
    with pytest.raises(ValueError, match="finite"):
        G.route(np.array([[np.inf, 0.0]]), np.eye(2), top_k=1)
    with pytest.raises(ValueError, match="exceeds"):
        G.route(np.zeros((2, 3)), np.eye(3), top_k=4)


def test_dropless_conservation_and_bit_exact_selection():
    rng = np.random.default_rng(1)
    for _ in range(50):
        t, e = int(rng.integers(1, 64)), int(rng.integers(2, 16))
        k = int(rng.integers(1, e + 1))
        logits = bf(rng.normal(size=(t, e)))
        d = from_logits(logits, k)
        assert int(d.counts.sum()) == t * k
        ref = R.route(logits, np.eye(e), top_k=k)
        assert np.array_equal(d.routing_map, ref.routing_map)
        assert np.array_equal(d.counts, ref.counts)


def test_route_vs_oracle_at_logits_boundary_with_bias():
    rng = np.random.default_rng(2)
    x, w = bf(rng.normal(size=(300, 64))), bf(rng.normal(size=(64, 16)) / 8)
    for score in ("softmax", "sigmoid"):
        d = G.route(x, w, score=score, top_k=4)
        logits = d._logits.double().cpu().numpy()
        ref = R.route(logits, np.eye(16), score=score, top_k=4)
        assert np.array_equal(d.routing_map, ref.routing_map)
        np.testing.assert_allclose(d.probs, ref.probs, rtol=1e-5, atol=1e-7)
        assert rel(logits, x @ w) < 1e-5
    bias = rng.normal(size=16) * 0.05
    d = G.route(x, w, top_k=2, selection_bias=bias)
    ref = R.route(d._logits.double().cpu().numpy(), np.eye(16), top_k=2, selection_bias=bias)
    # fp32 vs fp64 scores + bias: identical except at near-ties (reported, not hidden)
    diff_rows = np.flatnonzero((d.routing_map != ref.routing_map).any(1))
    srt = np.sort(ref.scores + bias, axis=1)[:, ::-1]
    margin = srt[:, 1] - srt[:, 2]
    assert np.all(margin[diff_rows] < 1e-6), margin[diff_rows]


# -- aux loss ---------------------------------------------------------------------

def test_aux_loss_and_grad():
    scores = np.full((4, 4), 0.25)
    routing = np.eye(4, dtype=bool)
    d = G.RoutingDecision(probs=np.where(routing, 0.25, 0), routing_map=routing,
                          counts=routing.sum(0), scores=scores)
    assert G.aux_loss(d, coeff=0.01) == pytest.approx(0.01)
    rng = np.random.default_rng(7)
    x, w = bf(rng.normal(size=(64, 12))), bf(rng.normal(size=(12, 6)))
    g = G.aux_loss_grad_wr(x, w, 2, 0.37)
    assert rel(g, R.aux_loss_grad_wr(x, w, 2, 0.37)) < 2e-2
    with pytest.raises(NotImplementedError):
        G.aux_loss_grad_wr(x, w, 2, 0.37, score="sigmoid")
    out = G.auxfree_bias_update(np.array([10, 2, 2, 2]), np.zeros(4), 0.5)
    assert out[0] == -0.5 and np.all(out[1:] == 0.5)
    with pytest.raises(ValueError, match="step"):
        G.auxfree_bias_update(np.array([1, 2]), np.zeros(2), 0.0)


# -- permutation (reference :181-204) --------------------------------------------

def test_permute_maps():
    x = np.arange(4.0).reshape(1, 4)
    p, rmap = G.permute(x, from_logits([[1.0, 0.0]], k=1))
    assert np.array_equal(p, x) and list(rmap) == [0]
    x = np.arange(6.0).reshape(3, 2)
    p, rmap = G.permute(x, from_logits(np.zeros((3, 2)), k=2))
    assert p.shape == (6, 2) and list(rmap) == [0, 1, 2, 0, 1, 2]


def test_permute_unpermute_vs_oracle():
    rng = np.random.default_rng(5)
    x = bf(rng.normal(size=(257, 24)))
    d = from_logits(bf(rng.normal(size=(257, 12))), k=3)
    ref_d = R.route(d._logits.double().cpu().numpy(), np.eye(12), top_k=3)
    rows, rmap = G.permute(x, d)
    rrows, rrmap = R.permute(x, ref_d)
    assert np.array_equal(rmap, rrmap)
    assert np.array_equal(rows, rrows)  # pure copies of bf16 values
    comb = G.unpermute_sum(rows, rmap, 257)
    assert rel(comb, 3 * x) < 1e-2


# -- combine (reference :209-256) ------------------------------------------------

@pytest.mark.parametrize("gated", [False, True])
def test_combine_standard_mem_efficient_vs_oracle(gated):
    rng = np.random.default_rng(8 + gated)
    e, h, m, t = 4, 48, 40, 200
    p = rparams(rng, e, h, m, gated)
    x = bf(rng.normal(size=(t, h)))
    d = from_logits(bf(rng.normal(size=(t, e))), k=2)
    ref_d = R.route(d._logits.double().cpu().numpy(), np.eye(e), top_k=2)
    a = G.combine_standard(x, d, p)
    b = G.combine_mem_efficient(x, d, p)
    ra = R.combine_standard(x, ref_d, oparams(p))
    assert rel(a, ra) < TOL
    assert rel(b, ra) < TOL
    assert rel(a, b) < TOL
    for i in range(e):
        assert rel(G.expert_forward(p, i, x[:17]), R.expert_forward(oparams(p), i, x[:17])) < TOL


# -- capacity (reference :261-301) -----------------------------------------------

def test_capacity_cases():
    assert G.expert_capacity(1.0, 128, 2, 8) == 32
    d = from_logits(np.tile(np.eye(4), (8, 1)), k=1)
    assert G.apply_capacity(d, 1.0).dropped.sum() == 0
    logits = np.zeros((12, 4))
    logits[:, 0] = 10.0
    capped = G.apply_capacity(from_logits(logits, k=1), 1.0)
    assert capped.dropped.sum() == 12 - 12 // 4
    d = from_logits(bf(np.random.default_rng(0).normal(size=(16, 4))), k=2)
    capped = G.apply_capacity(d, 1.0, pad=True)
    assert np.all(capped.effective_counts() == G.expert_capacity(1.0, 16, 2, 4))
    with pytest.raises(ValueError, match="capacity_factor"):
        G.apply_capacity(d, 0.0)


@pytest.mark.parametrize("cf,pad", [(1.0, False), (0.5, True), (1.25, True)])
def test_capacity_maps_and_residual_vs_oracle(cf, pad):
    rng = np.random.default_rng(12)
    e, h, m, t = 6, 32, 48, 180
    logits = bf(rng.normal(size=(t, e)) + np.array([2.0, 1.0, 0.0, -1.0, -1.0, -2.0]))
    d = from_logits(logits, k=2)
    c = G.apply_capacity(d, cf, pad=pad)
    rc = R.apply_capacity(R.route(logits, np.eye(e), top_k=2), cf, pad=pad)
    assert np.array_equal(c.dropped, rc.dropped)
    assert np.array_equal(c.effective_counts(), rc.effective_counts())
    x = bf(rng.normal(size=(t, h)))
    rows, rmap = G.permute(x, c)
    rrows, rrmap = R.permute(x, rc)
    assert np.array_equal(rmap, rrmap) and np.array_equal(rows, rrows)
    p = rparams(rng, e, h, m, gated=True)
    y = G.moe_output_with_residual(x, c, p)
    ry = R.moe_output_with_residual(x, rc, oparams(p))
    assert rel(y, ry) < TOL
    dead = ~(rc.routing_map & ~rc.dropped).any(1)
    if dead.any():
        assert rel(y[dead], x[dead] + R.combine_standard(x, rc, oparams(p))[dead]) < TOL


# -- latent / shared, routing-map pad, upcycling ----------------------------------

def test_latent_and_shared():
    rng = np.random.default_rng(13)
    h, lat, e, m, t = 24, 16, 3, 32, 40
    x = bf(rng.normal(size=(t, h)))
    d = from_logits(bf(rng.normal(size=(t, e))), k=2)
    ref_d = R.route(d._logits.double().cpu().numpy(), np.eye(e), top_k=2)
    ex = rparams(rng, e, lat, m, gated=True)
    sh = rparams(rng, 1, h, m, gated=True)
    wd, wu = bf(rng.normal(size=(lat, h)) / 5), bf(rng.normal(size=(h, lat)) / 4)
    out = G.latent_moe_forward(x, wd, wu, ex, d, sh)
    ref = R.latent_moe_forward(x, wd, wu, oparams(ex), ref_d, oparams(sh))
    assert rel(out, ref) < 2 * TOL  # two chained bf16 GEMM roundings


def test_routing_map_pad():
    d = from_logits(bf(np.random.default_rng(19).normal(size=(8, 2))), k=1)
    assert np.all(G.routing_map_pad(d, 16).effective_counts() == 16)
    d2 = from_logits(np.tile(np.eye(2), (16, 1)), k=1)
    assert np.all(G.routing_map_pad(d2, 16).phantom_rows == 0)
    rng = np.random.default_rng(20)
    d3 = G.routing_map_pad(from_logits(bf(rng.normal(size=(11, 3))), k=2), 8)
    x = bf(rng.normal(size=(11, 4)))
    rows, rmap = G.permute(x, d3)
    assert rows.shape[0] == d3.effective_counts().sum()
    assert all(c % 8 == 0 for c in d3.effective_counts())
    assert np.all(rows[rmap == -1] == 0)
    with pytest.raises(ValueError, match="filler"):
        G.routing_map_pad(from_logits(np.random.default_rng(21).normal(size=(5, 2)), 1), 128,
                          num_filler_tokens=1)


def test_upcycle_identity():
    rng = np.random.default_rng(15)
    w1, w2, gate = (bf(rng.normal(size=(256, 64)) / 8), bf(rng.normal(size=(64, 256)) / 16),
                    bf(rng.normal(size=(256, 64)) / 8))
    p, w_r = G.upcycle(w1, w2, granularity=2, duplication=2, dense_gate=gate)
    assert p.num_experts == 4
    x = bf(rng.normal(size=(100, 64)))
    d = G.route(x, w_r, top_k=2)
    moe = G.combine_standard(x, d, p)
    g = x @ gate.T
    dense = (g / (1 + np.exp(-g)) * (x @ w1.T)) @ w2.T
    assert rel(moe, dense) < TOL
    with pytest.raises(ValueError, match="divisible"):
        G.upcycle(rng.normal(size=(9, 4)), rng.normal(size=(4, 9)), 2, 2)


def test_torch_in_torch_out():
    x = torch.randn(64, 32, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(32, 8, device="cuda", dtype=torch.bfloat16)
    d = G.route(x, w, top_k=2)
    assert isinstance(d.routing_map, torch.Tensor) and d.routing_map.is_cuda
    rows, rmap = G.permute(x, d)
    assert rows.is_cuda and rmap.dtype == torch.int64


# -- edge cases of the top-k kernel (non-finite keys, fp64 score ties) ---------

@pytest.mark.parametrize("hp", [64, 128], ids=["gemm256_path", "small_n_tc_path"])
def test_nonfinite_rows_raise_and_select_valid_experts(hp):
    """A NaN hidden row (and an inf one with a selection bias) makes route() raise the
    reference's ValueError; the kernel itself still writes K valid, distinct experts per
    token and leaves the counts consistent (no out-of-range index, no stray writes)."""
    from paper_2603_07685_b200 import ops

    E, K = 8, 2
    logits = np.random.default_rng(3).normal(size=(64, E))
    logits[5] = np.nan
    with pytest.raises(ValueError, match="finite"):
        from_logits(logits, k=K)
    bias = np.linspace(0, 0.1, E)
    inf_row = np.random.default_rng(4).normal(size=(16, E))
    inf_row[3, 2] = np.inf
    with pytest.raises(ValueError, match="finite"):
        G.route(inf_row, np.eye(E), score="sigmoid", top_k=K, selection_bias=bias)
    # kernel level: every row keeps K distinct in-range experts, counts sum to T*K
    x = torch.as_tensor(logits, dtype=torch.float32).to(torch.bfloat16).cuda()
    x = torch.nn.functional.pad(x, (0, hp - E))
    w = torch.eye(hp, E, dtype=torch.bfloat16, device="cuda")
    for bias_t in (None, torch.as_tensor(bias, dtype=torch.float32, device="cuda")):
        r = ops.router_forward(x, w, K, "softmax", bias_t)
        assert r.path == ("tc" if hp == 128 else "gemm")
        idx = r.topk_idx.cpu().numpy()
        assert idx.min() >= 0 and idx.max() < E
        assert np.all(np.diff(idx, axis=1) > 0)
        assert int(r.counts.sum()) == 64 * K
        assert int(r.status.item()) & 1
    # the device is still healthy
    d = from_logits([[2.0, 1.0, 0.0, -1.0]], k=2)
    assert set(np.nonzero(d.routing_map[0])[0]) == {0, 1}


@pytest.mark.parametrize("score,row", [
    # fp64 sigmoid saturates to exactly 1.0 from l = 36.7368: experts 1..3 tie, the oracle's
    # stable argsort takes the lowest indices (fp32-logit order would take 2 and 3)
    ("sigmoid", [0.0, 36.75, 40.0, 38.0, -1.0]),
    # fp64 exp underflows to 0 below max - 745.13: experts 1..3 tie at probability 0
    ("softmax", [0.0, -1000.0, -800.0, -896.0, -2000.0]),
])
def test_selection_ties_of_saturated_fp64_scores(score, row):
    logits = np.asarray([row], dtype=np.float64)
    d = from_logits(logits, k=2, score=score)
    ref = R.route(logits, np.eye(logits.shape[1]), score=score, top_k=2)
    assert np.array_equal(d.routing_map, ref.routing_map), (d.routing_map, ref.routing_map)
    assert list(np.nonzero(d.routing_map[0])[0]) == ([0, 1] if score == "softmax" else [1, 2])


def test_layer_check_finite_raises():
    from paper_2603_07685_b200.layer import MoEConfig, moe_forward

    cfg = MoEConfig(8, 2, 256, 256, check_finite=True)
    x = torch.randn((128, 256), device="cuda").to(torch.bfloat16)
    x[7, 3] = float("nan")
    w_r = (torch.randn((256, 8), device="cuda") / 16).to(torch.bfloat16)
    w1 = (torch.randn((8, 512, 256), device="cuda") / 16).to(torch.bfloat16)
    w2 = (torch.randn((8, 256, 256), device="cuda") / 16).to(torch.bfloat16)
    with pytest.raises(ValueError, match="finite"):
        moe_forward(x, w_r, w1, w2, cfg)
