"""Pin oracle/torch_ref.py (the torch restatement the full-shape GPU parity tests use)
against oracle/backward_ref.py in fp64 on the CPU, every variant, to 1e-10."""
import numpy as np
import pytest
import torch

from oracle import backward_ref as B
from oracle import routing_ref as R
from oracle import torch_ref as TR

VARIANTS = [
    dict(score="softmax", variant="standard", cf=None),
    dict(score="softmax", variant="mem_efficient", cf=None),
    dict(score="sigmoid", variant="standard", cf=None),
    dict(score="sigmoid", variant="mem_efficient", cf=None),
    dict(score="softmax", variant="standard", cf=(0.6, True)),
    dict(score="sigmoid", variant="standard", cf=(0.5, False)),
    dict(score="softmax", variant="standard", cf=None, gated=False),
    dict(score="sigmoid", variant="standard", cf=None, shared=True),
]


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("v", VARIANTS, ids=lambda v: "-".join(f"{k}={v[k]}" for k in v))
def test_torch_ref_matches_backward_ref(v):
    rng = np.random.default_rng(7)
    T, E, K, h, m = 37, 6, 2, 12, 10
    x = rng.standard_normal((T, h))
    w_r = rng.standard_normal((h, E)) * 0.5
    # a hot expert so capacity drops happen (and some tokens lose every selection)
    x[:, 0] = 1.0
    w_r[0, 1] += 2.0
    gated = v.get("gated", True)
    up = rng.standard_normal((E, m, h)) * h ** -0.5
    gate = rng.standard_normal((E, m, h)) * h ** -0.5 if gated else None
    w2 = rng.standard_normal((E, h, m)) * m ** -0.5
    dy = rng.standard_normal((T, h))
    params = R.ExpertParams(w1=list(up), w2=list(w2), gate=list(gate) if gated else None)
    ref = B.moe_forward_backward(x, w_r, params, dy, score=v["score"], top_k=K, coeff=1e-2,
                                 variant=v["variant"], capacity=v["cf"])
    dec = ref["decision"]
    idx = np.sort(np.argsort(~dec.routing_map, axis=1, kind="stable")[:, :K], axis=1)
    cap = None
    if v["cf"] is not None:
        cap = R.expert_capacity(v["cf"][0], T, K, E)
        assert dec.dropped.any()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    shared = None
    y_ref, dx_ref = ref["y"], ref["dx"]
    if v.get("shared"):
        ms = 8
        sg = rng.standard_normal((ms, h)) * h ** -0.5
        su = rng.standard_normal((ms, h)) * h ** -0.5
        sw2 = rng.standard_normal((h, ms)) * ms ** -0.5
        sp = R.ExpertParams(w1=[su], w2=[sw2], gate=[sg])
        rs = B.moe_forward_backward(x, np.zeros((h, 1)), sp, dy, top_k=1, coeff=0.0)
        y_ref = y_ref + rs["y"]
        dx_ref = dx_ref + rs["dx"]
        shared = (t(sg), t(su), t(sw2))
    got = TR.moe_forward_backward(t(x), t(w_r), t(gate) if gated else None, t(up), t(w2),
                                  t(dy), t(idx), score=v["score"], coeff=1e-2,
                                  variant=v["variant"], capacity=cap, shared=shared)
    tol = 1e-10
    assert rel(got["y"], y_ref) < tol
    assert abs(got["aux"] - ref["aux"]) < 1e-14
    assert rel(got["dx"], dx_ref) < tol
    assert rel(got["dw_r"], ref["dw_r"]) < tol
    for e in range(E):
        if got["dup"][e] is None:
            assert not np.any(ref["dw1"][e])
            continue
        assert rel(got["dup"][e], ref["dw1"][e]) < tol
        assert rel(got["dw2"][e], ref["dw2"][e]) < tol
        if gated:
            assert rel(got["dgate"][e], ref["dgate"][e]) < tol
    if shared is not None:
        assert rel(got["shared"]["dgate"], rs["dgate"][0]) < tol
        assert rel(got["shared"]["dup"], rs["dw1"][0]) < tol
        assert rel(got["shared"]["dw2"], rs["dw2"][0]) < tol
