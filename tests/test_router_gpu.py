"""Router kernels on the GPU: the small-E fused path (logits on the CUDA cores inside the
top-k kernel, E <= 16) and the tcgen05 path (larger E) against the oracle / fp64 references.

  * logits vs the fp64 product of the same bf16 values (relFro <= 1e-5, fp32 accumulate);
  * selections, counts bit-exact against routing_ref.route on the device logits;
  * probs, aux loss and its per-expert gradient vs the oracle;
  * backward: dlogits vs backward_ref's score Jacobian, dW_r = x^T dl and router dX = dl W_r^T
    vs fp64 products of the device dl (relFro <= 1e-5; dX is bf16: <= 4e-3).
"""
import numpy as np
import pytest
import torch

from oracle import routing_ref as R

pytestmark = pytest.mark.gpu

from paper_2603_07685_b200 import ops  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


CASES = [  # (T, h, E, K, score, bias)
    (1000, 4096, 8, 2, "softmax", False),     # Mixtral router shape (T not a multiple of 64)
    (333, 256, 8, 2, "sigmoid", True),
    (517, 1024, 16, 4, "softmax", True),
    (64, 512, 3, 1, "sigmoid", False),
    (1, 256, 2, 2, "softmax", False),
    (777, 512, 32, 4, "sigmoid", False),      # E > 16: tcgen05 logits path
    (600, 512, 128, 8, "softmax", True),      # Qwen3-like E
    (4096, 7168, 256, 8, "sigmoid", True),    # DeepSeek shape: small-N tiles split h over
                                              # an 8-CTA cluster (32 token tiles)
    (4096, 256, 8, 2, "softmax", False),      # BASELINE configs[0] router (h split in 4)
    (2000, 2048, 64, 6, "softmax", False),    # NPAD 64, K between the KMAX variants
]


@pytest.fixture(params=["tc", "gemm", "small"],
                ids=["small_n_tc_path", "tcgen05_256_path", "small_path"])
def router_path(request, monkeypatch):
    """tc: the default small-N tensor-core router (csrc/router_tc.cu); gemm: the round-1
    chain (logits GEMM padded to 256 + warp-per-token top-k); small: CUDA-core E <= 16."""
    monkeypatch.setattr(ops, "ROUTER_TC", request.param == "tc")
    monkeypatch.setattr(ops, "ROUTER_SMALL", request.param == "small")
    return request.param


@pytest.mark.parametrize("T,h,E,K,score,bias", CASES)
def test_router_forward_backward(T, h, E, K, score, bias, dev, router_path):
    g = torch.Generator(device=dev).manual_seed(T + E)
    x = torch.randn((T, h), device=dev, generator=g).to(torch.bfloat16)
    w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(torch.bfloat16)
    sb = (torch.rand((E,), device=dev, generator=g) * 0.05) if bias else None
    small = router_path == "small" and ops.router_small(E, h)
    r = ops.router_forward(x, w_r, K, score, sb, 1e-2, want_scores=True)
    want = {"tc": "tc", "gemm": "gemm", "small": "small" if small else "gemm"}[router_path]
    assert r.path == want
    torch.cuda.synchronize()
    logits = r.logits[:T, :E].double().cpu().numpy()
    xd, wd = x.double().cpu().numpy(), w_r.double().cpu().numpy()
    assert rel(logits, xd @ wd) < 1e-5
    dec = R.route(logits, np.eye(E), score=score, top_k=K,
                  selection_bias=None if sb is None else sb.double().cpu().numpy())
    idx = r.topk_idx.long().cpu().numpy()
    gmap = np.zeros((T, E), dtype=bool)
    np.put_along_axis(gmap, idx, True, axis=1)
    assert np.array_equal(gmap, dec.routing_map)
    assert np.array_equal(r.counts.cpu().numpy(), dec.counts)
    np.testing.assert_allclose(r.topk_prob.cpu().numpy(), np.take_along_axis(dec.probs, idx, 1),
                               rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(r.scores.cpu().numpy(), dec.scores, rtol=1e-5, atol=1e-7)
    assert abs(float(r.aux) - R.aux_loss(dec, 1e-2)) <= 1e-5 * R.aux_loss(dec, 1e-2)
    # backward with a random upstream dprob and the aux term
    dprob = torch.randn((T, K), device=dev, generator=g)
    w_r_pad = None if router_path != "gemm" else ops.stage_router_weight(w_r)[1]
    dw, dx = ops.router_backward(x, w_r_pad, r, dprob, score, aux_scale=1.0)
    torch.cuda.synchronize()
    # reference: ds = dprob at the selections + aux gradient, through the score Jacobian
    s = dec.scores
    ds = np.zeros((T, E))
    np.put_along_axis(ds, idx, dprob.double().cpu().numpy(), axis=1)
    ds += (1e-2 * E * dec.counts / (T * K) / T)[None, :]
    inner = (ds * s).sum(1, keepdims=True)
    if score == "softmax":
        dl = s * (ds - inner)
    else:
        sig = 1.0 / (1.0 + np.exp(-logits))
        dl = sig * (1 - sig) / sig.sum(1, keepdims=True) * (ds - inner)
    tol_dw = 1e-4 if small else 1e-2  # tcgen05 path rounds dl to bf16 (GEMM operand)
    assert rel(dw.double().cpu().numpy(), xd.T @ dl) < tol_dw
    assert rel(dx[:T].double().cpu().numpy(), dl @ wd.T) < (4e-3 if small else 1e-2)
