"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``moelab.routing`` and ``moelab.perf`` read-only from
/root/reference/pkg/src, runs them on seeded inputs, and writes
``tests/golden/routing_golden.npz``. Nothing on the GPU box reads /root/reference;
the committed .npz is what travels. ``tests/test_oracle.py`` pins
``oracle/routing_ref.py`` against this file.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "routing_golden.npz"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from moelab import perf, routing as r  # noqa: E402  (reference, read-only)

    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(2603)

    def put(prefix, d):
        g[f"{prefix}/probs"] = d.probs
        g[f"{prefix}/routing_map"] = d.routing_map
        g[f"{prefix}/counts"] = d.counts
        g[f"{prefix}/scores"] = d.scores
        g[f"{prefix}/effective_counts"] = d.effective_counts()
        if d.dropped is not None:
            g[f"{prefix}/dropped"] = d.dropped
        if d.phantom_rows is not None:
            g[f"{prefix}/phantom_rows"] = d.phantom_rows

    t, h, e, m = 40, 12, 6, 10
    x = rng.normal(size=(t, h))
    w_r = rng.normal(size=(h, e))
    bias = rng.normal(size=e) * 0.05
    g["x"], g["w_r"], g["bias"] = x, w_r, bias
    params = r.ExpertParams(
        w1=[rng.normal(size=(m, h)) for _ in range(e)],
        w2=[rng.normal(size=(h, m)) for _ in range(e)],
        gate=[rng.normal(size=(m, h)) for _ in range(e)],
    )
    plain = r.ExpertParams(w1=params.w1, w2=params.w2)
    for i in range(e):
        g[f"params/w1/{i}"] = params.w1[i]
        g[f"params/w2/{i}"] = params.w2[i]
        g[f"params/gate/{i}"] = params.gate[i]

    cases = {
        "softmax_k2": dict(score="softmax", top_k=2),
        "sigmoid_k3": dict(score="sigmoid", top_k=3),
        "softmax_k2_bias": dict(score="softmax", top_k=2, selection_bias=bias),
        "sigmoid_k1_bias": dict(score="sigmoid", top_k=1, selection_bias=bias),
    }
    for name, kw in cases.items():
        d = r.route(x, w_r, **kw)
        put(f"route/{name}", d)
        g[f"aux/{name}"] = np.array(r.aux_loss(d, 0.01))
        perm, rmap = r.permute(x, d)
        g[f"permute/{name}/rows"] = perm
        g[f"permute/{name}/row_id_map"] = rmap
        g[f"unpermute/{name}"] = r.unpermute_sum(perm, rmap, t)
        g[f"combine_standard/{name}/gated"] = r.combine_standard(x, d, params)
        g[f"combine_mem_efficient/{name}/gated"] = r.combine_mem_efficient(x, d, params)
        g[f"combine_standard/{name}/plain"] = r.combine_standard(x, d, plain)
        g[f"combine_mem_efficient/{name}/plain"] = r.combine_mem_efficient(x, d, plain)

    # ties: equal logits, lowest index wins
    d = r.route(np.zeros((3, 5)), np.eye(5), top_k=3)
    put("route/ties", d)

    # aux gradient (softmax), FD-pinned in the reference's own tests
    g["aux_grad/k2"] = r.aux_loss_grad_wr(x, w_r, 2, 0.37)

    # aux-free bias update
    g["auxfree/counts"] = np.array([10, 2, 2, 2, 7, 4])
    g["auxfree/out"] = r.auxfree_bias_update(g["auxfree/counts"], bias, 0.05)

    # capacity (skewed router), with and without pad
    skew = np.array([2.0, 1.0, 0.0, -1.0, -1.0, -2.0])
    logits = rng.normal(size=(t, e)) + skew
    g["cap/logits"] = logits
    d = r.route(logits, np.eye(e), top_k=2)
    for pad in (False, True):
        for cf in (1.0, 0.5, 1.25):
            c = r.apply_capacity(d, cf, pad=pad)
            key = f"cap/cf{cf}_pad{int(pad)}"
            put(key, c)
            perm, rmap = r.permute(x, c)
            g[f"{key}/row_id_map"] = rmap
            g[f"{key}/rows"] = perm
            g[f"{key}/residual_out"] = r.moe_output_with_residual(x, c, params)
    g["cap/expert_capacity"] = np.array([
        r.expert_capacity(1.0, 128, 2, 8), r.expert_capacity(1.0, 16384, 2, 8),
        r.expert_capacity(1.0, 32768, 8, 128), r.expert_capacity(1.0, 4096, 8, 256),
        r.expert_capacity(0.7, 999, 3, 7)])

    # routing-map pad
    d = r.route(x, w_r, top_k=2)
    for mult in (4, 8, 16):
        pd = r.routing_map_pad(d, mult)
        put(f"pad/m{mult}", pd)
        g[f"pad/m{mult}/row_id_map"] = r.permute(x, pd)[1]

    # latent MoE with a shared expert (DeepSeek composition)
    lat = 5
    experts = r.ExpertParams(
        w1=[rng.normal(size=(m, lat)) for _ in range(e)],
        w2=[rng.normal(size=(lat, m)) for _ in range(e)],
        gate=[rng.normal(size=(m, lat)) for _ in range(e)],
    )
    shared = r.ExpertParams(w1=[rng.normal(size=(m, h))], w2=[rng.normal(size=(h, m))],
                            gate=[rng.normal(size=(m, h))])
    w_down = rng.normal(size=(lat, h))
    w_up = rng.normal(size=(h, lat))
    for i in range(e):
        g[f"latent/experts/w1/{i}"] = experts.w1[i]
        g[f"latent/experts/w2/{i}"] = experts.w2[i]
        g[f"latent/experts/gate/{i}"] = experts.gate[i]
    g["latent/shared/w1"], g["latent/shared/w2"], g["latent/shared/gate"] = (
        shared.w1[0], shared.w2[0], shared.gate[0])
    g["latent/w_down"], g["latent/w_up"] = w_down, w_up
    d = r.route(x, w_r, top_k=2)
    g["latent/out"] = r.latent_moe_forward(x, w_down, w_up, experts, d, shared)
    eye = np.eye(h)
    g["latent/identity_shared_out"] = r.latent_moe_forward(x, eye, eye, params, d, shared)

    # upcycling
    dw1 = rng.normal(size=(8, 4))
    dw2 = rng.normal(size=(4, 8))
    dgate = rng.normal(size=(8, 4))
    up, wr0 = r.upcycle(dw1, dw2, 2, 2, dense_gate=dgate)
    g["upcycle/in_w1"], g["upcycle/in_w2"], g["upcycle/in_gate"] = dw1, dw2, dgate
    for i in range(up.num_experts):
        g[f"upcycle/w1/{i}"], g[f"upcycle/w2/{i}"], g[f"upcycle/gate/{i}"] = (
            up.w1[i], up.w2[i], up.gate[i])
    g["upcycle/w_r"] = wr0

    # EP all-to-all byte model at the BASELINE configs (perf.py:62-70)
    vol = []
    for (tok, k, hid) in ((16384, 2, 4096), (32768, 8, 4096), (4096, 8, 7168)):
        for ep in (1, 2, 4, 8, 64):
            vol.append([tok, k, hid, ep, perf.a2a_send_volume(tok, k, hid, ep, 2)])
    g["a2a/table"] = np.array(vol, dtype=np.float64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({len(g)} arrays)")


if __name__ == "__main__":
    main()
