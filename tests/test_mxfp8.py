"""MXFP8: the oracle (oracle/mxfp8_ref.py) against codes and scales
produced by the reference quantizer (tests/golden/mxfp8_golden.npz, quant.py:166-201); the
device quantizer bit-exact against both; the block-scaled tcgen05 grouped GEMMs against the
reference's dequantize-then-multiply GEMM (fp64) on the same codes."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import mxfp8_ref as M

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "mxfp8_golden.npz")


def test_oracle_matches_reference_golden():
    codes, scales = M.quantize_mxfp8(GOLD["x"].astype(np.float64))
    assert np.array_equal(codes, GOLD["codes"])
    assert np.array_equal(scales, GOLD["scales"])
    assert np.array_equal(M.dequantize_mxfp8(codes, scales), GOLD["dequant"])


def test_tiled_scale_layout():
    s = np.arange(256 * 8, dtype=np.int64).reshape(256, 8).astype(np.uint8)
    t = M.tile_scales(s, 256)
    for row, kb in [(0, 0), (5, 3), (37, 1), (127, 7), (128, 0), (200, 6)]:
        tile, rr = divmod(row, 128)
        off = (tile * 2 + kb // 4) * 512 + (rr % 32) * 16 + (rr // 32) * 4 + kb % 4
        assert t[off] == s[row, kb]


def _bf16(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16)


@pytest.mark.gpu
def test_device_quantizer_bit_exact():
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    x = torch.from_numpy(GOLD["x"]).to(torch.bfloat16).to(dev)
    codes, sf_t, sf_p = gemm.mxfp8_quantize(x, plain=True)
    r = x.shape[0]
    assert np.array_equal(codes[:r].cpu().numpy(), GOLD["codes"])
    assert np.array_equal(sf_p.cpu().numpy(), GOLD["scales"])
    assert np.array_equal(sf_t.cpu().numpy(), M.tile_scales(GOLD["scales"], codes.shape[0]))


def _plan(rows_per_expert, dev):
    be = np.concatenate([np.full(r // 128, e) for e, r in enumerate(rows_per_expert)])
    return (torch.tensor(be, dtype=torch.int32, device=dev),
            torch.tensor([len(be)], dtype=torch.int32, device=dev), int(sum(rows_per_expert)))


@pytest.mark.gpu
@pytest.mark.parametrize("wide", [False, True], ids=["n128", "n256"])
@pytest.mark.parametrize("pair", [False, True], ids=["cta1", "pair"])
@pytest.mark.parametrize("E,K,N", [(2, 256, 256), (3, 512, 512)])
def test_mxfp8_grouped_gemm_matches_dequant_gemm(E, K, N, pair, wide):
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(E * 7 + K)
    rows_e = ([256, 512, 256] if pair else [256, 128, 384])[:E]
    be, nmb, rows = _plan(rows_e, dev)
    a = (torch.randn((rows, K), generator=g) * 3).to(torch.bfloat16)
    a[100:128] = 0  # padding-like rows
    w = (torch.randn((E, N, K), generator=g) * 0.05).to(torch.bfloat16)
    aq, asf, asp = gemm.mxfp8_quantize(a.to(dev), plain=True)
    wq, wsf, wsp = gemm.mxfp8_quantize(w.reshape(E * N, K).to(dev), plain=True)
    out = gemm.mxfp8_gemm(aq, asf, wq, wsf, E, be, nmb, N, pair=pair,
                          wide=wide).float().cpu().numpy()
    ad = M.dequantize_mxfp8(aq.cpu().numpy()[:rows], asp.cpu().numpy())
    wd = M.dequantize_mxfp8(wq.cpu().numpy(), wsp.cpu().numpy()).reshape(E, N, K)
    ref = np.concatenate([ad[sum(rows_e[:e]):sum(rows_e[:e + 1])] @ wd[e].T
                          for e in range(E)])
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert err < 4e-3, err


@pytest.mark.gpu
@pytest.mark.parametrize("wide", [False, True], ids=["n128", "n256"])
@pytest.mark.parametrize("pair", [False, True], ids=["cta1", "pair"])
def test_mxfp8_fc1_swiglu_and_fused_act_quantisation(pair, wide):
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(11)
    E, h, m = 2, 256, 256
    rows_e = [256, 512] if pair else [128, 256]
    be, nmb, rows = _plan(rows_e, dev)
    x = torch.randn((rows, h), generator=g).to(torch.bfloat16)
    gate = (torch.randn((E, m, h), generator=g) * h ** -0.5).to(torch.bfloat16)
    up = (torch.randn((E, m, h), generator=g) * h ** -0.5).to(torch.bfloat16)
    xq, xsf, xsp = gemm.mxfp8_quantize(x.to(dev), plain=True)
    blk = 128 if wide else 64
    w1 = (gemm.interleave_gate_up if wide else gemm.interleave_gate_up_mx)(gate.to(dev),
                                                                          up.to(dev))
    wq, wsf, wsp = gemm.mxfp8_quantize(w1.reshape(E * 2 * m, h), plain=True)
    preact, act, act_q, act_sf, act_t, act_tsf = gemm.mxfp8_fc1(
        xq, xsf, wq, wsf, E, be, nmb, m, pair=pair, wide=wide, want_t=True)
    torch.cuda.synchronize()
    xd = M.dequantize_mxfp8(xq.cpu().numpy()[:rows], xsp.cpu().numpy())
    wd = M.dequantize_mxfp8(wq.cpu().numpy(), wsp.cpu().numpy()).reshape(E, 2 * m, h)
    gd = wd.reshape(E, m // blk, 2, blk, h)[:, :, 0].reshape(E, m, h)
    ud = wd.reshape(E, m // blk, 2, blk, h)[:, :, 1].reshape(E, m, h)
    off = np.cumsum([0] + rows_e)
    zg = np.concatenate([xd[off[e]:off[e + 1]] @ gd[e].T for e in range(E)])
    zu = np.concatenate([xd[off[e]:off[e + 1]] @ ud[e].T for e in range(E)])
    pg, pu = gemm.deinterleave_cols(preact)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(pg.float().cpu().numpy(), zg) < 4e-3
    assert rel(pu.float().cpu().numpy(), zu) < 4e-3
    a_ref = zg / (1 + np.exp(-zg)) * zu
    assert rel(act.float().cpu().numpy(), a_ref) < 1e-2
    # the fused quantisation equals quantize(act) of the kernel's own bf16 activation
    codes, scales = M.quantize_mxfp8(act.float().cpu().numpy().astype(np.float64))
    assert np.array_equal(act_q.cpu().numpy(), codes)
    assert np.array_equal(act_sf.cpu().numpy(), M.tile_scales(scales, rows))
    # ... and along the token rows (warp-shuffle block amax): quantise(act^T) of the same act
    ct, st = M.quantize_mxfp8(act.float().cpu().numpy().astype(np.float64).T)
    assert np.array_equal(act_t.cpu().numpy(), ct)
    assert np.array_equal(act_tsf.cpu().numpy(), M.tile_scales(st, m))


@pytest.mark.gpu
def test_w1_remap_quantisation_equals_interleave_then_quantise():
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(2)
    E, m, h = 2, 256, 256
    gate = torch.randn((E, m, h), generator=g).to(torch.bfloat16).to(dev)
    up = torch.randn((E, m, h), generator=g).to(torch.bfloat16).to(dev)
    a = gemm.mxfp8_quantize_w1(gemm.interleave_gate_up(gate, up))
    b = gemm.mxfp8_quantize_weight(gemm.interleave_gate_up_mx(gate, up))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.gpu
def test_transposing_quantiser_equals_quantise_of_transpose():
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(9)
    x = (torch.randn((3, 256, 384), generator=g) * 2).to(torch.bfloat16)
    codes, sf_t, sf_p = gemm.mxfp8_quantize_t(x.to(dev), plain=True)
    xt = x.transpose(1, 2).reshape(3 * 384, 256).float().numpy().astype(np.float64)
    want_c, want_s = M.quantize_mxfp8(xt)
    assert np.array_equal(codes.cpu().numpy(), want_c)
    assert np.array_equal(sf_p.cpu().numpy(), want_s)
    assert np.array_equal(sf_t.cpu().numpy(), M.tile_scales(want_s, 3 * 384))


@pytest.mark.gpu
@pytest.mark.parametrize("pair,wide", [(False, False), (True, True)], ids=["cta1", "pair_wide"])
def test_mxfp8_dgrad_chain_matches_dequant_oracle(pair, wide):
    """fc2 dgrad + dSwiGLU (fused d_preact quantisation) and fc1 dgrad on MXFP8 operands vs
    the dequantise-then-multiply oracle; the fused quantisation is bit-exact."""
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(17)
    E, h, m = 2, 256, 256
    rows_e = [256, 512] if pair else [128, 256]
    be, nmb, rows = _plan(rows_e, dev)
    d_o = torch.randn((rows, h), generator=g).to(torch.bfloat16)
    preact = torch.randn((rows, 2 * m), generator=g).to(torch.bfloat16)
    w2 = (torch.randn((E, h, m), generator=g) * m ** -0.5).to(torch.bfloat16)
    w1 = (torch.randn((E, 2 * m, h), generator=g) * h ** -0.5).to(torch.bfloat16)
    doq, dosf, dosp = gemm.mxfp8_quantize(d_o.to(dev), plain=True)
    w2tq, w2tsf, w2tsp = gemm.mxfp8_quantize_t(w2.to(dev), plain=True)
    d_pre, dq, dsf, dpt, dptsf = gemm.mxfp8_fc2_dgrad(doq, dosf, w2tq, w2tsf, E, be, nmb,
                                                      preact.to(dev), pair=pair, wide=wide,
                                                      want_t=True)
    w1tq, w1tsf, w1tsp = gemm.mxfp8_quantize_t(w1.to(dev), plain=True)
    dxp = gemm.mxfp8_gemm(dq, dsf, w1tq, w1tsf, E, be, nmb, h, pair=pair, wide=wide)
    torch.cuda.synchronize()
    off = np.cumsum([0] + rows_e)
    dod = M.dequantize_mxfp8(doq.cpu().numpy()[:rows], dosp.cpu().numpy())
    w2t = M.dequantize_mxfp8(w2tq.cpu().numpy(), w2tsp.cpu().numpy()).reshape(E, m, h)
    G = np.concatenate([dod[off[e]:off[e + 1]] @ w2t[e].T for e in range(E)])
    pg, pu = gemm.deinterleave_cols(preact)
    gg, uu = pg.double().numpy(), pu.double().numpy()
    s = 1 / (1 + np.exp(-gg))
    dg_ref = G * uu * s * (1 + gg * (1 - s))
    du_ref = G * gg * s
    got_g, got_u = gemm.deinterleave_cols(d_pre)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(got_g.double().cpu().numpy(), dg_ref) < 5e-3
    assert rel(got_u.double().cpu().numpy(), du_ref) < 5e-3
    codes, scales = M.quantize_mxfp8(d_pre.float().cpu().numpy().astype(np.float64))
    assert np.array_equal(dq.cpu().numpy(), codes)
    assert np.array_equal(dsf.cpu().numpy(), M.tile_scales(scales, rows))
    ct, st = M.quantize_mxfp8(d_pre.float().cpu().numpy().astype(np.float64).T)
    assert np.array_equal(dpt.cpu().numpy(), ct)
    assert np.array_equal(dptsf.cpu().numpy(), M.tile_scales(st, 2 * m))
    dpd = M.dequantize_mxfp8(codes, scales)
    w1t = M.dequantize_mxfp8(w1tq.cpu().numpy(), w1tsp.cpu().numpy()).reshape(E, h, 2 * m)
    dx_ref = np.concatenate([dpd[off[e]:off[e + 1]] @ w1t[e].T for e in range(E)])
    assert rel(dxp.double().cpu().numpy(), dx_ref) < 5e-3


@pytest.mark.gpu
@pytest.mark.parametrize("Mo,No", [(256, 256), (128, 384)], ids=["pair_wide", "cta1_narrow"])
def test_mxfp8_wgrad_matches_dequant_oracle(Mo, No):
    """Grouped-K weight gradient on column-quantised operands, incl. an expert without rows."""
    from paper_2603_07685_b200 import gemm

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(23)
    rows_e = [256, 0, 384]
    K = sum(rows_e)
    off = torch.tensor(np.cumsum([0] + rows_e), dtype=torch.int32, device=dev)
    a = torch.randn((K, Mo), generator=g).to(torch.bfloat16)
    b = torch.randn((K, No), generator=g).to(torch.bfloat16)
    dw = gemm.mxfp8_wgrad(a.to(dev), b.to(dev), off, 3).double().cpu().numpy()
    at, asf, asp = gemm.mxfp8_quantize_t(a.to(dev), plain=True)
    bt, bsf, bsp = gemm.mxfp8_quantize_t(b.to(dev), plain=True)
    ad = M.dequantize_mxfp8(at.cpu().numpy(), asp.cpu().numpy())  # [M, K]
    bd = M.dequantize_mxfp8(bt.cpu().numpy(), bsp.cpu().numpy())  # [N, K]
    o = np.cumsum([0] + rows_e)
    for e in range(3):
        ref = ad[:, o[e]:o[e + 1]] @ bd[:, o[e]:o[e + 1]].T
        if rows_e[e] == 0:
            assert not dw[e].any()
        else:
            assert np.linalg.norm(dw[e] - ref) / np.linalg.norm(ref) < 5e-3
