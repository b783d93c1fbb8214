"""tcgen05 grouped GEMM vs a plain torch fp32 reference (per expert)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_07685_b200 import gemm  # noqa: E402


ALIGN = 128  # set per test by the `pair` fixture (256 for the CTA-pair engine)


def _layout(counts, device):
    """Padded expert-major layout metadata for given per-expert row counts."""
    offs = [0]
    block_expert = []
    for e, c in enumerate(counts):
        nb = (c + ALIGN - 1) // ALIGN * (ALIGN // 128)
        block_expert += [e] * nb
        offs.append(offs[-1] + nb * 128)
    rows = offs[-1]
    max_rows = rows + 512  # slack: buffers sized by an upper bound
    be = torch.zeros(max_rows // 128, dtype=torch.int32)
    be[: len(block_expert)] = torch.tensor(block_expert, dtype=torch.int32)
    return (torch.tensor(offs, dtype=torch.int32, device=device), be.to(device),
            torch.tensor([len(block_expert)], dtype=torch.int32, device=device), rows, max_rows)


def _rows(counts, offs_host, width, device, gen):
    x = torch.zeros((offs_host[-1] + 512, width), dtype=torch.bfloat16, device=device)
    for e, c in enumerate(counts):
        x[offs_host[e]: offs_host[e] + c] = torch.randn((c, width), generator=gen).to(device, torch.bfloat16)
    return x


def _relerr(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


@pytest.fixture(params=[False, True], ids=["cta1", "cta_pair"])
def pair(request):
    global ALIGN
    ALIGN = 256 if request.param else 128
    yield request.param
    ALIGN = 128


COUNTS = [200, 0, 333, 128, 1]


def test_fc2_fwd_plain(dev, pair):
    g = torch.Generator().manual_seed(0)
    E, m, h = len(COUNTS), 256, 512
    offs, be, nmb, rows, max_rows = _layout(COUNTS, dev)
    oh = offs.tolist()
    act = _rows(COUNTS, oh, m, dev, g)
    w2 = (torch.randn((E, h, m), generator=g) / m ** 0.5).to(dev, torch.bfloat16)
    out = gemm.fc2_fwd(act, w2, be, nmb, pair=pair)
    torch.cuda.synchronize()
    for e, c in enumerate(COUNTS):
        ref = act[oh[e]: oh[e] + c].float() @ w2[e].float().T
        got = out[oh[e]: oh[e] + c]
        if c:
            assert _relerr(got, ref) < 1e-2, e
    # padding rows are zero in, zero out
    assert out[oh[0] + COUNTS[0]: oh[1]].abs().max().item() == 0


def test_fc1_fwd_swiglu(dev, pair):
    g = torch.Generator().manual_seed(1)
    E, m, h = len(COUNTS), 384, 256
    offs, be, nmb, rows, max_rows = _layout(COUNTS, dev)
    oh = offs.tolist()
    xp = _rows(COUNTS, oh, h, dev, g)
    gate = (torch.randn((E, m, h), generator=g) / h ** 0.5).to(dev, torch.bfloat16)
    up = (torch.randn((E, m, h), generator=g) / h ** 0.5).to(dev, torch.bfloat16)
    w1 = gemm.interleave_gate_up(gate, up)
    prob = torch.rand((xp.shape[0],), generator=g).to(dev)
    for rp in (None, prob):
        preact, act = gemm.fc1_fwd(xp, w1, be, nmb, row_prob=rp, pair=pair)
        torch.cuda.synchronize()
        gp, upre = gemm.deinterleave_cols(preact)
        for e, c in enumerate(COUNTS):
            if not c:
                continue
            xs = xp[oh[e]: oh[e] + c].float()
            rg = xs @ gate[e].float().T
            ru = xs @ up[e].float().T
            ra = torch.nn.functional.silu(rg) * ru
            if rp is not None:
                ra = ra * rp[oh[e]: oh[e] + c, None]
            assert _relerr(gp[oh[e]: oh[e] + c], rg) < 1e-2
            assert _relerr(upre[oh[e]: oh[e] + c], ru) < 1e-2
            assert _relerr(act[oh[e]: oh[e] + c], ra) < 1e-2


def test_fc2_dgrad_dswiglu(dev, pair):
    g = torch.Generator().manual_seed(2)
    E, m, h = len(COUNTS), 512, 256
    offs, be, nmb, rows, max_rows = _layout(COUNTS, dev)
    oh = offs.tolist()
    dout = _rows(COUNTS, oh, h, dev, g)
    preact = _rows(COUNTS, oh, 2 * m, dev, g)
    w2 = (torch.randn((E, h, m), generator=g) / m ** 0.5).to(dev, torch.bfloat16)
    prob = torch.rand((dout.shape[0],), generator=g).to(dev)
    for rp in (None, prob):
        dpre, part = gemm.fc2_dgrad(dout, w2, preact, be, nmb, row_prob=rp, want_dprob=True,
                                     pair=pair)
        torch.cuda.synchronize()
        dg, du = gemm.deinterleave_cols(dpre)
        pg, pu = gemm.deinterleave_cols(preact)
        for e, c in enumerate(COUNTS):
            if not c:
                continue
            sl = slice(oh[e], oh[e] + c)
            G = dout[sl].float() @ w2[e].float()
            gg, uu = pg[sl].float(), pu[sl].float()
            s = torch.sigmoid(gg)
            a = gg * s * uu
            da = G * (rp[sl, None] if rp is not None else 1.0)
            rdg = da * uu * s * (1 + gg * (1 - s))
            rdu = da * gg * s
            assert _relerr(dg[sl], rdg) < 1e-2
            assert _relerr(du[sl], rdu) < 1e-2
            rdp = (G * a).sum(1)
            assert _relerr(part[sl].sum(1), rdp) < 1e-3


def test_fc1_dgrad(dev, pair):
    g = torch.Generator().manual_seed(3)
    E, m, h = len(COUNTS), 256, 512
    offs, be, nmb, rows, max_rows = _layout(COUNTS, dev)
    oh = offs.tolist()
    dpre = _rows(COUNTS, oh, 2 * m, dev, g)
    w1 = (torch.randn((E, 2 * m, h), generator=g) / h ** 0.5).to(dev, torch.bfloat16)
    dx = gemm.fc1_dgrad(dpre, w1, be, nmb, pair=pair)
    torch.cuda.synchronize()
    for e, c in enumerate(COUNTS):
        if c:
            sl = slice(oh[e], oh[e] + c)
            assert _relerr(dx[sl], dpre[sl].float() @ w1[e].float()) < 1e-2


def test_wgrad(dev, pair):
    g = torch.Generator().manual_seed(4)
    E, M, N = len(COUNTS), (256 if pair else 128), 512  # M % 256 == 0 -> pair engine
    offs, be, nmb, rows, max_rows = _layout(COUNTS, dev)
    oh = offs.tolist()
    a = _rows(COUNTS, oh, M, dev, g)
    b = _rows(COUNTS, oh, N, dev, g)
    dw = gemm.wgrad(a, b, offs, E)
    torch.cuda.synchronize()
    for e, c in enumerate(COUNTS):
        sl = slice(oh[e], oh[e + 1])
        ref = a[sl].float().T @ b[sl].float()
        if c == 0:
            assert dw[e].abs().max().item() == 0
        else:
            assert _relerr(dw[e], ref) < 1e-2, e


def test_gemm_f32_large_k(dev):
    g = torch.Generator().manual_seed(5)
    counts = [1000, 2000]
    E, K, N = 2, 4096, 256
    offs, be, nmb, rows, max_rows = _layout(counts, dev)
    oh = offs.tolist()
    a = _rows(counts, oh, K, dev, g)
    b = (torch.randn((E, N, K), generator=g) / K ** 0.5).to(dev, torch.bfloat16)
    out = gemm.gemm_f32(a, b, be, nmb)
    torch.cuda.synchronize()
    for e, c in enumerate(counts):
        sl = slice(oh[e], oh[e] + c)
        assert _relerr(out[sl], a[sl].float() @ b[e].float().T) < 1e-4


def test_split_units_all_grouped_m_gemms(dev):
    """Split units (ops.Plan.units, flags pair | split): a 128-row aligned plan whose experts
    run as 256-row pairs on the CTA-pair engine plus an odd last 128-row block on the 1-CTA
    engine. Odd and even block counts, an empty expert and enough pairs for several waves;
    every grouped-M GEMM against torch fp32, and the unit table against its definition."""
    from paper_2603_07685_b200 import _lib

    g = torch.Generator().manual_seed(7)
    counts = [200, 0, 333, 128, 1, 2500, 640, 129]
    E, m, h = len(counts), 256, 512
    global ALIGN
    ALIGN = 128
    offs, be, nmb, rows, max_rows = _layout(counts, dev)
    oh = offs.tolist()
    cap = max_rows // 128
    meta = torch.tensor([rows // 128, rows, 0], dtype=torch.int32, device=dev)
    units = torch.full((2 + 2 * cap,), -7, dtype=torch.int32, device=dev)
    _lib.call("moe_split_units", meta.data_ptr(), be.data_ptr(), offs.data_ptr(), cap,
              units.data_ptr(), torch.cuda.current_stream().cuda_stream)
    u = units.cpu().tolist()
    pairs, singles = [], []
    for e in range(E):
        b0, b1 = oh[e] // 128, oh[e + 1] // 128
        pairs += list(range(b0, b1 - 1, 2))
        if (b1 - b0) % 2:
            singles.append(b1 - 1)
    assert u[0] == len(pairs) and u[1] == len(singles)
    assert u[2: 2 + u[0]] == pairs and u[2 + cap: 2 + cap + u[1]] == singles

    xp = _rows(counts, oh, h, dev, g)
    w1 = (torch.randn((E, 2 * m, h), generator=g) / h ** 0.5).to(dev, torch.bfloat16)
    w2 = (torch.randn((E, h, m), generator=g) / m ** 0.5).to(dev, torch.bfloat16)
    kw = dict(pair=True, units=units)
    preact, act = gemm.fc1_fwd(xp, w1, be, nmb, **kw)
    o = gemm.fc2_fwd(act, w2, be, nmb, **kw)
    dout = _rows(counts, oh, h, dev, g)
    d_pre, _ = gemm.fc2_dgrad(dout, w2, preact, be, nmb, **kw)
    dxp = gemm.fc1_dgrad(d_pre, w1, be, nmb, **kw)
    torch.cuda.synchronize()
    for e, c in enumerate(counts):
        if not c:
            continue
        sl = slice(oh[e], oh[e] + c)
        pre_ref = xp[sl].float() @ w1[e].float().T
        assert _relerr(preact[sl], pre_ref) < 1e-2, ("fc1", e)
        gate, up = gemm.deinterleave_cols(preact[sl].float())
        a_ref = torch.nn.functional.silu(gate) * up
        assert _relerr(act[sl], a_ref) < 1e-2, ("act", e)
        assert _relerr(o[sl], act[sl].float() @ w2[e].float().T) < 1e-2, ("fc2", e)
        da = dout[sl].float() @ w2[e].float()
        s = torch.sigmoid(gate)
        dg_ref = da * up * s * (1 + gate * (1 - s))
        du_ref = da * gate * s
        dg, du = gemm.deinterleave_cols(d_pre[sl].float())
        assert _relerr(dg, dg_ref) < 2e-2 and _relerr(du, du_ref) < 2e-2, ("fc2 dgrad", e)
        assert _relerr(dxp[sl], d_pre[sl].float() @ w1[e].float()) < 1e-2, ("fc1 dgrad", e)
