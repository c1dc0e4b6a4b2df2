"""GPU: K6 fused dequant + outlier GEMV / skinny GEMM vs dequantize_tensor +
an fp64 GEMV (the oracle's ezqo_gemv_f64). Parity is unpinned by the
reference (it has no GEMV); the bar is 1e-3 relative with fp32 accumulation
(BASELINE.json north_star)."""
import numpy as np
import pytest

from paper_2403_02775_b200.native import Config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols,sigma,bits", [
    (4096, 4096, 3.0, 4), (512, 1024, 2.5758, 4), (1024, 264, 2.8070, 4),
    (4096, 11008, 2.5758, 4), (11008, 4096, 2.5758, 4),  # the benched LLaMA-7B shapes
    (300, 77, 3.0, 4),      # generic path (odd cols)
    (256, 128, 3.0, 3),     # k=3 byte-per-level codes
])
@pytest.mark.parametrize("batch", [1, 2, 5, 8, 16, 21])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
def test_gemv_matches_dequant_f64(gpu, O, rows, cols, sigma, bits, batch, dtype):
    _gemv_case(gpu, O, rows, cols, sigma, bits, batch, dtype, "float32")


@pytest.mark.parametrize("rows,cols", [(4096, 11008), (1000, 200), (2048, 520)])
@pytest.mark.parametrize("batch", [1, 9])
@pytest.mark.parametrize("xdt", ["bfloat16", "float32"])
def test_gemv_half_outlier_values(gpu, O, rows, cols, batch, xdt):
    """N1: outlier values stored as f16 (6 bytes per outlier) stay within the
    1e-3 gate against dequantize + the fp64 GEMV."""
    _gemv_case(gpu, O, rows, cols, 2.5758, 4, batch, xdt, "float16")


def _gemv_case(gpu, O, rows, cols, sigma, bits, batch, dtype, odt):
    import torch
    W = O.gaussian(rows, cols, rows + cols, 0.02)
    O.plant_outliers(W, max(1, W.size // 200), 0.2, 1.0, 77)
    Wd = torch.from_numpy(W).cuda()
    b = gpu.quantize_batch([Wd], Config(bits=bits, sigma_n=sigma, steps=20), out_mem=gpu.MEM_DEVICE)
    q = b.to_host(0)
    What = gpu.dequantize(q)
    plan = gpu.GemvPlan(b, 0, outlier_dtype=odt)
    g = torch.Generator(device="cuda").manual_seed(batch)
    x = torch.randn(batch, rows, generator=g, device="cuda").to(getattr(torch, dtype))
    y = plan(x).cpu().numpy().astype(np.float64)
    xf = x.float().cpu().numpy()
    yref = O.gemv_f64(What, xf)
    err = np.abs(y - yref).max()
    assert err <= 1e-3 * np.abs(yref).max(), (err, np.abs(yref).max())
    if odt != "float32":
        # the kernel against the format it computes with: the outlier values
        # rounded to the storage dtype (the rounding itself is the format's
        # error, held to the max-norm gate above)
        o = q.outliers
        Wq = What.copy()
        v = torch.from_numpy(o["value"].copy()).to(getattr(torch, odt)).float().numpy()
        Wq[o["row"], o["col"]] = v
        yref = O.gemv_f64(Wq, xf)
    assert np.all(np.abs(y - yref) <= 1e-3 * np.abs(yref) + 1e-4 * np.abs(yref).max())
    plan.close()
    b.close()


def test_gemv_outlier_term_exact_path(gpu, O):
    """Outliers only (all-zero normals): y must equal sum x_i v exactly up to fp32."""
    import torch
    W = np.zeros((64, 64), np.float32)
    W[3, 5], W[40, 5], W[7, 63] = 50.0, -20.0, 33.0
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(sigma_n=1.0), out_mem=gpu.MEM_DEVICE)
    assert b.to_host(0).outliers.size == 3
    plan = gpu.GemvPlan(b, 0)
    x = torch.arange(64, dtype=torch.float32, device="cuda")[None, :]
    y = plan(x).cpu().numpy()[0]
    ref = O.gemv_f64(gpu.dequantize(b.to_host(0)), x.cpu().numpy())[0]
    assert np.allclose(y, ref, rtol=1e-6, atol=1e-4)
    assert y[5] == pytest.approx(3 * 50.0 - 40 * 20.0, rel=1e-6)


@pytest.mark.parametrize("rows,cols", [(1000, 200), (8192, 48), (64, 4096), (130, 17)])
@pytest.mark.parametrize("batch", [1, 9, 40])
def test_gemv_split_and_ragged(gpu, O, rows, cols, batch):
    """Split-K tiles (few columns, many rows), ragged K (rows % 64 != 0),
    partial 16-column tiles and multi-group batches; repeated calls reuse the
    workspace/tickets and must give bit-identical results (fixed-order
    reduction)."""
    import torch
    W = O.gaussian(rows, cols, rows ^ cols, 0.02)
    O.plant_outliers(W, max(1, W.size // 100), 0.2, 1.0, 6)
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(steps=10), out_mem=gpu.MEM_DEVICE)
    plan = gpu.GemvPlan(b, 0)
    x = torch.randn(batch, rows, generator=torch.Generator(device="cuda").manual_seed(3), device="cuda")
    y = plan(x).cpu().numpy()
    yref = O.gemv_f64(gpu.dequantize(b.to_host(0)), x.cpu().numpy())
    assert np.abs(y.astype(np.float64) - yref).max() <= 1e-3 * np.abs(yref).max()
    for _ in range(3):
        assert np.array_equal(plan(x).cpu().numpy().view(np.uint32), y.view(np.uint32))
    plan.close()
    b.close()


@pytest.mark.parametrize("rows,cols", [(1000, 700), (2048, 136), (4096, 2048)])
@pytest.mark.parametrize("batch", [1, 2, 5, 16])
@pytest.mark.parametrize("dtype", ["bfloat16", "float16", "float32"])
@pytest.mark.parametrize("odt", ["float32", "float16"])
def test_gemv_fused_vs_separate_outliers(gpu, O, monkeypatch, rows, cols, batch, dtype, odt):
    """The outlier term fused into the main kernel (512-row segments in the
    TMA ring, outlier warps) and the separate CSC pass (EZQ_GEMV_FUSED=0,
    also the path of f32 x at 9..16 rows and of segments too dense for the
    u16 header) both hold the 1e-3 gate, agree with each other to fp32
    rounding, and repeat bit for bit."""
    import torch
    W = O.gaussian(rows, cols, rows + 3 * cols, 0.02)
    O.plant_outliers(W, max(1, W.size // 50), 0.2, 1.0, 11)
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(sigma_n=2.5758, steps=10), out_mem=gpu.MEM_DEVICE)
    x = torch.randn(batch, rows, generator=torch.Generator(device="cuda").manual_seed(5), device="cuda")
    x = x.to(getattr(torch, dtype))
    ys = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("EZQ_GEMV_FUSED", fused)
        plan = gpu.GemvPlan(b, 0, outlier_dtype=odt)
        ys[fused] = plan(x).cpu().numpy()
        for _ in range(2):
            assert np.array_equal(plan(x).cpu().numpy().view(np.uint32), ys[fused].view(np.uint32))
        plan.close()
    q = b.to_host(0)
    Wq = gpu.dequantize(q)
    o = q.outliers
    Wq[o["row"], o["col"]] = torch.from_numpy(o["value"].copy()).to(getattr(torch, odt)).float().numpy()
    yref = O.gemv_f64(Wq, x.float().cpu().numpy())
    scale = np.abs(yref).max()
    for y in ys.values():
        assert np.abs(y.astype(np.float64) - yref).max() <= 1e-3 * scale
    assert np.abs(ys["1"].astype(np.float64) - ys["0"]).max() <= 1e-5 * scale
    b.close()


def test_gemv_dense_outliers(gpu, O):
    """Most entries outliers (sigma_n 0.5): large segments (fused when the ring
    still fits in shared memory, else the separate pass) stay exact."""
    import torch
    W = O.gaussian(1024, 256, 17, 0.02)
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(sigma_n=0.5, steps=5), out_mem=gpu.MEM_DEVICE)
    q = b.to_host(0)
    assert q.outliers.size > W.size // 2
    plan = gpu.GemvPlan(b, 0)
    for batch in (1, 3, 12):
        x = torch.randn(batch, 1024, generator=torch.Generator(device="cuda").manual_seed(batch), device="cuda")
        y = plan(x.to(torch.bfloat16)).cpu().numpy().astype(np.float64)
        yref = O.gemv_f64(gpu.dequantize(q), x.to(torch.bfloat16).float().cpu().numpy())
        assert np.abs(y - yref).max() <= 1e-3 * np.abs(yref).max()
    plan.close()
    b.close()


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("dims,batch", [((1024, 2048, 512, 768), 1), ((512, 4096, 1000, 300), 16),
                                        ((2048, 2048, 2048, 2048), 5)])
def test_gemv_chained_layers(gpu, O, graph, dims, batch):
    """A chain of GEMVs on one stream (each a programmatic dependent launch
    of the previous kernel): every layer's x is the previous layer's y, and
    every layer of a second pass writes one shared y -- the weight stream may
    start early, but x is read and y written only after the previous kernel
    (griddepcontrol.wait). Also inside a CUDA graph."""
    import torch
    Ws, plans, bs = [], [], []
    for i in range(len(dims) - 1):
        W = O.gaussian(dims[i], dims[i + 1], 31 + i, 0.02)
        O.plant_outliers(W, max(1, W.size // 100), 0.2, 1.0, 40 + i)
        b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(steps=5), out_mem=gpu.MEM_DEVICE)
        Ws.append(gpu.dequantize(b.to_host(0)).astype(np.float64))
        plans.append(gpu.GemvPlan(b, 0))
        bs.append(b)
    x0 = torch.randn(batch, dims[0], generator=torch.Generator(device="cuda").manual_seed(8), device="cuda")
    ys = [torch.empty(batch, d, device="cuda") for d in dims[1:]]
    shared = torch.empty(batch * max(dims[1:]), device="cuda")

    def out(d):  # contiguous [batch, d] view of the shared output buffer
        return shared[: batch * d].view(batch, d)

    zin = {d: torch.zeros(batch, d, device="cuda") for d in dims}

    def run():
        x = x0
        for p, y in zip(plans, ys):
            p(x, y)
            x = y
        for p, d in zip(plans, dims[1:]):  # WAW: the shared output keeps the last layer's result
            p(x0 if p is plans[0] else zin[p.rows], out(d))
        plans[0](x0, out(dims[1]))

    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            run()
        for y in ys:
            y.zero_()
        g.replay()
    else:
        run()
    torch.cuda.synchronize()
    ref = x0.cpu().numpy().astype(np.float64)
    for W, y in zip(Ws, ys):
        ref = ref @ W
        got = y.cpu().numpy().astype(np.float64)
        assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()
        ref = got  # each layer against its own input (the chain's errors do not compound in the check)
    first = x0.cpu().numpy().astype(np.float64) @ Ws[0]
    got = out(dims[1]).cpu().numpy().astype(np.float64)
    assert np.abs(got - first).max() <= 1e-3 * np.abs(first).max()
    for p in plans:
        p.close()
    for b in bs:
        b.close()


@pytest.mark.parametrize("tpc", [1, 2, 4, 8])
@pytest.mark.parametrize("batch,dtype", [(1, "bfloat16"), (2, "float32"), (5, "float16"), (16, "bfloat16"),
                                         (12, "float32")])
def test_gemv_every_colblock_width(gpu, O, monkeypatch, tpc, batch, dtype):
    """Every colblock width (EZQ_GEMV_TPC) with fused and separate outlier
    passes: QW > 1 reductions (TPC < 4), two tiles per warp (TPC = 8), the
    2-segment stages of batch groups <= 8 and the 1-segment ones of 9..16."""
    import torch
    W = O.gaussian(1536, 1000, 5 * tpc + batch, 0.02)
    O.plant_outliers(W, W.size // 80, 0.2, 1.0, 3)
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(sigma_n=2.5758, steps=5), out_mem=gpu.MEM_DEVICE)
    Wd = gpu.dequantize(b.to_host(0)).astype(np.float64)
    x = torch.randn(batch, 1536, generator=torch.Generator(device="cuda").manual_seed(tpc), device="cuda")
    x = x.to(getattr(torch, dtype))
    yref = x.float().cpu().numpy().astype(np.float64) @ Wd
    monkeypatch.setenv("EZQ_GEMV_TPC", str(tpc))
    for fused in ("1", "0"):
        monkeypatch.setenv("EZQ_GEMV_FUSED", fused)
        plan = gpu.GemvPlan(b, 0)
        y = plan(x).cpu().numpy().astype(np.float64)
        assert np.abs(y - yref).max() <= 1e-3 * np.abs(yref).max(), (tpc, fused)
        plan.close()
    b.close()


@pytest.mark.parametrize("rows,cols", [(2048, 12000), (4096, 4096), (1536, 700)])
@pytest.mark.parametrize("batch,dtype", [(1, "bfloat16"), (3, "float32"), (16, "bfloat16"), (12, "float16")])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_gemv_split_k_clusters(gpu, O, monkeypatch, rows, cols, batch, dtype, fused):
    """Split K over 2-CTA clusters (EZQ_GEMV_KS=2 with 1-tile colblocks):
    2048x12000 has 750 colblocks, more than the resident clusters, so every
    cluster loops over several colblocks (rank 0 frees rank 1's slot between
    them); 1536x700 gives rank 1 the shorter half. Within the 1e-3 gate
    against dequantize + the fp64 GEMV, within fp32 rounding of the unsplit
    kernel, and bit-identical across calls (fixed rank order)."""
    import torch
    W = O.gaussian(rows, cols, rows * 7 + cols, 0.02)
    O.plant_outliers(W, max(1, W.size // 100), 0.2, 1.0, 13)
    b = gpu.quantize_batch([torch.from_numpy(W).cuda()], Config(sigma_n=2.5758, steps=10), out_mem=gpu.MEM_DEVICE)
    x = torch.randn(batch, rows, generator=torch.Generator(device="cuda").manual_seed(9), device="cuda")
    x = x.to(getattr(torch, dtype))
    monkeypatch.setenv("EZQ_GEMV_TPC", "1")
    monkeypatch.setenv("EZQ_GEMV_FUSED", fused)
    monkeypatch.setenv("EZQ_GEMV_KS", "1")
    p1 = gpu.GemvPlan(b, 0)
    y1 = p1(x).cpu().numpy().astype(np.float64)
    monkeypatch.setenv("EZQ_GEMV_KS", "2")
    p2 = gpu.GemvPlan(b, 0)
    y2 = p2(x).cpu().numpy()
    yref = O.gemv_f64(gpu.dequantize(b.to_host(0)), x.float().cpu().numpy())
    scale = np.abs(yref).max()
    assert np.abs(y2.astype(np.float64) - yref).max() <= 1e-3 * scale
    assert np.abs(y2.astype(np.float64) - y1).max() <= 1e-5 * scale
    for _ in range(2):
        assert np.array_equal(p2(x).cpu().numpy().view(np.uint32), y2.view(np.uint32))
    p1.close()
    p2.close()
    b.close()


def test_gemv_bloom_shape_fused_vs_separate(gpu, monkeypatch):
    """The paper's practical-latency shape (BLOOM-176B FFN, 14336x53746, 1%
    outliers), which the bench times: the fused outlier term and the separate
    CSC pass agree to fp32 rounding and both hold the 1e-3 gate against
    dequantize + an fp64 matmul (batch 1 and 16, bf16 x)."""
    import torch
    r, c = 14336, 53746
    g = torch.Generator(device="cuda").manual_seed(5)
    W = torch.randn(r, c, generator=g, device="cuda") * 0.02
    b = gpu.quantize_batch([W], Config(sigma_n=2.5758), "outliers-only", out_mem=gpu.MEM_DEVICE)
    del W
    What = torch.empty(r, c, device="cuda")
    b.dequantize_into(0, What)
    monkeypatch.setenv("EZQ_GEMV_FUSED", "1")
    pf = gpu.GemvPlan(b, 0)
    monkeypatch.setenv("EZQ_GEMV_FUSED", "0")
    ps = gpu.GemvPlan(b, 0)
    Wd = What.double()
    for B in (1, 16):
        x = torch.randn(B, r, generator=g, device="cuda").to(torch.bfloat16)
        yf, ys = pf(x).double(), ps(x).double()
        ref = x.double() @ Wd
        sc = ref.abs().max().item()
        assert (yf - ref).abs().max().item() <= 1e-3 * sc
        assert (ys - ref).abs().max().item() <= 1e-3 * sc
        assert (yf - ys).abs().max().item() <= 1e-5 * sc
    pf.close()
    ps.close()
    b.close()
