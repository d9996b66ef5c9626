"""MaxK-GNN consumer shapes: scatter / gather kernels against
torch's scatter_/gather on the same indices, the autograd ops against a plain
PyTorch formulation of MaxK, and the CSR view against the dense form."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_00822_b200 as rtk  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_00822_b200 import _build

    _build.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("n,m,k", [(1, 1, 1), (7, 5, 3), (1000, 256, 32), (333, 97, 11), (64, 1500, 128),
                                   (4099, 2048, 64), (10, 4096, 4096)])
def test_scatter_gather_match_torch(n, m, k):
    g = torch.Generator(device="cuda").manual_seed(n * 7 + m)
    x = torch.randn(n, m, device="cuda", generator=g)
    res = rtk.batch_topk(x, rtk.BatchConfig(k=k))
    dense = rtk.scatter_rows(res.values, res.indices, m)
    want = torch.zeros(n, m, device="cuda").scatter_(1, res.indices.long(), res.values)
    assert torch.equal(dense, want)
    back = rtk.gather_rows(dense, res.indices)
    assert torch.equal(back, torch.gather(dense, 1, res.indices.long()))
    assert torch.equal(back, res.values)


def test_scatter_strided_and_unaligned_rows():
    x = torch.randn(300, 130, device="cuda")
    res = rtk.batch_topk(x, rtk.BatchConfig(k=9))
    dense = rtk.scatter_rows(res.values, res.indices, 130)  # m % 4 != 0: scalar stores
    assert torch.equal(dense, torch.zeros(300, 130, device="cuda").scatter_(1, res.indices.long(), res.values))
    big = torch.randn(300, 200, device="cuda")
    view = big[:, 3:133]  # gather from a strided, unaligned view
    assert torch.equal(rtk.gather_rows(view, res.indices), torch.gather(view, 1, res.indices.long()))


def _torch_maxk_dense(x, k):
    """Plain PyTorch MaxK (reference formulation): keep the top-k per row."""
    v, i = torch.topk(x, k, dim=1)
    return torch.zeros_like(x).scatter(1, i, v)


@pytest.mark.parametrize("search", [rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(4)])
def test_maxk_autograd(search):
    n, m, k = 2048, 256, 32
    x = torch.randn(n, m, device="cuda", requires_grad=True)
    vals, idx = rtk.maxk(x, k, search)
    want = rtk.batch_topk(x.detach(), rtk.BatchConfig(k=k, search=search))
    assert torch.equal(vals, want.values) and torch.equal(idx, want.indices)
    gv = torch.randn_like(vals)
    (vals * gv).sum().backward()
    expect = torch.zeros(n, m, device="cuda").scatter_(1, idx.long(), gv)
    assert torch.equal(x.grad, expect)


def test_maxk_dense_matches_torch_formulation():
    n, m, k = 1024, 256, 32
    x = torch.randn(n, m, device="cuda", dtype=torch.float32)
    x1 = x.clone().requires_grad_(True)
    x2 = x.clone().requires_grad_(True)
    y1 = rtk.maxk_dense(x1, k)
    y2 = _torch_maxk_dense(x2, k)  # exact mode = the true top-k on distinct N(0,1) values
    assert torch.equal(y1, y2)
    g = torch.randn(n, m, device="cuda")
    (y1 * g).sum().backward()
    (y2 * g).sum().backward()
    assert torch.equal(x1.grad, x2.grad)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_maxk_16bit_activations(dtype, oracle_lib):
    """MaxK on bf16 / fp16 activations (native 16-bit rows): the selection
    equals the oracle's on the float32 image (what the reference computes
    after as_matrix), including the tie-heavy rows 16-bit N(0,1) data has;
    dense output and gradients in the activation dtype; values float32."""
    n, m, k = 4096, 256, 32
    x = torch.randn(n, m, device="cuda").to(dtype)
    xf = x.float().cpu().numpy()
    for search, mode in ((rtk.SearchConfig.exact(), "exact"), (rtk.SearchConfig.early_stop(4), "early")):
        ov, oi, _, _ = oracle_lib.ref_batch(xf, k, mode, max_iter=4)
        vals, idx = rtk.maxk(x.clone().requires_grad_(True), k, search)
        assert vals.dtype == torch.float32
        assert np.array_equal(idx.detach().cpu().numpy(), oi), mode
        assert np.array_equal(vals.detach().cpu().numpy().view(np.uint32), ov.view(np.uint32)), mode
        x1 = x.clone().requires_grad_(True)
        y1 = rtk.maxk_dense(x1, k, search)
        keep = torch.zeros(n, m, dtype=torch.bool, device="cuda").scatter_(
            1, torch.from_numpy(oi).long().cuda(), True)
        y2 = torch.where(keep, x, torch.zeros((), dtype=dtype, device="cuda"))
        assert y1.dtype == dtype and torch.equal(y1, y2), mode
        g = torch.randn(n, m, device="cuda").to(dtype)
        (y1.float() * g.float()).sum().backward()
        assert x1.grad.dtype == dtype
        assert torch.equal(x1.grad, torch.where(keep, g, torch.zeros((), dtype=dtype, device="cuda"))), mode
    # bf16 N(0,1) rows tie at the k-th value often: the check above covers them
    if dtype == torch.bfloat16:
        kth = x.float().topk(k, dim=1).values[:, -1:]
        assert int(((x.float() >= kth).sum(1) > k).sum()) > 0


def test_sparse_csr_view_spmm():
    n, m, k = 500, 256, 32
    x = torch.randn(n, m, device="cuda")
    vals, idx = rtk.maxk(x, k)
    csr = rtk.to_sparse_csr(vals, idx, m)
    dense = rtk.scatter_rows(vals, idx, m)
    assert torch.equal(csr.to_dense(), dense)
    w = torch.randn(m, 64, device="cuda")
    assert torch.allclose(torch.sparse.mm(csr, w), dense @ w, rtol=1e-4, atol=1e-4)


def test_topk_device_is_sync_free_and_graph_capturable():
    """topk_device / maxk(check_nan=False) enqueue without host syncs, so a
    MaxK layer (top-k + scatter + SpMM-style matmul) captures into a CUDA
    graph; replays equal eager results and the NaN word reports the row."""
    n, m, k = 4096, 256, 32
    x = torch.randn(n, m, device="cuda")
    w = torch.randn(m, 64, device="cuda")
    nan_word = torch.empty(1, dtype=torch.int32, device="cuda")
    want_v, want_i = rtk.topk_device(x, k, nan_word=nan_word)
    assert int(nan_word.item()) == -1
    ref = rtk.batch_topk(x, rtk.BatchConfig(k=k))
    assert torch.equal(want_v, ref.values) and torch.equal(want_i, ref.indices)

    static_x = x.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up outside capture (allocator, library load)
            out = rtk.maxk_dense(static_x, k, check_nan=False) @ w
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = rtk.maxk_dense(static_x, k, check_nan=False) @ w
    for trial in range(3):
        static_x.copy_(torch.randn(n, m, device="cuda"))
        g.replay()
        torch.cuda.synchronize()
        eager = rtk.maxk_dense(static_x, k) @ w
        assert torch.equal(out, eager), trial

    bad = x.clone()
    bad[1234, 5] = float("nan")
    rtk.topk_device(bad, k, nan_word=nan_word)
    assert int(nan_word.item()) == 1234
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.topk_device(x, m + 1)


def test_maxk_bf16_layer_captures_in_cuda_graph():
    """The native 16-bit path (rtk_rowtopk_x16) enqueues without host syncs
    too: a bf16 MaxK layer captured in a CUDA graph replays equal to eager."""
    n, m, k = 8192, 256, 16
    static_x = torch.randn(n, m, device="cuda").to(torch.bfloat16)
    w = torch.randn(m, 32, device="cuda").to(torch.bfloat16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            out = rtk.maxk_dense(static_x, k, check_nan=False) @ w
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = rtk.maxk_dense(static_x, k, check_nan=False) @ w
    for trial in range(3):
        static_x.copy_(torch.randn(n, m, device="cuda").to(torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, rtk.maxk_dense(static_x, k) @ w), trial


def _rows(kind, n, m, dtype, g):
    if kind == "normal":
        return torch.randn(n, m, device="cuda", generator=g).to(dtype)
    if kind == "ties":  # few distinct values: ties at the k-th value on most rows (fill / tie paths)
        return torch.randint(-3, 4, (n, m), device="cuda", generator=g).to(dtype)
    x = torch.randn(n, m, device="cuda", generator=g).to(dtype)  # signed zeros and +-inf sprinkled in
    x[:, ::17] = -0.0
    x[::5, 3] = float("inf")
    x[::7, 9] = float("-inf")
    return x


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("m", [128, 256])
def test_maxk_dense_fused_matches_select_and_scatter(dtype, m):
    """rtk_maxk_dense (one kernel) equals batch_topk + scatter_rows bit for bit:
    values, indices and the dense rows in x's dtype, for exact and early-stop
    search, normal / tie-heavy / special-value rows, odd N (unpaired last row)
    and a strided input view."""
    g = torch.Generator(device="cuda").manual_seed(m + _DT.index(dtype))
    for kind in ("normal", "ties", "special"):
        for n in (1, 2, 1001):
            base = _rows(kind, n, m + 8, dtype, g)
            for x in (base[:, :m].contiguous(), base[:, 4:4 + m]):
                for k in (1, 17, 32, m - 1):
                    for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(3)):
                        dense, vals, idx = rtk.maxk_dense_fused(x, k, search)
                        want = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=search))
                        assert torch.equal(idx, want.indices), (kind, n, k, search.mode)
                        assert torch.equal(vals.view(torch.int32), want.values.view(torch.int32)), (kind, n, k)
                        sc = rtk.scatter_rows(want.values, want.indices, m).to(dtype)
                        assert dense.dtype == dtype
                        assert torch.equal(dense.view(torch.int16 if dtype != torch.float32 else torch.int32),
                                           sc.view(torch.int16 if dtype != torch.float32 else torch.int32)), (kind, n, k)


_DT = [torch.float32, torch.bfloat16, torch.float16]


def test_maxk_dense_fused_errors_and_fallback():
    x = torch.randn(64, 256, device="cuda")
    x[9, 100] = float("nan")
    x[40, 3] = float("nan")
    with pytest.raises(rtk.NaNInputError, match="first offending row: 9"):
        rtk.maxk_dense_fused(x, 8)
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.maxk_dense_fused(torch.randn(4, 128, device="cuda"), 0)
    with pytest.raises(ValueError, match="unsupported"):
        rtk.maxk_dense_fused(torch.randn(4, 200, device="cuda"), 8)  # m outside {128, 256}
    y = torch.randn(300, 200, device="cuda")  # maxk_dense falls back to select + scatter
    assert torch.equal(rtk.maxk_dense(y, 9), _torch_maxk_dense(y, 9))


def test_maxk_dense_uses_fused_kernel_and_grads():
    """maxk_dense on 256-wide rows goes through the fused kernel (same
    output as the formulation, gradients to the kept entries)."""
    n, m, k = 4096, 256, 32
    x = torch.randn(n, m, device="cuda", requires_grad=True)
    y = rtk.maxk_dense(x, k)
    assert torch.equal(y, _torch_maxk_dense(x.detach(), k))
    g = torch.randn(n, m, device="cuda")
    (y * g).sum().backward()
    assert torch.equal(x.grad, torch.where(y != 0, g, torch.zeros((), device="cuda")))


def _random_graph(n_out, n_in, g, max_deg=80):
    deg = torch.randint(0, max_deg, (n_out,), device="cuda", generator=g)
    deg[::97] = 0  # empty rows
    deg[5] = 300   # several 32-edge chunks
    row_ptr = torch.zeros(n_out + 1, dtype=torch.int64, device="cuda")
    row_ptr[1:] = torch.cumsum(deg, 0)
    nnz = int(row_ptr[-1])
    col = torch.randint(0, n_in, (nnz,), device="cuda", generator=g, dtype=torch.int32)
    aval = torch.rand(nnz, device="cuda", generator=g) + 0.5
    return row_ptr, col, aval


def _dense_adj(row_ptr, col, aval, n_in):
    n_out = row_ptr.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n_out, device="cuda"), row_ptr[1:] - row_ptr[:-1])
    a = torch.zeros(n_out, n_in, dtype=torch.float64, device="cuda")
    a.index_put_((rows, col.long()), aval.double(), accumulate=True)
    return a


@pytest.mark.parametrize("m,k", [(256, 32), (128, 8), (256, 64), (700, 48), (1024, 128)])
def test_maxk_spmm_forward_backward_against_float64(m, k):
    """MaxK-GNN aggregation over the fixed-k rows: forward and the gradient
    w.r.t. the kept values against float64 dense formulations (A @ scatter(H)
    and (A^T @ grad)[j, idx[j]]), deterministic across calls, uint8 indices
    equal to int32 ones (M <= 256), unit weights (aval = None)."""
    g = torch.Generator(device="cuda").manual_seed(m * 31 + k)
    n_in, n_out = 2500, 3000
    h = torch.randn(n_in, m, device="cuda", generator=g)
    res = rtk.batch_topk(h, rtk.BatchConfig(k=k))
    vals, idx = res.values, res.indices
    row_ptr, col, aval = _random_graph(n_out, n_in, g)
    a = _dense_adj(row_ptr, col, aval, n_in)
    hs = torch.zeros(n_in, m, dtype=torch.float64, device="cuda").scatter_(1, idx.long(), vals.double())
    want = a @ hs
    out = rtk.maxk_spmm(row_ptr, col, aval, vals, idx, m)
    assert torch.allclose(out.double(), want, rtol=1e-5, atol=1e-4)
    assert torch.equal(out, rtk.maxk_spmm(row_ptr, col, aval, vals, idx, m))  # deterministic
    if m <= 256:
        assert torch.equal(out, rtk.maxk_spmm(row_ptr, col, aval, vals, idx.to(torch.uint8), m))
    ones = rtk.maxk_spmm(row_ptr, col, None, vals, idx, m)
    a1 = _dense_adj(row_ptr, col, torch.ones_like(aval), n_in)
    assert torch.allclose(ones.double(), a1 @ hs, rtol=1e-5, atol=1e-4)
    # gradient w.r.t. the kept values
    v = vals.clone().requires_grad_(True)
    y = rtk.maxk_aggregate((row_ptr, col, aval), v, idx, m)
    gout = torch.randn(n_out, m, device="cuda", generator=g)
    (y * gout).sum().backward()
    gref = torch.gather(a.t() @ gout.double(), 1, idx.long())
    assert torch.allclose(v.grad.double(), gref, rtol=1e-5, atol=1e-4)
    gt = rtk.csr_transpose(row_ptr, col, aval, n_in)
    v2 = vals.clone().requires_grad_(True)
    (rtk.maxk_aggregate((row_ptr, col, aval), v2, idx, m, graph_t=gt) * gout).sum().backward()
    assert torch.equal(v2.grad, v.grad)


def test_maxk_sparse_u8_and_spmm_errors():
    x = torch.randn(513, 256, device="cuda")
    vals, idx8 = rtk.maxk_sparse_u8(x, 32)
    want = rtk.batch_topk(x, rtk.BatchConfig(k=32))
    assert idx8.dtype == torch.uint8 and torch.equal(idx8.long(), want.indices.long())
    assert torch.equal(vals, want.values)
    v, i8 = rtk.maxk_sparse_u8(x[:, :128].contiguous(), 16, rtk.SearchConfig.early_stop(4))
    w2 = rtk.batch_topk(x[:, :128].contiguous(), rtk.BatchConfig(k=16, search=rtk.SearchConfig.early_stop(4)))
    assert torch.equal(i8.long(), w2.indices.long()) and torch.equal(v, w2.values)
    rp = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
    c = torch.tensor([0], dtype=torch.int32, device="cuda")
    with pytest.raises(rtk.DeviceError, match="m <= 256"):
        rtk.maxk_spmm(rp, c, None, want.values, want.indices.to(torch.uint8), 300)
    with pytest.raises(rtk.DeviceError, match="m <= 1024"):
        rtk.maxk_spmm(rp, c, None, want.values, want.indices, 2000)
    with pytest.raises(ValueError, match="int64"):
        rtk.maxk_spmm(rp.int(), c, None, want.values, want.indices, 256)
