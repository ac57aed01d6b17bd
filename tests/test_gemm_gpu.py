"""tcgen05 3xTF32 GEMM vs a float64 torch reference of the same op."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2505_11564_b200 import gemm
    return gemm


def rel(a, b):
    return float((a.double() - b).norm() / b.norm())


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("shape", [(128, 128, 32), (256, 384, 768), (200, 300, 100), (1000, 520, 264), (256, 64, 1024), (300, 40, 200)])
def test_gemm_majors(G, a_t, b_t, shape):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda", generator=g)
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda", generator=g)
    ref = (A.double().t() if a_t else A.double()) @ (B.double().t() if b_t else B.double())
    C3 = G.matmul(A, B, True, a_t, b_t)
    C1 = G.matmul(A, B, False, a_t, b_t)
    e3, e1 = rel(C3, ref), rel(C1, ref)
    # fp32-faithful: 3xTF32 within 2e-6 rel-L2; 1xTF32 is ~1e-3
    assert e3 < 2e-6, (e3, e1)
    assert e1 < 5e-3


def test_gemm_alpha_beta_batched(G):
    # per-head slices of a packed [B*S, 3*d] activation: Q_h K_h^T for all (b, h)
    Bsz, S, H, dh = 2, 128, 4, 64
    d = H * dh
    qkv = torch.randn(Bsz * S, 3 * d, device="cuda")
    out = torch.ones(Bsz * H, S, S, device="cuda")
    qs = G.split(qkv)
    G.gemm(S, S, dh, qkv, 3 * d, False, qkv[:, d:], 3 * d, False, out, S, alpha=0.125, beta=1.0,
           a_small=qs, b_small=qs[:, d:], z1=H, z2=Bsz, sa=(dh, S * 3 * d), sb=(dh, S * 3 * d), sc=(S * S, H * S * S))
    q = qkv.double().view(Bsz, S, 3, H, dh)
    ref = 0.125 * torch.einsum("bshe,bthe->bhst", q[:, :, 0], q[:, :, 1]).reshape(Bsz * H, S, S) + 1.0
    assert rel(out, ref) < 2e-6


def test_tf32_truncation_split_mode(G):
    """The residual split must match what the tensor core reads (truncation)."""
    A = torch.randn(256, 256, device="cuda")
    B = torch.randn(256, 256, device="cuda")
    ref = A.double() @ B.double()
    e_trunc = rel(G.matmul(A, B, True, mode=0), ref)
    e_rna = rel(G.matmul(A, B, True, mode=1), ref)
    print(f"3xTF32 rel err: trunc-split {e_trunc:.3e}  rna-split {e_rna:.3e}")
    assert min(e_trunc, e_rna) < 2e-6


@pytest.mark.parametrize("a_t,b_t", [(True, True), (False, False)])
def test_gemm_split_k(G, a_t, b_t):
    """Few output tiles + long K (the Hv weight products over T tokens) take
    the deterministic split-K path; alpha/beta/bias/residual still apply."""
    M, N, K = 256, 384, 8192
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    bias = torch.randn(N, device="cuda")
    C = torch.randn(M, N, device="cuda")
    C0 = C.clone()
    Cs = torch.empty_like(C)
    G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, alpha=0.5, beta=2.0,
           a_small=G.split(A), b_small=G.split(B))
    ref = 0.5 * ((A.double().t() if a_t else A.double()) @ (B.double().t() if b_t else B.double())) + 2.0 * C0.double()
    assert rel(C, ref) < 2e-6
    first = C.clone()
    C.copy_(C0)
    G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, alpha=0.5, beta=2.0,
           a_small=G.split(A), b_small=G.split(B))
    assert torch.equal(C, first)  # deterministic split order


def test_gemm_split_k_concurrent_threads(G):
    """Split-K products issued concurrently from several threads on their own
    streams (the in-process worker pool's pattern) use per-thread workspaces:
    every thread's result equals the single-threaded one bitwise."""
    import threading
    M, N, K = 768, 768, 8192  # an Hv weight product: split 8 ways on the B200
    g = torch.Generator(device="cuda").manual_seed(11)
    ins = [(torch.randn(K, M, device="cuda", generator=g), torch.randn(K, N, device="cuda", generator=g))
           for _ in range(4)]
    sm = [(G.split(a), G.split(b)) for a, b in ins]

    def one(i, out):
        a, b = ins[i]
        c = torch.empty(M, N, device="cuda")
        for _ in range(3):
            G.gemm(M, N, K, a, M, True, b, N, True, c, N, a_small=sm[i][0], b_small=sm[i][1])
        out[i] = c

    want = [None] * 4
    for i in range(4):
        one(i, want)
    torch.cuda.synchronize()
    got = [None] * 4
    dev = torch.cuda.current_device()

    def body(i):
        torch.cuda.set_device(dev)
        with torch.cuda.stream(torch.cuda.Stream()):
            one(i, got)
            torch.cuda.current_stream().synchronize()

    ts = [threading.Thread(target=body, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(4):
        assert torch.equal(got[i], want[i]), i


def test_gemm_wide_tiles(G):
    """Shapes that select the 256-wide tile path (enough output tiles)."""
    for (M, N, K, a_t, b_t) in [(4096, 2304, 256, False, False), (4096, 1024, 512, False, True),
                                (2560, 2048, 300, True, False)]:
        A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
        B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
        ref = (A.double().t() if a_t else A.double()) @ (B.double().t() if b_t else B.double())
        assert rel(G.matmul(A, B, True, a_t, b_t), ref) < 2e-6


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("shape", [(256, 384, 768), (200, 300, 100), (1024, 64, 1024), (768, 768, 8192)])
def test_gemm_dual_source(G, a_t, b_t, shape):
    # C = alpha (A1 B1 + A2 B2) + beta C in one launch (the HVP tangent products)
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + K)
    mk = lambda r, c: torch.randn(r, c, device="cuda", generator=g)  # noqa: E731
    A1, A2 = [mk(*((K, M) if a_t else (M, K))) for _ in range(2)]
    B1, B2 = [mk(*((N, K) if b_t else (K, N))) for _ in range(2)]
    C0 = mk(M, N)
    op = lambda X, t: X.double().t() if t else X.double()  # noqa: E731
    alpha, beta = 0.75, 1.0
    ref = alpha * (op(A1, a_t) @ op(B1, b_t) + op(A2, a_t) @ op(B2, b_t)) + beta * C0.double()
    C = C0.clone()
    G.gemm_dual(M, N, K, A1, A1.shape[1], a_t, B1, B1.shape[1], not b_t, A2, A2.shape[1], B2, B2.shape[1], C, N,
                alpha=alpha, beta=beta, a_small=G.split(A1), b_small=G.split(B1), a2_small=G.split(A2),
                b2_small=G.split(B2))
    assert rel(C, ref) < 2e-6


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("shape", [(256, 384, 768), (200, 300, 100), (1024, 64, 1024), (768, 768, 8192), (8192, 256, 64)])
def test_gemm_onchip_residual_bitwise(G, a_t, b_t, shape):
    # residual tiles computed in shared memory == residual arrays from sd_split_tf32(mode 0), bit for bit
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + 7 * K)
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda", generator=g)
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda", generator=g)
    A2 = torch.randn_like(A)
    B2 = torch.randn_like(B)
    args = (M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t)
    C0 = torch.empty(M, N, device="cuda")
    C1 = torch.empty(M, N, device="cuda")
    G.gemm(*args, C0, N, a_small=G.split(A), b_small=G.split(B))
    G.gemm(*args, C1, N, onchip=True)
    assert torch.equal(C0, C1)
    D0 = torch.zeros(M, N, device="cuda")
    D1 = torch.zeros(M, N, device="cuda")
    G.gemm_dual(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, A2, A2.shape[1], B2, B2.shape[1], D0, N,
                alpha=0.5, a_small=G.split(A), b_small=G.split(B), a2_small=G.split(A2), b2_small=G.split(B2))
    G.gemm_dual(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, A2, A2.shape[1], B2, B2.shape[1], D1, N,
                alpha=0.5, onchip=True)
    assert torch.equal(D0, D1)


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("shape", [(256, 384, 768), (200, 300, 100), (1024, 64, 1024), (768, 768, 8192), (8192, 512, 64)])
def test_gemm_b_exact_bitwise(G, a_t, b_t, shape):
    # bf16-valued B (tf32-exact): SD_GEMM_B_EXACT skips the zero residual's load
    # and its MMA -- bit-identical to passing the all-zero residual array, and
    # still fp32-faithful against float64
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M + 5 * N + 11 * K)
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda", generator=g)
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda", generator=g).bfloat16().float()
    assert torch.count_nonzero(G.split(B)) == 0
    args = (M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t)
    C0 = torch.empty(M, N, device="cuda")
    C1 = torch.empty(M, N, device="cuda")
    G.gemm(*args, C0, N, a_small=G.split(A), b_small=G.split(B))
    G.gemm(*args, C1, N, a_small=G.split(A), b_exact=True)
    assert torch.equal(C0, C1)
    ref = (A.double().t() if a_t else A.double()) @ (B.double().t() if b_t else B.double())
    assert rel(C1, ref) < 2e-6
