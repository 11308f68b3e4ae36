"""tcgen05 grouped-GEMM engine vs a torch fp32 reference (bf16 in, fp32 accumulate)."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _lib():
    from paper_2604_19241_b200 import _lib as L
    return L.lib()


def _seg(counts):
    starts, s = [], 0
    for c in counts:
        starts.append(s)
        s += (c + 127) // 128 * 128
    return starts, s


def _iarr(v):
    return (ctypes.c_int * len(v))(*v)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("counts,N,K", [([128], 256, 64), ([300, 0, 77, 1024], 512, 256),
                                        ([1000, 513], 1536, 2048)])
def test_grouped_nt(counts, N, K, pair):
    lib = _lib()
    torch.manual_seed(0)
    starts, M = _seg(counts)
    E = len(counts)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(E, N, K, device="cuda") / K ** 0.5).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.uint8)
    fn = lib.eplab_grouped_gemm_nt_pair if pair else lib.eplab_grouped_gemm_nt
    rc = fn(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                   ctypes.c_void_p(C.data_ptr()), M, N, K, E, _iarr(starts),
                                   _iarr(counts), ctypes.c_void_p(ws.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    for e in range(E):
        s, c = starts[e], counts[e]
        if c == 0:
            continue
        ref = A[s:s + c].float() @ B[e].float().t()
        got = C[s:s + c].float()
        err = (got - ref).abs().max().item()
        assert err <= 2e-2 * ref.abs().max().item() + 1e-2, (e, err)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("counts,NA,NB", [([128], 256, 256), ([300, 0, 77], 256, 512),
                                          ([1000, 513], 768, 1024)])
def test_grouped_tn(counts, NA, NB, pair):
    lib = _lib()
    torch.manual_seed(1)
    starts, M = _seg(counts)
    E = len(counts)
    A = torch.zeros(M, NA, device="cuda", dtype=torch.bfloat16)
    Bm = torch.zeros(M, NB, device="cuda", dtype=torch.bfloat16)
    for e in range(E):
        s, c = starts[e], counts[e]
        A[s:s + c] = torch.randn(c, NA, device="cuda").bfloat16()
        Bm[s:s + c] = torch.randn(c, NB, device="cuda").bfloat16()
    C = torch.full((E, NA, NB), 7.0, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.uint8)
    padded = [(c + 127) // 128 * 128 for c in counts]
    fn = lib.eplab_grouped_gemm_tn_pair if pair else lib.eplab_grouped_gemm_tn
    rc = fn(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(Bm.data_ptr()),
                                   ctypes.c_void_p(C.data_ptr()), M, NA, NB, E, _iarr(starts),
                                   _iarr(padded), ctypes.c_void_p(ws.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    for e in range(E):
        s, c = starts[e], counts[e]
        ref = A[s:s + c].float().t() @ Bm[s:s + c].float()
        got = C[e].float()
        err = (got - ref).abs().max().item()
        assert err <= 2e-2 * max(ref.abs().max().item(), 1.0) + 1e-2, (e, err)
