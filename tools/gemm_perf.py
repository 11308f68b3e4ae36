"""Quick throughput probe of the grouped NT/TN GEMMs (CUDA events, L2-sized inputs)."""
import ctypes
import sys
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2604_19241_b200 import _lib as L

lib = L.lib()


def iarr(v):
    return (ctypes.c_int * len(v))(*v)


def bench_nt(E, rows, N, K, iters=10, pair=False):
    M = E * rows
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(E, N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.uint8)
    starts = [e * rows for e in range(E)]
    cnt = [rows] * E
    g = lib.eplab_grouped_gemm_nt_pair if pair else lib.eplab_grouped_gemm_nt
    f = lambda: g(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), M, N, K, E, iarr(starts), iarr(cnt),
                                          ctypes.c_void_p(ws.data_ptr()), None)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2.0 * M * N * K / ms / 1e9
    ref = A[:rows].float() @ B[0].float().t()
    err = (C[:rows].float() - ref).abs().max().item()
    print(f"{'pair ' if pair else ''}NT E={E} rows={rows} N={N} K={K}: {ms:.3f} ms  {tf:.1f} TFLOP/s  maxerr={err:.3g}", flush=True)


def bench_tn(E, rows, NA, NB, iters=10, pair=False):
    M = E * rows
    A = torch.randn(M, NA, device="cuda").bfloat16()
    B = torch.randn(M, NB, device="cuda").bfloat16()
    C = torch.empty(E, NA, NB, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.uint8)
    starts = [e * rows for e in range(E)]
    cnt = [rows] * E
    g = lib.eplab_grouped_gemm_tn_pair if pair else lib.eplab_grouped_gemm_tn
    f = lambda: g(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), M, NA, NB, E, iarr(starts), iarr(cnt),
                                          ctypes.c_void_p(ws.data_ptr()), None)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2.0 * M * NA * NB / ms / 1e9
    ref = A[:rows].float().t() @ B[:rows].float()
    err = (C[0].float() - ref).abs().max().item()
    print(f"{'pair ' if pair else ''}TN E={E} rows={rows} NA={NA} NB={NB}: {ms:.3f} ms  {tf:.1f} TFLOP/s  maxerr={err:.3g}", flush=True)


if __name__ == "__main__":
    torch.manual_seed(0)
    for pair in (False, True):
        bench_nt(8, 4096, 28672, 4096, pair=pair)
        bench_nt(8, 4096, 4096, 14336, pair=pair)
        bench_nt(128, 1024, 1536, 2048, pair=pair)
        bench_tn(8, 4096, 28672, 4096, iters=3, pair=pair)
        bench_tn(128, 1024, 1536, 2048, pair=pair)
    x = torch.randn(8192, 8192, device="cuda").bfloat16()
    for _ in range(3):
        y = x @ x
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10):
        y = x @ x
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"cuBLAS 8192^3: {ms:.3f} ms {2*8192**3/ms/1e9:.1f} TFLOP/s")
