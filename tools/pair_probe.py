import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19241_b200 import _lib as L
lib = L.lib()
E, rows, N, K = 8, 4096, 4096, 14336
M = E * rows
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(E, N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); ws = torch.empty(64 << 20, device="cuda", dtype=torch.uint8)
ia = lambda v: (ctypes.c_int * len(v))(*v)
for fn in (lib.eplab_grouped_gemm_nt, lib.eplab_grouped_gemm_nt_pair):
    fn(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()), M, N, K, E,
       ia([e * rows for e in range(E)]), ia([rows] * E), ctypes.c_void_p(ws.data_ptr()), None)
torch.cuda.synchronize()
