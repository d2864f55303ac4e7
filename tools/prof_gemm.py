"""One GEMM shape, a few launches (for ncu).  usage: prof_gemm.py M N K epi"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_23414_b200 import _lib
lib = _lib.load()
M, N, K, epi = map(int, sys.argv[1:5])
rows = 2 * N if epi == 2 else N
Ws = [(torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(4)]
X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 2 else torch.float32)
ws = torch.empty(lib.srl_op_gemm_workspace(M, N, K, epi), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for i in range(6):
    lib.srl_op_gemm_bf16(X.data_ptr(), M, Ws[i % 4].data_ptr(), N, K, epi, out.data_ptr(), ws.data_ptr(), s)
torch.cuda.synchronize()
print("done")
