"""Op-level timing of the decode GEMMs / attention at cfg2 shapes (CUDA events,
weights rotated over > L2 bytes so every launch streams from HBM)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_23414_b200 import _lib

lib = _lib.load()
if os.environ.get("BENCH_TUNING"):  # e.g. "gemm_h=2,gemm_stages=4" (tools/gemm_sweep.sh)
    _lib.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in os.environ["BENCH_TUNING"].split(","))})
s = torch.cuda.current_stream().cuda_stream
res = {}
PACKED = os.environ.get("BENCH_PACKED", "1") == "1"
def t_gemm(name, M, N, K, epi, nrot=4, it=20):
    rows = 2 * N if epi == 2 else N
    Ws = [(torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(nrot)]
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 2 else torch.float32)
    ws = torch.empty(lib.srl_op_gemm_workspace(M, N, K, epi), dtype=torch.uint8, device="cuda")
    if PACKED:
        packed = []
        for Wr in Ws:
            d = torch.empty(lib.srl_op_packed_weight_bytes(rows, K), dtype=torch.uint8, device="cuda")
            lib.srl_op_pack_weight(Wr.data_ptr(), rows, K, d.data_ptr(), s)
            packed.append(d)
        Ws = packed
        epi |= 0x100
    for i in range(3):
        lib.srl_op_gemm_bf16(X.data_ptr(), M, Ws[i % nrot].data_ptr(), N, K, epi, out.data_ptr(), ws.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(it):
        lib.srl_op_gemm_bf16(X.data_ptr(), M, Ws[i % nrot].data_ptr(), N, K, epi, out.data_ptr(), ws.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    gbs = rows * K * 2 / (ms * 1e-3) / 1e9
    res[name] = dict(M=M, N=N, K=K, us=ms * 1e3, weight_GBs=gbs, TFs=2 * M * rows * K / (ms * 1e-3) / 1e12)
    print(name, json.dumps(res[name]), flush=True)

for M in map(int, os.environ.get("BENCH_M", "256,128,64,16").split(",")):
    t_gemm(f"qkv_M{M}", M, 6144, 4096, 0)
    t_gemm(f"o_M{M}", M, 4096, 4096, 1)
    t_gemm(f"gu_M{M}", M, 14336, 4096, 2)
    t_gemm(f"down_M{M}", M, 4096, 14336, 1)
t_gemm("lmhead_M256", 256, 128256, 4096, 0, nrot=2)
t_gemm("prefill_qkv_M4096", 4096, 6144, 4096, 0, nrot=2, it=5)
t_gemm("prefill_gu_M4096", 4096, 14336, 4096, 2, nrot=2, it=5)
