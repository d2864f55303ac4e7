"""Op-level timing of the decode MLP at the LLaMA-8B shape: the fused gate/up + down
kernel (srl_op_mlp_bf16) against the two separate GEMMs (SiLU-mul, then down with the
residual epilogue), CUDA events, weights rotated over > L2 bytes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_23414_b200 import _lib  # noqa: E402

lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
d, ff = 4096, 14336
NROT = 3


def pack(W):
    dst = torch.empty(lib.srl_op_packed_weight_bytes(W.shape[0], W.shape[1]), dtype=torch.uint8, device="cuda")
    assert lib.srl_op_pack_weight(W.data_ptr(), W.shape[0], W.shape[1], dst.data_ptr(), s) == 0
    return dst


gu = [pack((torch.randn(2 * ff, d, device="cuda") * 0.02).to(torch.bfloat16)) for _ in range(NROT)]
dn = [pack((torch.randn(d, ff, device="cuda") * 0.02).to(torch.bfloat16)) for _ in range(NROT)]
ws = torch.zeros(lib.srl_op_gemm_workspace(256, d, ff, 1), dtype=torch.uint8, device="cuda")


def timeit(fn, it=30):
    for i in range(3):
        fn(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(it):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


res = {}
for M in (256, 224, 192, 160, 128):
    X = (torch.randn(M, d, device="cuda") * 0.5).to(torch.bfloat16)
    act = torch.empty(M, ff, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(M, d, dtype=torch.float32, device="cuda")
    part = torch.empty(8, M, d, dtype=torch.float32, device="cuda")
    for S2 in (8, 4):
        us = timeit(lambda i: lib.srl_op_mlp_bf16(X.data_ptr(), M, gu[i % NROT].data_ptr(), dn[i % NROT].data_ptr(),
                                                  d, ff, S2, act.data_ptr(), part.data_ptr(), ws.data_ptr(), s))
        res[f"fused_S{S2}_M{M}"] = us

    def sep(i):
        lib.srl_op_gemm_bf16(X.data_ptr(), M, gu[i % NROT].data_ptr(), ff, d, 2 | 0x100, act.data_ptr(),
                             ws.data_ptr(), s)
        lib.srl_op_gemm_bf16(act.data_ptr(), M, dn[i % NROT].data_ptr(), d, ff, 1 | 0x100, out.data_ptr(),
                             ws.data_ptr(), s)
    res[f"separate_M{M}"] = timeit(sep)
    print(M, {k: round(v, 1) for k, v in res.items() if k.endswith(f"M{M}")}, flush=True)
print(json.dumps(res))
