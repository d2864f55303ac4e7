"""Op-level timing of the paged decode attention (srl_op_attention, bf16 KV) at
the decode shapes: rows x contexts, achieved GB/s of algorithmic KV bytes.
Includes the plan kernel (as in the engine, once per launch here).

  python tools/bench_attn.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_23414_b200 import _lib  # noqa: E402

lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
if len(sys.argv) > 1:  # srl_tuning overrides, e.g. attn_stages=6
    _lib.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in sys.argv[1].split(","))})


def case(name, M, Hq, Hkv, ctx_mean, sigma=0.5, dh=128, it=20, seed=0):
    rng = np.random.default_rng(seed)
    ctxs = np.clip(np.rint(np.exp(np.log(ctx_mean) + sigma * rng.standard_normal(M))), 2, 16384).astype(np.int64)
    pages = [(c + 63) // 64 for c in ctxs]
    n_pages = int(sum(pages)) + 8
    max_ctx = int(ctxs.max())
    max_pages = (max_ctx + 63) // 64
    pt = np.zeros((M, max_pages), dtype=np.int32)
    perm = rng.permutation(n_pages)
    u = 0
    for r in range(M):
        pt[r, :pages[r]] = perm[u:u + pages[r]]
        u += pages[r]
    q = torch.randn(M, Hq, dh, device="cuda").to(torch.bfloat16)
    kp = torch.randn(n_pages, Hkv, 64, dh, device="cuda").to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 64, dh, device="cuda").to(torch.bfloat16)
    tpt = torch.from_numpy(pt).cuda()
    tpos = torch.from_numpy((ctxs - 1).astype(np.int32)).cuda()
    ws = torch.zeros(lib.srl_op_attention_workspace(M, Hq, Hkv, dh, max_ctx), dtype=torch.uint8, device="cuda")
    out = torch.empty(M, Hq, dh, device="cuda")

    def run():
        return lib.srl_op_attention(q.data_ptr(), kp.data_ptr(), vp.data_ptr(), n_pages, tpt.data_ptr(), max_pages,
                                    tpos.data_ptr(), M, Hq, Hkv, dh, 0, max_ctx, ws.data_ptr(), out.data_ptr(), st)
    for _ in range(3):
        assert run() == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / it * 1e3
    alg = 2 * Hkv * dh * 2 * int(ctxs.sum())
    print(f"{name:28s} M={M:4d} pairs={M * Hkv:5d} mean_ctx={ctxs.mean():7.0f} {us:8.1f} us  "
          f"{alg / us / 1e3:7.0f} GB/s", flush=True)


case("8B steady (cfg2)", 256, 32, 8, 1700)
case("8B half occupancy", 128, 32, 8, 2500)
case("32B steady (cfg4 slice)", 64, 40, 8, 1130)
case("8B drain", 32, 32, 8, 6000)
case("8B deep drain", 16, 32, 8, 7600)
case("8B tail", 4, 32, 8, 8000, sigma=0.1)
