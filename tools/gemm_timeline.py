"""Per-CTA phase timeline (globaltimer stamps) of GEMM launches.

  gemm_timeline.py op M N K epi      one srl_op_gemm_bf16 launch
  gemm_timeline.py engine [L]        layer-0 QKV / O / GU / DOWN launches of an
                                     8B-width decode step (no graphs, L layers)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_23414_b200 import _lib

lib = _lib.load()
lib.srl_debug_gemm_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int32]
NAMES = ["start", "setup", "tma0", "tma_done", "mma0", "mma_done", "e_full0", "e_full1", "e_full2", "e_done0",
         "e_done1", "e_done2", "end", "csync1/xwait0", "pushed/epi_end", "reduced/xwait1"]


def report(title, dbg):
    d = dbg.view(200, 16).cpu().numpy().astype(np.float64)
    d = d[d[:, 0] > 0]
    if not len(d):
        print(title, "no stamps")
        return
    t0 = d[:, 0].min()
    r = (d - t0) / 1e3
    r[d == 0] = np.nan
    print(f"== {title}: {len(d)} CTAs (us from first CTA start)")
    for i, nme in enumerate(NAMES):
        if nme == "end":
            continue
        col = r[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {nme:10s} min {np.nanmin(col):8.2f} med {np.nanmedian(col):8.2f} max {np.nanmax(col):8.2f}")
    iss, arr = r[:, 16:112], r[:, 112:208]
    if not np.all(np.isnan(iss)):
        lat = arr - iss
        print("  q: median W issue / arrival / latency (us)")
        for q in list(range(0, 16)) + list(range(16, 96, 8)):
            if np.all(np.isnan(lat[:, q])):
                continue
            print(f"    {q:3d} {np.nanmedian(iss[:, q]):8.2f} {np.nanmedian(arr[:, q]):8.2f} {np.nanmedian(lat[:, q]):7.2f}")


def op(M, N, K, epi):
    rows = 2 * N if epi == 2 else N
    Ws = [(torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(4)]
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 2 else torch.float32)
    ws = torch.empty(lib.srl_op_gemm_workspace(M, N, K, epi), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    dbg = torch.zeros(200 * 16, dtype=torch.int64, device="cuda")
    for i in range(5):
        if i == 4:
            lib.srl_debug_gemm_timestamps(dbg.data_ptr(), 0)
        lib.srl_op_gemm_bf16(X.data_ptr(), M, Ws[i % 4].data_ptr(), N, K, epi, out.data_ptr(), ws.data_ptr(), s)
        torch.cuda.synchronize()
    lib.srl_debug_gemm_timestamps(None, 0)
    report(f"op M={M} N={N} K={K} epi={epi}", dbg)


def engine(L):
    from paper_2603_23414_b200 import _lib as _L
    _L.set_tuning(graphs=0)
    from paper_2603_23414_b200.engine import RolloutEngine
    from workload.configs import LLAMA8B, SchedConfig, KV_BF16
    from workload.lengths import LengthModel, sample_lengths
    from workload.prompts import make_prompts
    from workload.weights import fill_engine_weights
    m = LLAMA8B.with_layers(L)
    cfg = SchedConfig(Q_g=256, U=64, pool_prompts=1024, cap=8192, kv_pages=3000, kv_dtype=KV_BF16)
    eng = RolloutEngine(m, cfg, max_traj=1024, max_prompt=256, prefill_chunk=4096)
    fill_engine_weights(eng, m, 0)
    eng.load_policy_weights(0)
    off, toks = make_prompts(1, 1024, m.V, 256)
    Ls = sample_lengths(LengthModel(cap=8192), 0, 1024)
    eng.submit_prompts(np.arange(1024, dtype=np.uint64), off, toks, Ls)
    for _ in range(3):
        eng.decode_step()
    for idx, name in enumerate(["qkv", "o", "gate_up", "down"]):
        dbg = torch.zeros(200 * 16, dtype=torch.int64, device="cuda")
        lib.srl_debug_gemm_timestamps(dbg.data_ptr(), idx)
        eng.decode_step()
        torch.cuda.synchronize()
        report(f"engine layer-0 {name}", dbg)
    lib.srl_debug_gemm_timestamps(None, 0)
    eng.set_profiling(True)
    for _ in range(5):
        eng.decode_step()
    print({k: round(v[0] / 5 / (L if k.startswith("gemm") else 1), 4) for k, v in eng.profile().items()})


def mlp(M, S2, d=4096, ff=14336):
    """one srl_op_mlp_bf16 launch (fused gate/up + down)"""
    def pack(W):
        dst = torch.empty(lib.srl_op_packed_weight_bytes(W.shape[0], W.shape[1]), dtype=torch.uint8, device="cuda")
        lib.srl_op_pack_weight(W.data_ptr(), W.shape[0], W.shape[1], dst.data_ptr(), s)
        return dst
    s = torch.cuda.current_stream().cuda_stream
    gu = [pack((torch.randn(2 * ff, d, device="cuda") * 0.02).to(torch.bfloat16)) for _ in range(3)]
    dn = [pack((torch.randn(d, ff, device="cuda") * 0.02).to(torch.bfloat16)) for _ in range(3)]
    X = torch.randn(M, d, device="cuda").to(torch.bfloat16)
    act = torch.empty(M, ff, dtype=torch.bfloat16, device="cuda")
    part = torch.empty(8, M, d, dtype=torch.float32, device="cuda")
    ws = torch.zeros(lib.srl_op_gemm_workspace(M, d, ff, 1), dtype=torch.uint8, device="cuda")
    dbg = torch.zeros(200 * 16, dtype=torch.int64, device="cuda")
    for i in range(5):
        if i == 4:
            lib.srl_debug_gemm_timestamps(dbg.data_ptr(), 0)
        lib.srl_op_mlp_bf16(X.data_ptr(), M, gu[i % 3].data_ptr(), dn[i % 3].data_ptr(), d, ff, S2, act.data_ptr(),
                            part.data_ptr(), ws.data_ptr(), s)
        torch.cuda.synchronize()
    lib.srl_debug_gemm_timestamps(None, 0)
    report(f"mlp M={M} S2={S2}", dbg)


if __name__ == "__main__":
    if sys.argv[1] == "mlp":
        mlp(int(sys.argv[2]), int(sys.argv[3]))
    elif sys.argv[1] == "op":
        op(*map(int, sys.argv[2:6]))
    else:
        engine(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
