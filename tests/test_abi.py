"""The C-ABI library loads and exports every function include/*.h declares (CPU only,
no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")
LIB = os.path.join(ROOT, "paper_2603_23414_b200", "libsrl.so")


def _declared():
    names = []
    for h in sorted(os.listdir(INC)):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(INC, h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(srl_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2603_23414_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_headers_declare_the_boundary():
    names = _declared()
    for n in ("srl_create", "srl_submit_prompts", "srl_decode_step", "srl_harvest_finished",
              "srl_load_policy_weights", "srl_op_gemm_bf16", "srl_op_attention", "srl_op_sample"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_and_uses_tcgen05_tma():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", LIB], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass             # tcgen05.ld
    assert "HMMA" in sass             # attention mma.sync


def test_arena_sizes_and_validation_on_cpu(lib):
    """Pure host calls (no GPU needed): sizing, weight layout, argument validation."""
    from paper_2603_23414_b200 import _lib
    from workload.configs import LLAMA8B, TINY
    L = _lib.load()
    m = _lib.ModelCfg(TINY.L, TINY.d, TINY.Hq, TINY.Hkv, TINY.dh, TINY.ff, TINY.V, 1e4, 1e-5, 0)
    s = _lib.SchedCfg(16, 4, -1, 16, 1, 64, 64, 64, 0, 0, 0, 0, -1, 1, 1.0, 3, 64, 16, 256, 0, 1.0)
    w, k, sc = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    assert L.srl_arena_sizes(ctypes.byref(m), ctypes.byref(s), 1, ctypes.byref(w), ctypes.byref(k), ctypes.byref(sc)) == 0
    assert k.value == 2 * TINY.L * 64 * TINY.Hkv * 64 * TINY.dh * 4
    n = ctypes.c_int64()
    off_q = L.srl_weight_offset(ctypes.byref(m), b"L0.wq", ctypes.byref(n))
    off_k = L.srl_weight_offset(ctypes.byref(m), b"L0.wk", None)
    assert n.value == TINY.Hq * TINY.dh * TINY.d and off_k == off_q + 2 * n.value   # q,k,v contiguous
    assert L.srl_weight_offset(ctypes.byref(m), b"nope", None) == -1
    s.U = 999                                   # U > pool
    assert L.srl_arena_sizes(ctypes.byref(m), ctypes.byref(s), 1, None, None, None) == -1
    assert b"pool" in L.srl_last_error()
    m8 = _lib.ModelCfg(LLAMA8B.L, LLAMA8B.d, LLAMA8B.Hq, LLAMA8B.Hkv, LLAMA8B.dh, LLAMA8B.ff, LLAMA8B.V, 5e5, 1e-5, 0)
    s8 = _lib.SchedCfg(256, 64, -1, 1024, 1, 8192, 64, 12000, 0, 0, 0, 0, -1, 0, 1.0, 3, 2048, 256, 4096, 0, 1.0)
    assert L.srl_arena_sizes(ctypes.byref(m8), ctypes.byref(s8), 1, ctypes.byref(w), ctypes.byref(k), ctypes.byref(sc)) == 0
    # bf16 LLaMA-3.1-8B weights (staging image) + packed copies of the projection matrices
    mats = LLAMA8B.L * ((LLAMA8B.Hq + 2 * LLAMA8B.Hkv) * LLAMA8B.dh * 4096 + 4096 * 4096 + 2 * 14336 * 4096
                        + 4096 * 14336) + LLAMA8B.V * 4096
    assert abs(w.value - (16.06e9 + 2 * mats)) / 16.06e9 < 0.01


def test_compact_weights_sizing_on_cpu(lib):
    """weights_compact: no staging copy of the projections (about half the bytes);
    packed-only tensors are not addressable; q/k/v must tile by 128 rows."""
    from paper_2603_23414_b200 import _lib
    from workload.configs import QWEN32B, TINY
    L = _lib.load()
    s = _lib.SchedCfg(64, 64, -1, 256, 1, 16384, 64, 5000, 0, 0, 0, 0, -1, 0, 1.0, 3, 1024, 256, 4096, 0, 1.0)
    sizes = []
    for compact in (0, 1):
        m = _lib.ModelCfg(QWEN32B.L, QWEN32B.d, QWEN32B.Hq, QWEN32B.Hkv, QWEN32B.dh, QWEN32B.ff, QWEN32B.V, 1e6,
                          1e-5, 1, compact)
        w = ctypes.c_uint64()
        assert L.srl_arena_sizes(ctypes.byref(m), ctypes.byref(s), 1, ctypes.byref(w), None, None) == 0
        sizes.append(w.value)
        off = L.srl_weight_offset(ctypes.byref(m), b"L3.wg", None)
        assert (off >= 0) == (compact == 0)
        assert L.srl_weight_offset(ctypes.byref(m), b"L3.bq", None) >= 0
    assert abs(sizes[1] - 65.5e9) / 65.5e9 < 0.02 and sizes[0] > 1.9 * sizes[1]
    mt = _lib.ModelCfg(TINY.L, TINY.d, TINY.Hq, TINY.Hkv, TINY.dh, TINY.ff, TINY.V, 1e4, 1e-5, 0, 1)
    s.U = 4
    assert L.srl_arena_sizes(ctypes.byref(mt), ctypes.byref(s), 1, None, None, None) < 0


def test_emission_sort_capacity_is_validated(lib):
    """the emission sort keeps the ready list in shared memory
    (16384 keys).  SORTED can hold U-1+Q_tot ready trajectories and POSTHOC the
    whole pool, so configurations beyond that are rejected up front."""
    from paper_2603_23414_b200 import _lib
    from workload.configs import TINY
    L = _lib.load()
    m = _lib.ModelCfg(TINY.L, TINY.d, TINY.Hq, TINY.Hkv, TINY.dh, TINY.ff, TINY.V, 1e4, 1e-5, 0)

    def ok(Q_g, U, pool, mode, world=1):
        s = _lib.SchedCfg(Q_g, U, -1, pool, 1, 64, 64, 64, mode, 0, 0, 0, -1, 1, 1.0, 3, 64, 16, 256, 0, 1.0)
        return L.srl_arena_sizes(ctypes.byref(m), ctypes.byref(s), world, None, None, None) == 0
    assert ok(4096, 2048, 8192, 0)                      # U-1+Q_tot = 6143 <= 16384
    assert ok(512, 64, 8192, 2, world=8)                # bench --mode posthoc --gpus 8: pool 8192
    assert not ok(512, 64, 16384, 2, world=8)           # POSTHOC pool + U - 1 > 16384
    assert b"POSTHOC" in L.srl_last_error()
    assert ok(512, 64, 16384, 0, world=8)               # SORTED with the same pool is fine
    assert ok(512, 64, 16384, 1, world=8)               # SYNC never sorts


def test_tuning_roundtrip_and_validation(lib):
    """srl_tuning replaces every environment override: defaults are the
    production choices, out-of-range values are rejected without changing anything."""
    from paper_2603_23414_b200 import _lib
    d = _lib.get_tuning()
    assert d["gemm_split"] == 1 and d["gemm_pair"] == -1 and d["partial_norm"] == 1 and d["pdl"] == 1
    assert d["graphs"] == 1 and d["mixed_prefill"] == 1 and d["fused_sample"] == 0 and d["qkv_finish"] == 0
    old = _lib.set_tuning(fused_sample=1, attn_l2_prefetch=4)
    try:
        t = _lib.get_tuning()
        assert t["fused_sample"] == 1 and t["attn_l2_prefetch"] == 4 and t["gemm_split"] == 1
        with pytest.raises(_lib.SRLError):
            _lib.set_tuning(gemm_split=7)
        assert _lib.get_tuning() == t
    finally:
        _lib.set_tuning(**old)
    assert _lib.get_tuning() == d
    _lib.set_tuning(defaults=True)
    assert _lib.get_tuning() == d


def test_gate_up_staging_interleave_on_cpu(lib):
    """srl.h srl_weight_layout: L<i>.wg / L<i>.wu rows interleaved in 16-row blocks
    (row_block 16, block_stride 32, wu 16 rows after wg) -- the layout the SiLU-mul
    epilogue pairs with one xor-16 shuffle; every other tensor dense row-major."""
    from paper_2603_23414_b200 import _lib
    from workload.configs import LLAMA8B
    L = _lib.load()
    m = _lib.ModelCfg(LLAMA8B.L, LLAMA8B.d, LLAMA8B.Hq, LLAMA8B.Hkv, LLAMA8B.dh, LLAMA8B.ff, LLAMA8B.V, 5e5, 1e-5, 0)
    v = [ctypes.c_int64() for _ in range(5)]

    def lay(name):
        assert L.srl_weight_layout(ctypes.byref(m), name, *[ctypes.byref(x) for x in v]) == 0
        return [x.value for x in v]
    og, rg, cg, rbg, bsg = lay(b"L5.wg")
    ou, ru, cu, rbu, bsu = lay(b"L5.wu")
    assert (rg, cg, rbg, bsg) == (LLAMA8B.ff, LLAMA8B.d, 16, 32) and (ru, cu, rbu, bsu) == (rg, cg, 16, 32)
    assert ou - og == 16 * LLAMA8B.d * 2
    od, rd, cd, rbd, bsd = lay(b"L5.wd")
    assert (rd, cd) == (LLAMA8B.d, LLAMA8B.ff) and rbd == bsd == rd
    assert od >= og + 2 * LLAMA8B.ff * LLAMA8B.d * 2   # wd after the whole interleaved region


def test_tuning_defaults_of_the_r02_kernels(lib):
    """The production choices measured in r02: 512-row gate/up pair units
    on, the QKV finish inside attention on, the 4-stage attention ring, the fused MLP off;
    attn_stages accepts 3 / 4 / 6 only."""
    from paper_2603_23414_b200 import _lib
    d = _lib.get_tuning()
    assert d["pair_h2"] == 1 and d["qkv_attn"] == 1 and d["attn_stages"] == 4 and d["fuse_mlp"] == 0
    for bad in (dict(attn_stages=5), dict(pair_h2=2)):
        with pytest.raises(_lib.SRLError):
            _lib.set_tuning(**bad)
        assert _lib.get_tuning() == d
    old = _lib.set_tuning(attn_stages=3)
    _lib.set_tuning(**old)
    assert _lib.get_tuning() == d


def test_library_reads_no_environment():
    """No getenv in the product library (the knobs moved to srl_tuning)."""
    import glob
    for f in glob.glob(os.path.join(ROOT, "paper_2603_23414_b200", "csrc", "*")):
        assert "getenv" not in open(f).read(), f
