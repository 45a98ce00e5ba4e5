"""CPU tests of the C-ABI library: it loads, exports every symbol include/paradyse.h
declares, and its host-only logic (Algorithm 1, memory plan, cost bundle) agrees
bit-exactly with the oracle.  No GPU compute is called."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import memory as OM
from oracle import selector as OA

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def B():
    from paper_2511_13198_b200 import binding
    binding.lib()
    return binding


def test_exports_every_declared_symbol(B):
    hdr = open(os.path.join(ROOT, "include", "paradyse.h")).read()
    names = set(re.findall(r"^\s*(?:pds_status|const char\*)\s+(pds_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 30
    L = ctypes.CDLL(B.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n
    assert B.lib().pds_version().decode().startswith("paradyse-b200")


def test_plan_ex_bit_exact_vs_oracle(B):
    rng = np.random.default_rng(0)
    n_inf = n_early = 0
    for trial in range(4000):
        k = int(rng.integers(1, 6))
        L = int(rng.choice([1, 2, 3, 5, 8, 32]))
        t = [float(v) for v in rng.random(k)]
        m = [float(v) for v in rng.random(k)]
        if trial % 7 == 0:                       # exact ties
            t[-1] = t[0]
        en = [bool(e) for e in (rng.random(k) < 0.85)]
        if not any(en):
            en[0] = True
        cap = float(rng.random() * L * 0.9 + 1e-3)
        enabled = [i for i in range(k) if en[i]]
        # per-strategy workspace (reading R-22) in half of the trials
        w = [float(v) for v in rng.random(k) * 0.5] if trial % 2 else None
        wd = dict(enumerate(w)) if w is not None else None
        plan, flags, ctr = B.plan_ex(L, t, m, en, cap, counters=True, w=w)
        ctr_o = OA.Counters()
        ref, inf = OA.alg1(L, dict(enumerate(t)), dict(enumerate(m)), enabled, cap, ctr=ctr_o, w=wd)
        assert plan == ref, (trial, k, L, t, m, en, cap)
        assert bool(flags & B.PLAN_INFEASIBLE) == inf
        assert ctr[0] == ctr_o.layer_checks and ctr[1] == ctr_o.plans
        n_inf += inf
        n_early += bool(flags & B.PLAN_EARLY)
        # smoothing against a random previous plan
        prev = [int(rng.choice(enabled)) for _ in range(L)]
        g = float(rng.choice([0.0, 0.05, 0.3]))
        p2, f2 = B.plan_ex(L, t, m, en, cap, gamma=g, prev=prev, w=w)
        r2, kept = OA.smooth(ref, prev, dict(enumerate(t)), dict(enumerate(m)), cap, g, enabled, w=wd)
        assert p2 == r2 and bool(f2 & B.PLAN_SMOOTHED) == kept
    assert n_inf > 50 and n_early > 50


def test_plan_ex_worked_examples(B):
    assert B.plan_ex(3, [1.0, 2.0], [10.0, 4.0], [1, 1], 25.0)[0] == [0, 0, 1]
    assert B.plan_ex(2, [0.0, 2.9, 3.0], [10.0, 6.0, 0.0], [1, 1, 1], 11.0)[0] == [0, 2]   # R-17
    plan, fl = B.plan_ex(3, [1.0, 2.0], [10.0, 5.0], [1, 1], 1.0)
    assert plan == [1, 1, 1] and fl & B.PLAN_INFEASIBLE
    with pytest.raises(B.PdsError) as e:
        B.plan_ex(0, [1.0], [1.0], [1], 1.0)
    assert e.value.code == -1


@pytest.mark.parametrize("cfg", [(256, 4, 1024, 512, 2), (4096, 32, 16384, 32768, 8), (4096, 32, 16384, 4096, 1),
                                 (4096, 32, 16384, 638976, 8), (1024, 8, 4096, 1024, 4)])
def test_mem_bytes_vs_oracle(B, cfg):
    h, n, F, s, P = cfg
    m = B.Model(h=h, n_heads=n, ffn=F)
    for pi in (0, 1, 2, 3, 4):
        if not OM.valid(pi, h, n, F, s, P):
            with pytest.raises(B.PdsError) as e:
                B.mem_bytes(m, P, pi, s)
            assert e.value.code == -2                # R-15: divisibility is a hard error
            continue
        saved, tr, pers = B.mem_bytes(m, P, pi, s)
        assert saved == OM.saved(pi, h, n, F, s, P), (pi, cfg)
        assert pers == OM.persistent(h, F, P)
        # the workspace is the implementation's own (pinned by device measurement in
        # tests/test_gpu_memory.py); it can never be below the dataflow floor
        assert tr >= OM.transient_floor(pi, h, n, F, s, P), (pi, cfg)


@pytest.mark.parametrize("cfg", [(256, 4, 1024, 512, 2), (4096, 32, 16384, 638976, 8), (4096, 32, 16384, 65536, 1)])
def test_mem_bytes_metp_full_vs_oracle(B, cfg):
    # metp_recompute = 1 ('full'): saved 3u + 2l + lam, Q/K/V in the workspace instead
    h, n, F, s, P = cfg
    m = B.Model(h=h, n_heads=n, ffn=F, metp_recompute=1)
    saved, tr, pers = B.mem_bytes(m, P, 2, s)
    assert saved == OM.saved(2, h, n, F, s, P, metp_recompute="full")
    assert tr >= OM.transient_floor(4, h, n, F, s, P)
    saved0, tr0, _ = B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F), P, 2, s)
    assert saved0 - saved == 3 * (s // P) * h * 2
    # strategy METP-full (4) == METP with metp_recompute = full, whatever the knob says
    assert B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F), P, 4, s) == (saved, tr, pers)
    assert B.mem_bytes(m, P, 4, s) == (saved, tr, pers)
    assert saved == OM.saved(4, h, n, F, s, P)
    assert tr - tr0 == (s // P) * 3 * h * 2          # Q/K/V of the own heads move to the workspace
    with pytest.raises(B.PdsError) as e:
        B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F, metp_recompute=2), P, 2, s)
    assert e.value.code == -1


def test_mem_bytes_errors(B):
    m = B.Model(h=256, n_heads=4, ffn=1024)
    with pytest.raises(B.PdsError) as e:
        B.mem_bytes(m, 2, 0, 500)                    # P does not divide s (hard error, R-15)
    assert e.value.code == -2
    with pytest.raises(B.PdsError) as e:
        B.mem_bytes(m, 2, 9, 512)
    assert e.value.code == -3
    with pytest.raises(B.PdsError) as e:
        B.mem_bytes(B.Model(h=256, n_heads=4, ffn=1024, batch=0), 2, 0, 512)
    assert e.value.code == -1


@pytest.mark.parametrize("b", [2, 3])
def test_mem_bytes_batch_vs_oracle(B, b):
    # b sequences in the [s/P, b, h] layout: every token buffer holds positions x b rows
    for (h, n, F, s, P) in [(256, 4, 1024, 512, 2), (4096, 32, 16384, 8192, 4)]:
        for pi in (0, 1, 2, 3, 4):
            saved, tr, pers = B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F, batch=b), P, pi, s)
            assert saved == OM.saved(pi, h, n, F, s, P, b=b), (pi, b)
            assert tr >= OM.transient_floor(pi, h, n, F, s, P, b=b), (pi, b)
            # token buffers scale with b: every term of the workspace but the weights does
            _, tr1, _ = B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F, batch=1), P, pi, s)
            assert tr > tr1


def test_product_library_is_tcgen05_only(B):
    """Every tensor-core instruction in libparadyse.so is tcgen05 (UTCHMMA / UTCQMMA):
    no warp-level mma.sync (HMMA) kernel ships in the product (the round-1 FA2
    baseline lives in tools/fa2_sync_baseline.cu)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", B.LIB_PATH], capture_output=True, text=True, check=True).stdout
    ops = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+([A-Z0-9_]+)", sass, re.M)
    assert "UTCHMMA" in ops and "UTMALDG" in ops
    assert not [o for o in ops if o.startswith("HMMA")], "legacy mma.sync in the product library"


@pytest.mark.parametrize("P,n_kv,act", [(1, 2, 1), (2, 2, 1), (4, 4, 1), (2, 8, 1), (2, 2, 0)])
def test_mem_bytes_llama_variant_vs_oracle(B, P, n_kv, act):
    """Llama variant (R-GQA / R-SWIGLU): the library's saved bytes and persistent
    weights equal the oracle's formulas (which the oracle's ledger recount pins) for
    every strategy; P must divide n_kv."""
    h, n, F, s = 4096, 32, 11264, 8192           # F/P a multiple of 64 at P <= 4 (11008 is not)
    a = "swiglu" if act else "gelu"
    m = B.Model(h=h, n_heads=n, ffn=F, n_kv_heads=n_kv, ffn_act=act, batch=2)
    for pi in (0, 1, 2, 3, 4, 5):
        saved, tr, pers = B.mem_bytes(m, P, pi, s)
        assert saved == OM.saved(pi, h, n, F, s, P, b=2, n_kv=n_kv, act=a), pi
        assert pers == OM.persistent(h, F, P, n, n_kv, a)
    with pytest.raises(B.PdsError) as e:
        B.mem_bytes(B.Model(h=h, n_heads=n, ffn=F, n_kv_heads=2, ffn_act=act), 4, 0, s)
    assert e.value.code == -2
    # MHA + GELU (n_kv = 0 or n) is the round-1 plan byte for byte
    base = B.mem_bytes(B.Model(h=h, n_heads=n, ffn=4 * h), P, 0, s)
    assert base == B.mem_bytes(B.Model(h=h, n_heads=n, ffn=4 * h, n_kv_heads=n), P, 0, s)
