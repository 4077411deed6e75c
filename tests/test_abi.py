"""CPU-side checks of the C-ABI library (no compute calls without a GPU)."""
import ctypes
import re
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def csph():
    from paper_2103_15196_b200 import build, csph
    build.build()
    return csph


def test_library_exports_every_declared_symbol(csph):
    """Every function include/csph.h declares is exported by libcsph.so."""
    hdr = open(os.path.join(ROOT, "include", "csph.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(csph_[a-z_]+)\s*\(", hdr))
    assert declared == set(csph.EXPORTS), declared ^ set(csph.EXPORTS)
    L = ctypes.CDLL(csph.SO_PATH)
    for name in declared:
        assert hasattr(L, name), name


def test_default_params(csph):
    p = csph.csph_default_params()
    assert p.g == 9.81 and p.K == 0.25 and p.eps_dry == 1e-6 and p.m_grass == 2
    assert p.precision == 64 and p.neg_tol == 1e-12 and p.dt_max == float("inf")


def test_strip_partition_host_logic(csph):
    """Row strips (P:210 Ny_dev): contiguous, covering, sizes differ by <= 1."""
    for ny, n in [(16384, 8), (1000, 7), (9, 3), (100, 1)]:
        rows = [csph.csph_strip_rows(ny, n, r) for r in range(n)]
        assert rows[0][0] == 0 and rows[-1][1] == ny
        for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
            assert a1 == b0
        sizes = [b - a for a, b in rows]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(csph.CsphError):
        csph.csph_strip_rows(8, 4, 0)  # 2-row strips are thinner than the 3-row halo


def test_errors_are_codes_not_crashes(csph):
    assert csph.csph_strerror(csph.CSPH_EDRY).startswith("no wet cell")
    assert csph.lib().csph_step(None, 1) == csph.CSPH_EINVAL
    p = csph.csph_default_params(K=1.5)
    assert not csph.lib().csph_create(10, 10, 1.0, ctypes.byref(p))
    assert "K" in csph.csph_last_error()


def test_no_cpu_fallback_without_gpu(csph):
    """With no CUDA device the product path fails loudly (ECUDA), never computes on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(csph.CsphError) as e:
        csph.csph_create(16, 16, 1.0)
    assert e.value.code == csph.CSPH_ECUDA


def _minmax_dp(w, n, m=3):
    """Brute force: the smallest achievable largest-strip weight over all partitions of w
    into n contiguous strips of >= m rows."""
    import functools
    import math
    ny = len(w)
    pre = [0.0]
    for x in w:
        pre.append(pre[-1] + x)

    @functools.lru_cache(None)
    def f(j, k):  # rows [j, ny) into k strips
        if k == 1:
            return pre[ny] - pre[j] if ny - j >= m else math.inf
        best = math.inf
        for e in range(j + m, ny - m * (k - 1) + 1):
            best = min(best, max(pre[e] - pre[j], f(e, k - 1)))
        return best
    return f(0, n)


def test_balance_rows_partition(csph):
    """csph_balance_rows: valid strips, the optimal largest strip cost
    (brute force on small cases), the even split for uniform or zero costs."""
    import numpy as np
    rng = np.random.default_rng(5)
    for trial in range(40):
        ny = int(rng.integers(9, 60))
        n = int(rng.integers(1, min(4, ny // 3) + 1))
        w = rng.random(ny) ** 3 * (rng.random(ny) < 0.6)
        b = csph.csph_balance_rows(ny, n, w)
        assert b[0] == 0 and b[-1] == ny and all(b[r + 1] - b[r] >= 3 for r in range(n))
        worst = max(w[b[r]:b[r + 1]].sum() for r in range(n))
        opt = _minmax_dp(tuple(w), n)
        assert worst <= opt * (1 + 1e-9) + 1e-15, (ny, n, worst, opt)
    for n in (1, 2, 3, 8):
        even = [csph.csph_strip_rows(1000, n, r) for r in range(n)]
        for w in (np.ones(1000), np.zeros(1000)):
            b = csph.csph_balance_rows(1000, n, w)
            assert all(abs((b[r + 1] - b[r]) - (even[r][1] - even[r][0])) <= 1 for r in range(n))
    # a heavy band: the strip holding it gets few rows
    w = np.full(4096, 0.05)
    w[1000:1400] = 100.0
    b = csph.csph_balance_rows(4096, 4, w)
    sizes = [b[r + 1] - b[r] for r in range(4)]
    assert min(sizes) < 300 and max(sizes) > 1500
    with pytest.raises(csph.CsphError):
        csph.csph_balance_rows(8, 3, np.ones(8))
    with pytest.raises(csph.CsphError):
        csph.csph_balance_rows(10, 2, -np.ones(10))
