#!/usr/bin/env python3
"""Mutation run over the CUDA path (dev aid): does the GPU parity suite notice a slip in a
rarely taken branch of the fused kernel -- the HLL fast path and its dry-side speeds, the
dry-CTA fast path, HGS identity tiles and band flags, the halo push, the sediment donor tie,
wall-corner ghosts, minmod at zero, the fp32 seed?

  python tools/mutate_kernel.py build      # variants/kmut_*.so (+ kmut_base.so), here
  python tools/mutate_kernel.py run        # on the GPU box: each variant in place of
                                           # libcsph.so against the GPU parity subset

Each mutant is one textual change of a source file in a scratch copy of csrc/; nothing in
the repo's sources is modified.  `run` restores the original library at the end."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CSRC = os.path.join(ROOT, "paper_2103_15196_b200", "csrc")
SO = os.path.join(ROOT, "paper_2103_15196_b200", "libcsph.so")
VAR = os.path.join(ROOT, "variants")

# (name, file, old, new, occurrence index)
MUTANTS = [
    ("HLL fast path: dissipation sign", "csph_fused.cu",
     "const T h0 = ((SR * mm - SL * mp) + SLSR * d0) * inv;",
     "const T h0 = ((SR * mm - SL * mp) - SLSR * d0) * inv;", 0),
    ("HLL general path: dissipation sign", "csph_fused.cu",
     "const T h0 = ((SR * mm - SL * mp) + SLSR * d0) * inv;",
     "const T h0 = ((SR * mm - SL * mp) - SLSR * d0) * inv;", 1),
    ("HLL fast path: supercritical upwind side", "csph_fused.cu",
     "F0 = up ? mm : (dn ? mp : h0);", "F0 = up ? mp : (dn ? mp : h0);", 0),
    ("HLL dry-right speed -2c", "csph_fused.cu", "fma(T(-2), cp, un_p)", "fma(T(-1), cp, un_p)", 0),
    ("HLL dry-left speed +2c", "csph_fused.cu", "fma(T(2), cm, un_m)", "fma(T(1), cm, un_m)", 0),
    ("halo push: 2 rows instead of 3", "csph_fused.cu", "min(y1, GY)", "min(y1, GY - 1)", 0),
    ("HGS identity tile: source sign", "csph_fused.cu",
     "const T bn = fma(-(lam * W3), z, b3) + (tau * W3) * Q.src;",
     "const T bn = fma(-(lam * W3), z, b3) - (tau * W3) * Q.src;", 0),
    ("HGS band flag BOT row", "csph_fused.cu", "(j == y1 - 1 ? HGS_BOT : 0u)",
     "(j == y1 - 2 ? HGS_BOT : 0u)", 0),
    ("dry CTA path: u~/v~ carry swapped", "csph_fused.cu",
     "ut2 = X2(1, 0); vt2 = X2(2, 0);", "ut2 = X2(2, 0); vt2 = X2(1, 0);", 0),
    ("dry CTA path: K8 y-flux sign", "csph_fused.cu",
     "const T dQx = dF3[1] + (Gn[1] - Gs[1]);", "const T dQx = dF3[1] - (Gn[1] - Gs[1]);", 0),
    ("dry CTA path: bed source sign", "csph_fused.cu",
     "const T bn = fma(-(lam * W3), dJ, b3) + (tau * W3) * Q.src;",
     "const T bn = fma(-(lam * W3), dJ, b3) - (tau * W3) * Q.src;", 0),
    ("sediment donor tie: 0.25 average", "csph_real.cuh",
     "T(0.5) * (JnL + JnR)", "T(0.25) * (JnL + JnR)", 0),
    ("wall x-ghost: Qx not negated (hot path)", "csph_real.cuh",
     "oH[g] = Hn; oQx[g] = -Qxn; oQy[g] = Qyn; ob[g] = bn;",
     "oH[g] = Hn; oQx[g] = Qxn; oQy[g] = Qyn; ob[g] = bn;", 0),
    ("wall x-ghost: Qx not negated (general path)", "csph_internal.cuh",
     "oQx[g] = nx_[a] ? -Qxn : Qxn;", "oQx[g] = Qxn;", 0),
    ("minmod: zero operand test dropped", "csph_real.cuh", " & (pick != 0.0);", ";", 0),
    ("K4: theta -> tau (control)", "csph_fused.cu", "fma(-theta, div, T(1))",
     "fma(-tau, div, T(1))", 0),
    ("fp32 icbrt seed", "csph_real.cuh", "0x54A2FA8C", "0x54A2FA9C", 0),
    # ---- second batch: the ctrl kernel, open edges, NEXT-3 fields, strips, math recipes
    ("ctrl Eq.7: t2 tie to t2", "csph_api.cu", "if (t2 < m) { m = t2; lim = 1; }",
     "if (t2 <= m) { m = t2; lim = 1; }", 0),
    ("ctrl Eq.7: t3 tie to t3", "csph_api.cu", "if (t3 < m) { m = t3; lim = 2; }",
     "if (t3 <= m) { m = t3; lim = 2; }", 0),
    ("ctrl Eq.7: h^2 -> h/h", "csph_api.cu", "double t3 = (h * h) / (2.0 * M[2]);",
     "double t3 = (h / h) / (2.0 * M[2]);", 0),
    ("peer combine: min instead of max", "csph_api.cu",
     "m[k] = e[k] > m[k] ? e[k] : m[k];", "m[k] = e[k] > m[k] ? m[k] : e[k];", 0),
    ("open lo edge: ghost negated", "csph_internal.cuh",
     "for (int g = 1; g <= 3; ++g) { t[k] = -g; neg[k++] = false; }",
     "for (int g = 1; g <= 3; ++g) { t[k] = -g; neg[k++] = true; }", 0),
    ("open hi edge: 2 ghost layers", "csph_internal.cuh",
     "for (int g = 0; g < 3; ++g) { t[k] = n + g; neg[k++] = false; }",
     "for (int g = 0; g < 2; ++g) { t[k] = n + g; neg[k++] = false; }", 0),
    ("NEXT-3 source sign", "csph_internal.cuh", "Hn = (Hn + tau * S.src[c]) * a;",
     "Hn = (Hn - tau * S.src[c]) * a;", 0),
    ("NEXT-3 friction field row", "csph_fused.cu", "S.cg[fidx(col, L)]", "S.cg[fidx(col, L - 1)]", 0),
    ("HGS ghost flag slot", "csph_fused.cu", "S.ngflag[0][g + hg.ntx] = (unsigned char)m;",
     "S.ngflag[0][g] = (unsigned char)m;", 0),
    ("rcp all-ones fix dropped", "csph_internal.cuh", "| (ones == 0xFFFFFFFFu))", "| 0u)", 0),
    ("icbrt 4 Newton steps", "csph_internal.cuh", "for (int k = 0; k < 5; ++k) {",
     "for (int k = 0; k < 4; ++k) {", 0),
    ("sediment slope: * inv_h -> / inv_h", "csph_real.cuh", "(bR - bL) * P.inv_h",
     "(bR - bL) / P.inv_h", 0),
    ("K8 bed: lam -> tau", "csph_fused.cu",
     "const T bn = fma(-(lam * W3), dJ, b3) + (tau * W3) * Q.src;",
     "const T bn = fma(-(tau * W3), dJ, b3) + (tau * W3) * Q.src;", 1),
    # ---- third batch: host / service logic of csph_api.cu
    ("ctrl: simulated time not accumulated", "csph_api.cu", "C->t += C->tau;", "C->t = C->tau;", 0),
    ("dt log ring: off by one", "csph_api.cu", "long long first = (done - m) % LOGCAP;",
     "long long first = (done - m + 1) % LOGCAP;", 0),
    ("peer-copy halo: send_hi row", "csph_api.cu", "m.send_hi = off(v.pitch, -GX, v.ny - GY);",
     "m.send_hi = off(v.pitch, -GX, v.ny - GY + 1);", 0),
    ("peer-copy flags: hi into lo slot", "csph_api.cu", "m.frecv_hi = m.frecv_lo + s.ntx;",
     "m.frecv_hi = m.frecv_lo;", 0),
    ("get_state_rows: row offset", "csph_api.cu", "sk + off(v.pitch, 0, lo - s.gj0), (size_t)v.pitch * 8,",
     "sk + off(v.pitch, 0, lo - s.gj0 + 1), (size_t)v.pitch * 8,", 0),
    ("set_state: upper halo rows", "csph_api.cu", "int hi = s.gj0 + v.ny + (v.wall_hi ? 0 : GY);",
     "int hi = s.gj0 + v.ny + (v.wall_hi ? 0 : GY - 1);", 0),
    ("save: owned-row offset", "csph_api.cu", "dst[k] + (size_t)s.gj0 * H->nx,", "dst[k],", 0),
    ("validate: psi = 1 accepted", "csph_api.cu", "if (!(p >= 0.0 && p < 1.0)) f |= 4;",
     "if (!(p >= 0.0 && p <= 1.0)) f |= 4;", 0),
    ("validate: negative depth accepted", "csph_api.cu", "if (H < 0.0) f |= 2;",
     "if (H < -1.0) f |= 2;", 0),
    ("W = 1/(1-psi) -> 1/(1+psi)", "csph_api.cu", "W[k] = 1.0 / (1.0 - psi[k]);",
     "W[k] = 1.0 / (1.0 + psi[k]);", 0),
]

GPU_TESTS = ["tests/test_gpu_parity.py", "tests/test_gpu_strips.py", "tests/test_gpu_fp32.py",
             "tests/test_next3_fields.py", "tests/test_next4_closures.py", "tests/test_gpu_save.py"]


def build_one(i, name, fname, old, new, occ):
    from paper_2103_15196_b200 import build
    tmp = tempfile.mkdtemp(prefix="kmut_")
    try:
        src = os.path.join(tmp, "pkg", "csrc")  # csph_api.cu includes ../../include/csph.h
        shutil.copytree(CSRC, src)
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
        p = os.path.join(src, fname)
        text = open(p).read()
        k = -1
        for _ in range(occ + 1):
            k = text.find(old, k + 1)
            if k < 0:
                return name, "NOMATCH"
        open(p, "w").write(text[:k] + new + text[k + len(old):])
        out = os.path.join(VAR, "kmut_%02d.so" % i)
        cmd = build.nvcc_cmd(out)
        cmd = [c.replace(CSRC, src) for c in cmd]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return name, "built" if r.returncode == 0 else "BUILD FAILED " + r.stderr[-300:]
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def cmd_build():
    os.makedirs(VAR, exist_ok=True)
    from paper_2103_15196_b200 import build
    build.build()
    shutil.copy2(SO, os.path.join(VAR, "kmut_base.so"))
    only = {int(x) for x in sys.argv[2].split(",")} if len(sys.argv) > 2 else None
    with cf.ThreadPoolExecutor(4) as ex:
        futs = [ex.submit(build_one, i, *m) for i, m in enumerate(MUTANTS)
                if only is None or i in only]
        for f in futs:
            print("%-45s %s" % f.result(), flush=True)


def cmd_run():
    base = os.path.join(VAR, "kmut_base.so")
    only = {int(x) for x in sys.argv[2].split(",")} if len(sys.argv) > 2 else None
    res = []
    try:
        for i, (name, *_r) in enumerate(MUTANTS):
            if only is not None and i not in only:
                continue
            so = os.path.join(VAR, "kmut_%02d.so" % i)
            if not os.path.exists(so):
                res.append((name, "not built"))
                continue
            shutil.copy(so, SO)
            os.utime(SO, None)  # newer than the sources: build() keeps it
            t0 = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                                "-p", "no:cacheprovider"] + GPU_TESTS,
                               cwd=ROOT, capture_output=True, text=True, timeout=1500)
            dt = time.time() - t0
            if r.returncode == 0:
                st = "SURVIVED"
            else:
                failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
                st = "caught by " + (failed[0].split(" ")[1][:70] if failed else "rc %d" % r.returncode)
            res.append((name, st))
            print("%-45s %6.1fs  %s" % (name, dt, st), flush=True)
    finally:
        shutil.copy(base, SO)
        os.utime(SO, None)
    sv = [n for n, s in res if not s.startswith("caught")]
    print("\n%d kernel mutants, %d caught; not caught: %s" % (len(res), len(res) - len(sv), sv))


if __name__ == "__main__":
    {"build": cmd_build, "run": cmd_run}[sys.argv[1]]()
