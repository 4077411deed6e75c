#!/usr/bin/env python3
"""Mutation run over the CPU oracle (test infrastructure): does every plausible slip in
oracle/csph_oracle.c fail at least one `-m "not gpu"` pin?

Each mutation is one textual change (a wrong time level, sign, index, operand or
factor).  For each, the repo's oracle/, synth/ and tests/ are copied to a scratch
directory, the mutation is applied there (it must match exactly once), the oracle is
rebuilt and the oracle pin tests run with -x.  A mutation is "caught" when pytest
fails.  Nothing in the repo is modified.

    python tools/mutate_oracle.py            # all mutations, summary table
    python tools/mutate_oracle.py -k K5      # only those whose name contains K5
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/csph_oracle.c"
PIN_TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_bruteforce.py",
             "tests/test_next3_fields.py", "tests/test_next4_closures.py",
             "tests/test_oracle_sweep_pins.py"]

# (name, original text, mutated text)
MUTATIONS = [
    # ---- the five time-level slips that survived round 1's pins
    ("K5 centre eta uses H_n", "real ec = o->Hh[c] + b[c];", "real ec = H[c] + b[c];"),
    ("K7 reconstructs H_half", "const real* q[4] = {o->eta, H, un, utn};",
     "const real* q[4] = {o->eta, o->Hh, un, utn};"),
    ("gate reads H_half", "r_shamov_gate(o->kappa, s2, H[c], o->C_Sh) && r_bed_mobile(H[c], o->hbm)",
     "r_shamov_gate(o->kappa, s2, o->Hh[c], o->C_Sh) && r_bed_mobile(H[c], o->hbm)"),
    ("film cut-off reads H_half", "r_shamov_gate(o->kappa, s2, H[c], o->C_Sh) && r_bed_mobile(H[c], o->hbm)",
     "r_shamov_gate(o->kappa, s2, H[c], o->C_Sh) && r_bed_mobile(o->Hh[c], o->hbm)"),
    ("dry H_half = 0", "if (!o->w[c]) { o->Hh[c] = H[c];", "if (!o->w[c]) { o->Hh[c] = RL(0);"),
    # ---- K1 / K2 / friction
    ("K1 wet test >=", "o->w[c] = H[c] > eps;", "o->w[c] = H[c] >= eps;"),
    ("K1 v from Qx", "o->v[c] = Qy[c] * o->r[c];", "o->v[c] = Qx[c] * o->r[c];"),
    ("K2 force sign", "o->phix[c] = -(PE + PW);", "o->phix[c] = (PE + PW);"),
    ("K2 west face swapped", "real PW = face_force(o->cPh, o->eta[wv], b[wv], o->eta[c], b[c]);",
     "real PW = face_force(o->cPh, o->eta[c], b[c], o->eta[wv], b[wv]);"),
    ("face force b* = min", "real bs = sel_max(bL, bR);", "real bs = sel_min(bL, bR);"),
    ("face force mean factor", "return (cPh * (HsL + HsR)) * (HsR - HsL);",
     "return (cPh * (HsL + HsR + HsR)) * (HsR - HsL);"),
    ("friction H^(-1/3) dropped", "o->gam[c] = (o->cgam * sp) * (o->r[c] * r_icbrt(H[c]));",
     "o->gam[c] = (o->cgam * sp) * o->r[c];"),
    ("icbrt 4 Newton steps", "for (int k = 0; k < 5; ++k) {", "for (int k = 0; k < 2; ++k) {"),
    # ---- K4 / K6
    ("K4 theta = tau", "o->Hh[c] = H[c] * FMA(-theta, div, RL(1));", "o->Hh[c] = H[c] * FMA(-tau, div, RL(1));"),
    ("K4 div sign v", "(o->v[c + sy] - o->v[c - sy])", "(o->v[c - sy] - o->v[c + sy])"),
    ("K4 u~ uses Phi_half", "o->ut[c] = (FMA(theta, o->phix[c], Qx[c]) * f) * o->r[c];",
     "o->ut[c] = (FMA(theta, o->phix2[c], Qx[c]) * f) * o->r[c];"),
    ("K4 friction factor tau", "real f = RL(1) / FMA(theta, o->gam[c], RL(1));",
     "real f = RL(1) / FMA(tau, o->gam[c], RL(1));"),
    ("K6 uses Phi^n", "o->QLx[c] = FMA(tau, o->phix2[c], Qx[c]) * f;", "o->QLx[c] = FMA(tau, o->phix[c], Qx[c]) * f;"),
    ("K6 theta", "o->QLy[c] = FMA(tau, o->phiy2[c], Qy[c]) * f;", "o->QLy[c] = FMA(theta, o->phiy2[c], Qy[c]) * f;"),
    # ---- K7
    ("minmod picks max", "if (a > RL(0) && b > RL(0)) return sel_min(a, b);", "if (a > RL(0) && b > RL(0)) return sel_max(a, b);"),
    ("face state - sign", "qm[k] = FMA(RL(0.5), sL[k], q[k][L]);", "qm[k] = FMA(RL(-0.5), sL[k], q[k][L]);"),
    ("slope R wrong cells", "sR[k] = r_minmod(q[k][R] - q[k][L], q[k][RR] - q[k][R]);",
     "sR[k] = r_minmod(q[k][L] - q[k][LL], q[k][RR] - q[k][R]);"),
    ("HLL S_R dry factor 2", "SR = un_m + RL(2) * c_m;", "SR = un_m + c_m;"),
    ("HLL S_L both wet", "SL = sel_min(un_m - c_m, un_p - c_p);", "SL = sel_min(un_m - c_m, un_p + c_p);"),
    ("HLL dissipation sign", "out[k] = ((SR * FL[k] - SL * FR[k]) + SLSR * (UR[k] - UL[k])) * inv;",
     "out[k] = ((SR * FL[k] - SL * FR[k]) - SLSR * (UR[k] - UL[k])) * inv;"),
    ("hydrostatic b* = min", "real bs = sel_max(b_m, b_p);", "real bs = sel_min(b_m, b_p);"),
    ("donor reversed", "if (us > RL(0)) { Jn = J0n[L]; Ja = o->J0a[L]; }", "if (us < RL(0)) { Jn = J0n[L]; Ja = o->J0a[L]; }"),
    ("slope term sign", "return FMA(-(C_J * J0abs), db_dn, J0n);", "return FMA((C_J * J0abs), db_dn, J0n);"),
    ("grass |J0| drops sqrt", "*jabs = c * a;", "*jabs = c;"),
    ("sediment gradient L/R", "(b[R] - b[L]) * o->inv_h", "(b[L] - b[R]) * o->inv_h"),
    # ---- K8 / Eq.7
    ("K8 W dropped", "real bn = FMA(-(lam * W[c]), dJ, b[c]) + (tau * W[c]) * src;",
     "real bn = FMA(-lam, dJ, b[c]) + (tau * W[c]) * src;"),
    ("K8 y-flux of Qx from normal", "real dQx = (o->FQx[e] - o->FQx[c]) + (o->GQx[n] - o->GQx[c]);",
     "real dQx = (o->FQx[e] - o->FQx[c]) + (o->GQy[n] - o->GQy[c]);"),
    ("K8 no dry zeroing", "if (!(Hn > eps)) { Qxn = RL(0); Qyn = RL(0); }", "if (!(Hn > RL(0))) { Qxn = RL(0); Qyn = RL(0); }"),
    ("Eq.7 t1 factor", "double t1 = h / (2.0 * sqrt(M[0]));", "double t1 = h / sqrt(M[0]);"),
    ("Eq.7 M3 without W", "t3 = ((cell_aj(o, c, Hc) * pw) * a) * o->W[c];", "t3 = (cell_aj(o, c, Hc) * pw) * a;"),
    ("Eq.7 M2 drops |v|", "real t2 = a + SQRT(o->g * Hc);", "real t2 = SQRT(o->g * Hc);"),
    ("W = 1 - psi", "o->W[d] = RL(1.0 / (1.0 - (psi ? psi[s] : 0.0)));", "o->W[d] = RL(1.0 - (psi ? psi[s] : 0.0));"),
    ("wall ghost Qx not negated", "o->Qx[d] = negx ? -o->Qx[s] : o->Qx[s];", "o->Qx[d] = o->Qx[s];"),
    # ---- NEXT-4 closures
    ("Grass odd m drops |v|", "if (m % 2) pw = pw * a;", "if (m % 2) pw = pw * RL(1);"),
    ("Eq.4 sqrt(gH) -> gH", "(((s_rel - RL(1)) * SQRT(g * H)) * d50)", "(((s_rel - RL(1)) * (g * H)) * d50)"),
    ("Eq.4 A_J at H_half", "r_grass_mr(cell_aj(o, c, H[c]),", "r_grass_mr(cell_aj(o, c, o->Hh[c]),"),
    ("sources: absorption explicit", "real a = RL(1) / (RL(1) + tau * o->beta[c]);", "real a = RL(1) - tau * o->beta[c];"),
]


def run_one(name, old, new, k_tests, quiet=True):
    tmp = tempfile.mkdtemp(prefix="mut_")
    try:
        for d in ("oracle", "synth", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__", "libcsph_oracle.so"))
        path = os.path.join(tmp, SRC)
        src = open(path).read()
        n = src.count(old)
        if n != 1:
            return "NOMATCH(%d)" % n, 0.0
        open(path, "w").write(src.replace(old, new))
        # the pin tests import `oracle` and `synth` from the scratch root (tests/conftest.py)
        t0 = time.time()
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu",
                            "-p", "no:cacheprovider"] + k_tests,
                           cwd=tmp, capture_output=True, text=True, timeout=1800)
        dt = time.time() - t0
        if r.returncode == 0:
            return "SURVIVED", dt
        last = [l for l in r.stdout.splitlines() if l.startswith("FAILED") or "Error" in l]
        return "caught" + ((" by " + last[0].split("::")[-1][:60]) if last else ""), dt
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="", help="only mutations whose name contains this")
    a = ap.parse_args()
    res = []
    for name, old, new in MUTATIONS:
        if a.k and a.k not in name:
            continue
        st, dt = run_one(name, old, new, PIN_TESTS)
        res.append((name, st))
        print("%-32s %6.1fs  %s" % (name, dt, st), flush=True)
    surv = [n for n, s in res if s.startswith("SURVIVED") or s.startswith("NOMATCH")]
    print("\n%d mutations, %d caught, %d survived/unmatched: %s"
          % (len(res), len(res) - len(surv), len(surv), surv))
    sys.exit(1 if surv else 0)


if __name__ == "__main__":
    main()
