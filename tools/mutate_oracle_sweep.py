#!/usr/bin/env python3
"""Systematic mutation sweep over the CPU oracle's arithmetic (test infrastructure).

tools/mutate_oracle.py applies a hand-picked list of plausible slips; this sweep generates
every single-operator mutant of the lines that compute R -- the helpers (minmod, icbrt, pow,
Grass, Eq.2/4/5, face force, HLL), the ghosts, the Eq.7 reduction and the step itself
(orc_tau_from_M, orc_step_tau) -- and reports which ones no `-m "not gpu"` pin catches:

  arithmetic   ' + ' <-> ' - ',  ' * ' -> ' / ',  'FMA(-' -> 'FMA('
  relational   ' > ' <-> ' < ',  ' >= ' <-> ' <= '
  boundary     ' > ' -> ' >= ',  ' < ' -> ' <= ',  ' >= ' -> ' > ',  ' <= ' -> ' < '
  index        'sx' <-> 'sy'
  constant     'RL(0.5)' -> 'RL(0.25)', 'RL(1)' -> 'RL(2)', 'RL(2)' -> 'RL(3)'

Boundary mutants that survive are mostly equivalent on the pins' inputs (a strict test of a
continuous value that never sits exactly on the threshold); they are listed separately.
Loop headers and comments are not mutated.  Runs N workers, each mutant in a scratch copy
(nothing in the repo is modified).

    python tools/mutate_oracle_sweep.py [-j 6] [--limit N] [--kind arithmetic,index]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import re
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import mutate_oracle as mo  # noqa: E402

ROOT = mo.ROOT
SRC = os.path.join(ROOT, mo.SRC)

OPS = [
    ("arithmetic", " + ", " - "), ("arithmetic", " - ", " + "), ("arithmetic", " * ", " / "),
    ("arithmetic", "FMA(-", "FMA("),
    ("relational", " > ", " < "), ("relational", " < ", " > "),
    ("relational", " >= ", " <= "), ("relational", " <= ", " >= "),
    ("boundary", " > ", " >= "), ("boundary", " < ", " <= "),
    ("boundary", " >= ", " > "), ("boundary", " <= ", " < "),
    ("index", "sx", "sy"), ("index", "sy", "sx"),
    ("constant", "RL(0.5)", "RL(0.25)"), ("constant", "RL(1)", "RL(2)"),
    ("constant", "RL(2)", "RL(3)"),
]

# the functions that compute R (name -> mutated); the API / validation / allocation code is not
FUNCS = ["sel_min", "sel_max", "r_minmod", "r_icbrt", "pow_pinned", "grass_pow", "r_grass_mr",
         "r_aj_eq4", "r_slope_flux", "r_shamov_gate", "r_bed_mobile", "face_force", "r_hll_face",
         "ghost_copy", "mirror_fill", "cell_aj", "reduce_M", "orc_tau_from_M", "orc_step_tau"]


def function_lines(src: str) -> set[int]:
    """0-based line numbers inside the bodies of FUNCS (brace matching from the header)."""
    lines = src.splitlines()
    keep = set()
    i = 0
    while i < len(lines):
        m = re.match(r"^(?:static\s+)?(?:[a-z_0-9]+\s+)+\*?\s*([a-z_A-Z0-9]+)\(", lines[i])
        if m and m.group(1) in FUNCS and not lines[i].rstrip().endswith(";"):
            depth = 0
            j = i
            started = False
            while j < len(lines):
                depth += lines[j].count("{") - lines[j].count("}")
                started = started or "{" in lines[j]
                keep.add(j)
                if started and depth <= 0:
                    break
                j += 1
            i = j + 1
            continue
        i += 1
    return keep


def code_part(line: str) -> str:
    """The line without a trailing comment (mutations apply to the code only)."""
    for tok in ("/*", "//"):
        k = line.find(tok)
        if k >= 0:
            line = line[:k]
    return line


def mutants(kinds: set[str]):
    src = open(SRC).read()
    lines = src.splitlines(keepends=True)
    keep = function_lines(src)
    offs = [0]
    for l in lines:
        offs.append(offs[-1] + len(l))
    out = []
    for i in sorted(keep):
        line = lines[i]
        st = line.lstrip()
        if st.startswith(("/*", "*", "//", "#")) or re.search(r"\bfor\s*\(", line):
            continue
        code = code_part(line)
        for kind, old, new in OPS:
            if kind not in kinds:
                continue
            start = 0
            while True:
                k = code.find(old, start)
                if k < 0:
                    break
                start = k + 1
                if kind == "index" and not re.search(r"\b%s\b" % old, code[k - 1:k + len(old) + 1]):
                    continue
                # a boundary/relational mutant of ' > ' must not hit the '>' of '>='
                mutated = src[:offs[i] + k] + new + src[offs[i] + k + len(old):]
                name = "L%d %s '%s'->'%s': %s" % (i + 1, kind, old.strip(), new.strip(),
                                                    code.strip()[:70])
                out.append((name, kind, mutated))
    return out


def run_mutant(name, mutated):
    tmp = mo.tempfile.mkdtemp(prefix="mutsw_")
    try:
        for d in ("oracle", "synth", "tests"):
            mo.shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                               ignore=mo.shutil.ignore_patterns("__pycache__", "libcsph_oracle.so"))
        open(os.path.join(tmp, mo.SRC), "w").write(mutated)
        t0 = time.time()
        try:
            r = mo.subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu",
                                   "-p", "no:cacheprovider"] + mo.PIN_TESTS,
                                  cwd=tmp, capture_output=True, text=True, timeout=900)
            code = r.returncode
        except mo.subprocess.TimeoutExpired:
            return "caught (timeout)", time.time() - t0
        if code == 0:
            return "SURVIVED", time.time() - t0
        if code not in (1,):  # build failure / crash: the mutant does not compile or run
            return "caught (rc %d)" % code, time.time() - t0
        return "caught", time.time() - t0
    finally:
        mo.shutil.rmtree(tmp, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--kind", default="arithmetic,relational,boundary,index,constant")
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--grep", default="", help="only mutants whose name contains this")
    a = ap.parse_args()
    ms = mutants(set(a.kind.split(",")))
    if a.grep:
        ms = [m for m in ms if a.grep in m[0]]
    if a.limit:
        ms = ms[:a.limit]
    if a.list:
        for n, _, _ in ms:
            print(n)
        print(len(ms), "mutants")
        return
    t0 = time.time()
    res = []
    with cf.ThreadPoolExecutor(a.j) as ex:
        futs = {ex.submit(run_mutant, n, m): (n, k) for n, k, m in ms}
        for f in cf.as_completed(futs):
            n, k = futs[f]
            st, dt = f.result()
            res.append((n, k, st))
            if st == "SURVIVED":
                print("SURVIVED %s" % n, flush=True)
    print("\n%d mutants in %.0f s" % (len(res), time.time() - t0))
    for kind in sorted({k for _, k, _ in res}):
        rk = [r for r in res if r[1] == kind]
        sv = [r for r in rk if r[2] == "SURVIVED"]
        print("%-11s %4d mutants, %4d caught, %3d survived" % (kind, len(rk), len(rk) - len(sv),
                                                               len(sv)))
    sv = sorted(r[0] for r in res if r[2] == "SURVIVED")
    print("\nsurvivors:")
    for n in sv:
        print("  " + n)


if __name__ == "__main__":
    main()
