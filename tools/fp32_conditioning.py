"""Conditioning of R under fp32 rounding, CPU only.

Runs the fp64 oracle for 100 steps from the exact initial state and from the same state
rounded to fp32, and prints the 3.10 errors between the two (h, hu, hv, b) and the 99.9 %
quantile of the h error.  Usage: PYTHONPATH=. python tools/fp32_conditioning.py"""
import math

import numpy as np

import oracle
import synth

G = 9.81


def errs(gpu, ref):
    h, hu, hv, b = ref
    sh = np.max(np.abs(h)); sq = max(np.max(np.abs(hu)), np.max(np.abs(hv)), sh*math.sqrt(G*sh)); sb = max(np.max(np.abs(b)), sh)
    return [float(np.max(np.abs(g - r)) / s) for g, r, s in zip(gpu, ref, [sh, sq, sq, sb])]
for name,n,ny in (("C5",300,260),("C3",256,200)):
    c = synth.config(name, n, ny)
    f = list(synth.fill(c))
    outs=[]
    for r32 in (False, True):
        ff=[x.astype(np.float32).astype(np.float64) if r32 else x for x in f]
        o=oracle.Oracle(c.nx,c.ny,c.dx,oracle.Params(**c.params)); o.set_state(*ff); o.step(100); outs.append(o.get_state())
    e=errs(outs[1],outs[0]); sh=np.max(np.abs(outs[0][0]))
    print(name, e, np.quantile(np.abs(outs[1][0]-outs[0][0])/sh,0.999))
