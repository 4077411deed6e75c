"""First step where the fused path parts from the oracle on C1 (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
from paper_2103_15196_b200 import csph
c = synth.config("C1")
f = synth.fill(c)
ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params)); ref.set_state(*f)
for hgs in (1, 0):
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params)); ref.set_state(*f)
    g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, graphs=0, hgs=hgs))
    g.set_state(*f)
    for k in range(100):
        ref.step(1); g.step(1)
        a, r = g.get_state(), ref.get_state()
        bad = [np.argwhere(x != y) for x, y in zip(a, r)]
        if any(len(b) for b in bad):
            print("hgs", hgs, "step", k + 1)
            for q, b in enumerate(bad):
                for (j, i) in b[:4]:
                    print("  field", q, (j, i), a[q][j, i].hex(), r[q][j, i].hex(), "H", r[0][j, i])
            break
    else:
        print("hgs", hgs, "no diff")
