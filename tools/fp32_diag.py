"""Where does the fp32 GPU path part from the binary32 oracle?  (dev aid)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
from paper_2103_15196_b200 import csph

for name, n, ny in (("C3", 256, 200), ("C4", 192, 256)):
    c = synth.config(name, n, ny)
    f = synth.fill(c)
    for hgs in (1, 0):
        ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params), precision=32)
        ref.set_state(*f)
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, precision=32, hgs=hgs, graphs=0))
        g.set_state(*f)
        for k in range(100):
            ref.step(1); g.step(1)
            a = g.get_state(); r = ref.get_state()
            bad = [int(np.sum(x != y)) for x, y in zip(a, r)]
            if any(bad):
                j, i = np.argwhere(a[0] != r[0])[0] if bad[0] else np.argwhere(a[[0,1,2,3][bad.index(max(bad))]] != r[bad.index(max(bad))])[0]
                fi = [q for q in range(4) if bad[q]]
                print(name, "hgs", hgs, "first diff at step", k + 1, "fields", fi, bad)
                for q in fi:
                    jj, ii = np.argwhere(a[q] != r[q])[0]
                    print("  field", q, "at", (jj, ii), "gpu", a[q][jj, ii], "orc", r[q][jj, ii], "H", r[0][jj, ii], "b", r[3][jj, ii])
                break
        else:
            print(name, "hgs", hgs, "no diff in 100 steps")
        g.destroy()
