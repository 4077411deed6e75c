"""C1 fused vs oracle at step 11 for library variants (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
from paper_2103_15196_b200 import csph
csph.SO_PATH = os.path.abspath(sys.argv[1])
c = synth.config("C1"); f = synth.fill(c)
ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params)); ref.set_state(*f); ref.step(11)
out = []
for path in (0, 1):
    g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, graphs=0, path=path))
    g.set_state(*f); g.step(11)
    a = g.get_state()
    out.append(f"path{path} Qx83 {a[1][0,83].hex()} ndiff {sum(int(np.sum(x != y)) for x, y in zip(a, ref.get_state()))}")
print(os.path.basename(sys.argv[1]), "oracle", ref.get_state()[1][0, 83].hex(), " | ".join(out))
