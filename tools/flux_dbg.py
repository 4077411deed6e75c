"""x-face fluxes of the fused kernel vs the oracle (dev aid; needs variants/libcsph_dbg.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2103_15196_b200 import csph
csph.SO_PATH = os.path.abspath("variants/libcsph_dbg.so")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 28
c = synth.config("C1"); f = synth.fill(c)
ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params)); ref.set_state(*f); ref.step(K)
buf = torch.zeros(c.ny * (c.nx + 1) * 4, dtype=torch.float64, device="cuda")
L = csph.lib(); L.csph_debug_buffer.argtypes = [ctypes.c_void_p]
print("set", L.csph_debug_buffer(buf.data_ptr()))
buf2 = torch.zeros(c.ny * c.nx * 6, dtype=torch.float64, device="cuda")
L.csph_debug_buffer2.argtypes = [ctypes.c_void_p]; L.csph_debug_buffer2(buf2.data_ptr())
g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, graphs=0))
g.set_state(*f); g.step(K); torch.cuda.synchronize()
d = buf.cpu().numpy().reshape(c.ny, c.nx + 1, 4)
FQ = ref.debug("FQx")[3:-3, 3:4 + c.nx]; FH = ref.debug("FH")[3:-3, 3:4 + c.nx]
ut = ref.debug_interior("ut")
n = 0
for i in range(c.nx + 1):
    j = 0
    if d[j, i, 1] != FQ[j, i] or d[j, i, 0] != FH[j, i]:
        n += 1
        if n <= 6:
            print("face", i, "FH gpu", d[j,i,0].hex(), "orc", FH[j,i].hex(), "| FQ gpu", d[j,i,1].hex(), "orc", FQ[j,i].hex())
for i in range(c.nx):
    if i >= 1 and d[0, i, 2] != ut[0, i - 1]:
        print("ut differs at cell", i - 1, d[0, i, 2].hex(), ut[0, i - 1].hex()); break
d2 = buf2.cpu().numpy().reshape(c.ny, c.nx, 6)
phix = ref.debug_interior("phix"); tau = ref.time()[2]
H, Qx, _, _ = ref.get_state()
for i in (75, 76, 77, 78, 79):
    print("cell", i, "gpu phix", d2[0, i, 0].hex(), "orc", phix[0, i].hex(), "Q", d2[0, i, 1].hex(), "theta", d2[0,i,2].hex(), (0.5*tau).hex(), "uu", d2[0,i,3].hex(), "f", d2[0,i,4], "r", d2[0,i,5].hex())
print("faces differing:", n, "state diff:", sum(int(np.sum(a != b)) for a, b in zip(g.get_state(), ref.get_state())))
