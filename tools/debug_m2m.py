import sys, numpy as np
sys.path.insert(0, '.')
from oracle import ref
import paper_2006_15367_b200 as hb
pos, q2 = ref.generate_inputs("cube", 20000, 3.0, 31)
q = q2[:, 0] + 1j * q2[:, 1]
rs = ref.RefSetup(pos, q2, ref.config(digits=3))
setup = hb.build_setup(pos, q, hb.RunConfig(digits=3))
eng = hb.RankEngine(setup)
eng.c2m_phase(); eng.m2m_pass()
a = eng.multipole(4); b = rs.expansions(2, 0, 4)
err = np.abs(a - b) / np.abs(b).max()
bad_nodes = np.where(err.max(1) > 1e-10)[0]
print('bad nodes', bad_nodes.size, 'of', a.shape[0], bad_nodes[:20])
co = setup.array("L4.child_off", np.uint64)
print('children count of bad', [int(co[i+1]-co[i]) for i in bad_nodes[:20]])
print('children count of good', [int(co[i+1]-co[i]) for i in range(10)])
n = 28
e = err[bad_nodes[0]].reshape(n, n)
print('bad samples rows/cols', np.argwhere(e > 1e-10)[:40].tolist())
from oracle import hfmm_np
mp5 = eng.multipole(5)
node = int(bad_nodes[0])
ch = setup.array("L4.children", np.uint64)[int(co[node]):int(co[node+1])].astype(int)
c4 = setup.array("L4.centers", np.float64).reshape(-1, 3); c5 = setup.array("L5.centers", np.float64).reshape(-1, 3)
dirs = hfmm_np.directions(28, 28)
contrib = []
for c in ch:
    up = hfmm_np.fft_interpolate(mp5[c].reshape(18, 18), 28, 28).reshape(-1)
    contrib.append(up * np.exp(1j * 2 * np.pi * (dirs @ (c5[c] - c4[node]))))
contrib = np.array(contrib)
print('ref vs sum contrib', np.abs(contrib.sum(0) - b[node]).max())
d = a[node] - b[node]
# least squares: d ~ sum_c w_c contrib_c
w, *_ = np.linalg.lstsq(contrib.T, d, rcond=None)
print('diff as combination of child contributions:', np.round(w, 3), 'resid', np.abs(contrib.T @ w - d).max())
