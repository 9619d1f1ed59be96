"""Ad-hoc per-phase parity + timing check on a GPU box (development tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import ref
import paper_2006_15367_b200 as hb

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

shape, n, ext, seed, dig = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
pos, q2 = ref.generate_inputs(shape, n, ext, seed)
q = q2[:, 0] + 1j * q2[:, 1]
t = time.time()
rs = ref.RefSetup(pos, q2, ref.config(digits=dig))
print('levels', rs.levels, 'leaves', rs.num_leaves, 'setup', time.time() - t, flush=True)
setup = hb.build_setup(pos, q, hb.RunConfig(digits=dig))
eng = hb.RankEngine(setup)
L, top = setup.levels, setup.top_level
eng.c2m_phase()
t = time.time(); r = rs.expansions(1, 0, L); print('ref c2m', time.time() - t, flush=True)
print('C2M leaf mp rel', rel(eng.multipole(L), r), flush=True)
eng.m2m_pass()
for l in range(L - 1, top - 1, -1):
    print(f'M2M L{l} mp rel', rel(eng.multipole(l), rs.expansions(2, 0, l)), flush=True)
eng.m2l_pass()
for l in range(top, L + 1):
    print(f'M2L L{l} loc rel', rel(eng.local_expansion(l), rs.expansions(3, 1, l)), flush=True)
eng.l2l_pass()
for l in range(top + 1, L + 1):
    print(f'L2L L{l} loc rel', rel(eng.local_expansion(l), rs.expansions(4, 1, l)), flush=True)
pot_sorted = eng.l2o_near_phase()
_, rpot = rs.expansions(5, 1, L, want_pot=True)
print('final sorted pot rel', rel(pot_sorted, rpot), flush=True)
res = eng.evaluate()
t = time.time(); rp, sec, fl = rs.evaluate(); print('ref eval', time.time() - t, sec)
print('evaluate() input-order rel', rel(res.potentials, rp), res.phase_ms)
for i in range(3):
    res = eng.evaluate()
    print('gpu ms', res.phase_ms)
obs = np.arange(1000) * (n // 1000)
d = hb.direct_potential(pos, q, obs)
dr = ref.direct(pos, q2, obs[:100], nthreads=16)
print('gpu direct vs ref direct (100)', rel(d[:100], dr))
print('fmm err vs direct: gpu', rel(res.potentials[obs], d), 'ref', rel(rp[obs], d))
