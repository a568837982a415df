import dataclasses, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import rsk_synth as S
from oracle import pipeline as opipe, operators as ops
from paper_2306_15049_b200.pipeline import GpuSolver
cfg = dataclasses.replace(S.CONFIGS['C6'], n=32, M=8, gamma_lo=1e-4, gamma_hi=1e1, idx=(4, 5, 6, 6, 7, 7), inner='minres', tol=1e-10, n_c=16, J=4, K_out=2)
inp = S.make_inputs(cfg)
ref = opipe.run(cfg, inp, keep_steps=True)
dev = torch.device('cuda', 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
sol = GpuSolver(cfg, None, inp['gamma'], check_every=4)
sol.set_data(t(inp['x_true'].ravel()), t(inp['xi']))
n = cfg.n
wx, wy = ops.identity_weights(n)
st = opipe.StepState(0, wx, wy, None, None, None)
for k, rs in enumerate(ref['steps']):
    sol.h.set_weights(t(st.wx.ravel()), t(st.wy.ravel()))
    dst = {}
    if st.V_i1 is not None: dst['V_i1'] = t(st.V_i1.T)
    if st.X_prev is not None: dst['X_prev'] = t(st.X_prev.T); dst['G_prev'] = t(st.G_prev.T)
    o, X = sol.outer_step(k, dst)
    print('k', k, 'gpu its', o.iters, 'ref', rs.iters)
    print('   gpu applies-iters', o.applies - o.iters, 'ref', rs.applies - rs.iters)
    print('   gpu relres', o.relres, 'ref', rs.relres)
    print('   gpu m_used', o.m_used, 'keep', o.keep_ghat)
    wx, wy = ops.irn_weights(rs.X[:, rs.lstar].reshape(n, n), cfg.tau)
    st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1, st.wx, st.wy)
