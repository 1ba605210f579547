import numpy as np, sys
sys.path.insert(0, '.')
import oracle as O, synth, paper_1708_05357_b200 as D
d, n = 2000, 1000
A, b = synth.lasso_dense(d, n, seed=2200)
lam = 0.05
for ctas in (1, 16):
    for m in (16, 32, 48, 64, 250):
        for W in (4, 16):
            order = synth.permutation(np.arange(m), 5)
            with D.create(A, b, lam, D.LASSO, scd_block=W, m=m, scd_ctas=ctas) as P:
                P.select(D.SEL_SEQUENTIAL, m=m, round=0)
                P.scd_epoch(perm=order)
                a_gpu, v_gpu, _ = P.get_state()
            alpha = np.zeros(n); vt = -b.copy()
            O.scd_pass(O.LASSO, A, O.col_norms(A), None, lam, alpha, vt, order)
            err = np.abs(a_gpu - alpha)
            bad = np.nonzero(err > 1e-12)[0]
            pos = {j: t for t, j in enumerate(order)}
            print(ctas, m, W, err.max(), sorted(pos[j] for j in bad)[:6])
