import numpy as np, sys
sys.path.insert(0, '.')
import oracle as O, synth, paper_1708_05357_b200 as D
A, b = synth.lasso_dense(1000, 800, seed=3)
lam = 0.05
ref_set = np.sort(O.select_policy(O.SEL_UNIFORM, 800, 200, 3, 11))
for passes in (1, 2):
    for mode in ("internal", "explicit"):
        with D.create(A, b, lam, D.LASSO, seed=11) as P:
            sel, _ = P.select(D.SEL_UNIFORM, m=200, round=3)
            if mode == "internal":
                P.scd_epoch(passes=passes, seed=11, round=3)
            else:
                for p in range(passes):
                    P.scd_epoch(perm=O.make_perm(ref_set, 11, 3, p))
            a_gpu, v_gpu, _ = P.get_state()
        alpha, vt = np.zeros(800), -b.copy()
        for p in range(passes):
            O.scd_pass(O.LASSO, A, O.col_norms(A), None, lam, alpha, vt, O.make_perm(ref_set, 11, 3, p))
        print(passes, mode, np.abs(a_gpu - alpha).max(), np.abs(v_gpu - vt).max())
