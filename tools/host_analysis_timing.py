import time
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model
from paper_2307_16830_b200 import kkt, sparse
am=build_model('C3'); m=am.model
cs=kkt.symbolic_condense(m.hess_rows,m.hess_cols,m.jac_rows,m.jac_cols,m.n_var)
perm=sparse.amd_order(cs.matrix)
for i in range(3):
    t=time.perf_counter()
    cs=kkt.symbolic_condense(m.hess_rows,m.hess_cols,m.jac_rows,m.jac_cols,m.n_var)
    t1=time.perf_counter()
    sym=sparse.symbolic_cholesky(cs.matrix, perm)
    t2=time.perf_counter()
    print(f"condense {1e3*(t1-t):.1f} symbolic {1e3*(t2-t1):.1f}")
