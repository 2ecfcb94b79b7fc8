import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2008_01938_b200 as pd
from oracle import pyoracle
o = pyoracle.load_c()
offs, init = o.generate_sdp(20000, 1024, 11, False, 4096)
t = pd.solve_sequential(pd.SdpInstance(20000, offs, init, "min"))
w, _ = o.sdp_solve(offs, init, 20000, "min")
print("equal", np.array_equal(t.cells, w))
