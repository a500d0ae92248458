import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18995_b200 import qsv, workloads as W
cir = W.cfg1_circuit(24, trainable=True)
qsv.adjoint_gradients(cir, dtype=qsv.C128)
