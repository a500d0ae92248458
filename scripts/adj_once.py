import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18995_b200 import qsv, workloads as W
cir = W.cfg1_circuit(20, trainable=True)
g = qsv.adjoint_gradients(cir, dtype=qsv.C128)
g = qsv.adjoint_gradients(cir, dtype=qsv.C64)
