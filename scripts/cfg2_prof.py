"""One cfg2 forward + <Z_i> (for an ncu launch list)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18995_b200 import qsv, workloads as W
cir, data = W.cfg2_circuit()
p = qsv.Plan(12, cir.gates(), dtype=qsv.C64)
st = qsv.QubitState(12, batch=4096, dtype=qsv.C64)
for _ in range(3):
    qsv.check(qsv.lib().qsv_state_set_basis(st.h, 0)); p.execute(st, data); z = st.expect_z_all()
print("ok", z[0][:3])
