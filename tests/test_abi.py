"""The C-ABI library on a GPU-less host: it builds, loads, exports exactly the
symbols include/qsv.h declares, runs its host-only calls, and fails LOUDLY
(QSV_ERR_INTERNAL, never a silent CPU path) when asked to compute."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import build as B
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200.qsv import make_gate

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "qsv.h"


@pytest.fixture(scope="module", autouse=True)
def _built():
    B.build()
    O.build()


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(qsv_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    syms = declared_symbols()
    assert len(syms) >= 30
    assert set(syms) == set(qsv._SIGS), set(syms) ^ set(qsv._SIGS)


def test_library_exports_every_declared_symbol():
    L = C.CDLL(str(B.LIB))
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert qsv.lib().qsv_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(B.LIB)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly():
    L = qsv.lib()
    if L.qsv_device_count() > 0:
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = L.qsv_ctx_create(0, C.byref(h))
    assert rc == qsv.ERR_INTERNAL
    assert b"no CPU fallback" in L.qsv_last_error()
    with pytest.raises(qsv.QsvError):
        qsv.Context(0)
    # the multi-device context fails the same way (and validates its world first)
    with pytest.raises(qsv.InvalidInput):
        qsv.Context.multi([0, 0, 0])
    with pytest.raises(qsv.QsvError):
        qsv.Context.multi([0, 0])
    assert b"no CPU fallback" in L.qsv_last_error()


@pytest.mark.parametrize("name,wires,params", [
    ("h", [0], []), ("rx", [0], [0.3]), ("ry", [0], [-1.2]), ("rz", [0], [2.9]), ("p", [0], [0.7]),
    ("u3", [0], [0.1, -0.4, 2.2]), ("swap", [0, 1], []), ("rxx", [0, 1], [0.9]), ("ryy", [0, 1], [-2.1]),
    ("rzz", [0, 1], [1.3]), ("s", [0], []), ("t", [0], []), ("y", [0], []),
])
def test_abi_gate_matrix_matches_reference(name, wires, params):
    g = make_gate(name, wires, [], params)
    want = O.ref_gate_matrix(g) if O.REF_LIB.exists() else O.port_gate_matrix(g)
    assert np.max(np.abs(qsv.gate_matrix(g) - want)) <= 1e-16


def test_abi_gate_matrix_errors_mirror_reference():
    with pytest.raises(qsv.InvalidInput, match="unknown gate"):
        qsv.gate_matrix(make_gate("nope", [0]))
    with pytest.raises(qsv.InvalidInput, match="expected 1 params"):
        qsv.gate_matrix(make_gate("rx", [0], [], []))
    with pytest.raises(qsv.InvalidInput, match="not unitary"):
        qsv.gate_matrix(make_gate("custom", [0], custom=np.array([[1, 1], [0, 1]])))
    with pytest.raises(qsv.InvalidInput, match="disjoint"):
        make_gate("x", [0], [0])


def test_rng_fill_matches_reference_stream():
    for kind, k in (("u64", 0), ("uniform", 1), ("normal", 2)):
        for cnt in (1, 7, 1000, 300001):
            got = qsv.rng_fill(0, "cfg3", kind, cnt, nthreads=4)
            want = O.port_rng(0, "cfg3", k, cnt)
            assert np.array_equal(got, want), (kind, cnt)


def test_super_pass_planning_is_opt_in():
    # L2 super-passes pair consecutive passes only when asked (opts.super_bits)
    # and only when both tiles fit one chunk; the schedule marks head / tail
    from paper_2512_18995_b200 import workloads as W

    cir = W.cfg3_circuit(30)
    off, _ = qsv.plan_dry(30, cir.gates())
    assert off["npasses"] == off["ntile_passes"] == 4
    on, _ = qsv.plan_dry(30, cir.gates(), opts={"super_bits": 19})
    assert on["npasses"] == 2 and on["ntile_passes"] == 4
    assert on["bytes_per_exec"] == off["bytes_per_exec"] / 2
    sch = qsv.plan_schedule(30, cir.gates(), opts={"super_bits": 19})
    assert [s["pair"] for s in sch["steps"]] == [1, 2, 1, 2]
    small, _ = qsv.plan_dry(30, cir.gates(), opts={"super_bits": 15})  # no two tiles fit 2^15
    assert small["npasses"] == 4
    _, src = qsv.plan_dry(30, cir.gates(), opts={"super_bits": 19}, source_of_pass=0)
    assert "qsv_pair" in src and "ld.acquire.gpu" in src and "namespace pb" in src


@pytest.mark.parametrize("dtype,variant", [("c64", ""), ("c64", "QSV_X_NOPACK"), ("c128", ""),
                                           ("c128", "QSV_X_NOSCALE")])
def test_generated_pass_sources_compile_for_sm100a(dtype, variant, monkeypatch, tmp_path):
    # the codegen's arithmetic forms (host logic, no GPU): complex64 passes
    # compute on packed f32x2 registers unless QSV_X_NOPACK=1, the tangent
    # form leaves +-1 terms, and every variant's source cross-compiles with
    # nvcc for sm_100a exactly as NVRTC builds it on the GPU box
    import shutil
    import subprocess

    from paper_2512_18995_b200 import workloads as W

    if variant:
        monkeypatch.setenv(variant, "1")
    n = 20
    dt = qsv.C64 if dtype == "c64" else qsv.C128
    cir = W.cfg5_circuit(n, 2) if dtype == "c64" else W.cfg4_circuit(n, 2)
    info, src = qsv.plan_dry(n, cir.gates(), dtype=dt, source_of_pass=1)
    assert info["npasses"] >= 2 and "qsv_pass" in src
    packed = "fma.rn.f32x2" in src
    assert packed == (dtype == "c64" and variant != "QSV_X_NOPACK")
    if dtype == "c128":
        # tangent-form rows: a real rotation output is x0 + t*x1 (no multiply on x0)
        assert "mk(x0.x+" in src or "mk(x1.x+" in src
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    cu = tmp_path / "pass.cu"
    cu.write_text(src)
    r = subprocess.run([nvcc, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o",
                        str(tmp_path / "pass.cubin"), str(cu)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


def test_dense_block_planning_on_host():
    """opts.dense_blocks: the host-side fusion into <= 5-qubit blocks and their
    packing into 12-bit-tile passes (plan_dry, no GPU): every circuit family
    plans, blocks never exceed 3 per pass, and what the tensor-core pass does
    not cover is refused."""
    from paper_2512_18995_b200 import workloads as W
    from tests.helpers import random_circuit

    rng = qsv.Rng(3, "dense-plan")
    for n, cir in ((12, W.dense_brickwork_circuit(12, 10)), (20, W.dense_brickwork_circuit(20, 20)),
                   (16, W.cfg5_circuit(16, 4)), (14, random_circuit(rng, 14, 200))):
        info, _ = qsv.plan_dry(n, cir.gates(), dtype=qsv.C64, opts={"dense_blocks": 1})
        assert info["nblocks"] >= 1 and 1 <= info["npasses"] <= info["nblocks"]
        assert info["nblocks"] <= 3 * info["npasses"]
        assert info["ngates"] == len(cir.gates())
    # auto (dense_blocks = 0): deep local blocks take the tensor cores, the
    # BASELINE config families and shallow dense brickworks do not
    auto, _ = qsv.plan_dry(20, W.dense_local_circuit(20, 5, 20).gates(), dtype=qsv.C64)
    assert auto["nblocks"] > 0
    for n, cir in ((20, W.dense_brickwork_circuit(20, 20)), (16, W.cfg5_circuit(16, 4)), (12, W.cfg2_circuit()[0]),
                   (16, W.cfg4_circuit(16, 4))):
        info, _ = qsv.plan_dry(n, cir.gates(), dtype=qsv.C64)
        assert info["nblocks"] == 0, n
    off, _ = qsv.plan_dry(20, W.dense_local_circuit(20, 5, 20).gates(), dtype=qsv.C64, opts={"dense_blocks": -1})
    assert off["nblocks"] == 0
    with pytest.raises(qsv.InvalidInput):
        qsv.plan_dry(14, W.dense_brickwork_circuit(14, 2).gates(), dtype=qsv.C128, opts={"dense_blocks": 1})
    with pytest.raises(qsv.InvalidInput):
        qsv.plan_dry(10, W.dense_brickwork_circuit(10, 2).gates(), dtype=qsv.C64, opts={"dense_blocks": 1})


def header_struct_fields(name):
    """Field names of `typedef struct name { ... } name;` in include/qsv.h, in
    declaration order (array fields by their name)."""
    text = HEADER.read_text()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return re.findall(r"(\w+)\s*(?:\[[^\]]*\])?\s*;", body)


@pytest.mark.parametrize("name", ["qsv_gate", "qsv_obs", "qsv_opts", "qsv_plan_info"])
def test_ctypes_structs_mirror_the_header(name):
    """The Python mirror's ctypes structs lay out the header's fields in the
    same order (an option added to one and not the other would shift every
    later field across the boundary)."""
    py = [f for f, _ in getattr(qsv, name)._fields_]
    assert py == header_struct_fields(name), (py, header_struct_fields(name))


def test_lazy_layout_plans_the_qft_in_three_12bit_passes():
    """Host-only planning (qsv_plan_dry): with lazy layouts the 30q QFT + swaps
    needs no layout-restoring pass, so 12-bit complex128 tiles take it in 3
    passes (9 + 9 + 12 Hadamard wires) where the eager plan needs 4
    (DESIGN.md 4.1g); the default 11-bit geometry needs 4 either way."""
    from paper_2512_18995_b200 import workloads as W

    gates = W.cfg3_circuit(30).gates()
    npass = lambda o: qsv.plan_dry(30, gates, qsv.C128, 1, o)[0]["npasses"]
    assert npass({"tile_bits": 12, "lazy_layout": 1}) == 3
    assert npass({"tile_bits": 12}) == 4
    assert npass({"lazy_layout": 1}) == 4
    assert npass({}) == 4
