"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

  ref()     oracle/_ref/libquasar_ref.so: the reference's own qubit headers
            (/root/reference/proj/include/quasar, unmodified) compiled here
            against include/eigen_subset by oracle/Makefile.
  port()    oracle/_build/libqsv_oracle.so: the plain-C restatement
            (oracle/qsv_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module, and only as the checker / the CPU
baseline. The product (paper_2512_18995_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libquasar_ref.so"
PORT_LIB = HERE / "_build" / "libqsv_oracle.so"
REFERENCE_INCLUDE = Path("/root/reference/proj/include")


class RefGate(C.Structure):
    _fields_ = [
        ("name", C.c_char * 16),
        ("nwires", C.c_int32),
        ("wires", C.c_int32 * 2),
        ("ncontrols", C.c_int32),
        ("controls", C.c_int32 * 6),
        ("nparams", C.c_int32),
        ("params", C.c_double * 3),
        ("trainable", C.c_int32),
        ("encode", C.c_int32),
        ("custom", C.POINTER(C.c_double)),
    ]


class RefObs(C.Structure):
    _fields_ = [("nwires", C.c_int32), ("wires", C.POINTER(C.c_int32)), ("basis", C.c_char_p)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(force: bool = False) -> None:
    """Builds the C restatement, and the reference library when /root/reference exists."""
    targets = [str(PORT_LIB)]
    if REFERENCE_INCLUDE.exists():
        targets.append("ref")
    subprocess.run(["make", "-C", str(HERE)] + (["-B"] if force else []) + targets, check=True,
                   capture_output=True)


_ref = _port = None


def ref():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} missing (built from /root/reference by oracle/Makefile)")
        L = C.CDLL(str(REF_LIB))
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


def port():
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            build()
        L = C.CDLL(str(PORT_LIB))
        L.qo_norm2.restype = C.c_double
        L.qo_rng_next_u64.restype = C.c_uint64
        L.qo_rng_uniform.restype = C.c_double
        L.qo_rng_normal.restype = C.c_double
        L.qo_rng_next_below.restype = C.c_uint64
        L.qo_rng_sizeof.restype = C.c_size_t
        L.qo_gate_sizeof.restype = C.c_size_t
        _port = L
    return _port


def gate_struct(g, keep) -> RefGate:
    """g: any object with name/wires/controls/params/trainable/encode/custom."""
    r = RefGate()
    r.name = g.name.encode()
    r.nwires = len(g.wires)
    for i, w in enumerate(g.wires):
        r.wires[i] = w
    r.ncontrols = len(g.controls)
    for i, w in enumerate(g.controls):
        r.controls[i] = w
    r.nparams = len(g.params)
    for i, p in enumerate(g.params):
        r.params[i] = p
    r.trainable = int(bool(g.trainable))
    r.encode = int(bool(g.encode))
    if getattr(g, "custom", None) is not None:
        m = np.ascontiguousarray(np.asarray(g.custom, dtype=np.complex128)).view(np.float64).ravel().copy()
        keep.append(m)
        r.custom = m.ctypes.data_as(C.POINTER(C.c_double))
    return r


def gate_structs(gates):
    keep = []
    arr = (RefGate * max(1, len(gates)))()
    for i, g in enumerate(gates):
        arr[i] = gate_struct(g, keep)
    return arr, keep


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------ reference ---
def ref_forward(n, gates, init=None, data=None):
    """Circuit::forward through the reference itself. Returns (rows, 2^n) complex."""
    L = ref()
    arr, keep = gate_structs(gates)
    rows = 0 if data is None or len(data) == 0 else len(data)
    slots = 0
    d = None
    if rows:
        d = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(rows, -1))
        slots = d.shape[1]
    out = np.zeros((max(rows, 1), 1 << n), dtype=np.complex128)
    ini = None if init is None else np.ascontiguousarray(init, dtype=np.complex128)
    rc = L.ref_forward(n, arr, len(gates), None if ini is None else _p(ini), None if d is None else _p(d), rows,
                       slots, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


def _obs_array(obs):
    arr = (RefObs * max(1, len(obs)))()
    keep = []
    for i, (wires, basis) in enumerate(obs):
        w = (C.c_int32 * max(1, len(wires)))(*wires)
        b = basis.encode()
        keep += [w, b]
        arr[i].nwires = len(wires)
        arr[i].wires = C.cast(w, C.POINTER(C.c_int32))
        arr[i].basis = b
    return arr, keep


def ref_expectation(n, amps, obs):
    """expectation_one per (wires, basis)."""
    L = ref()
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    arr, keep = _obs_array(obs)
    out = np.zeros(max(1, len(obs)))
    rc = L.ref_expectation(n, _p(a), len(obs), arr, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out[: len(obs)]


def ref_marginal(n, amps, wires):
    L = ref()
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    w = (C.c_int32 * len(wires))(*wires)
    out = np.zeros(1 << len(wires))
    rc = L.ref_marginal_probabilities(n, _p(a), len(wires), w, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


def ref_measure(n, amps, shots, wires, seed, label):
    L = ref()
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    w = (C.c_int32 * len(wires))(*wires)
    out = np.zeros(1 << len(wires), dtype=np.uint64)
    rc = L.ref_measure(n, _p(a), shots, len(wires), w, C.c_uint64(seed), label.encode(), _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


def ref_gate_matrix(g):
    L = ref()
    keep = []
    s = gate_struct(g, keep)
    out = np.zeros(32)
    rc = L.ref_gate_matrix(C.byref(s), _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    d = 2 if len(g.wires) == 1 else 4
    return out[: 2 * d * d].view(np.complex128).reshape(d, d)


def ref_qft_gates(n):
    L = ref()
    cap = n * (n + 1) // 2 + 1
    arr = (RefGate * cap)()
    cnt = L.ref_qft_gates(n, arr, cap)
    if cnt < 0:
        raise OracleError(-cnt, L.ref_last_error().decode())
    return [arr[i] for i in range(cnt)]


def ref_rng(seed, label, kind, count, arg=0):
    """kind: 0 u64, 1 uniform, 2 normal, 3 next_below(arg)."""
    L = ref()
    out = np.zeros(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    rc = L.ref_rng_draw(C.c_uint64(seed), None if label is None else label.encode(), kind, C.c_uint64(arg), count,
                        _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


def ref_adjoint(n, gates, obs, data=()):
    L = ref()
    arr, keep = gate_structs(gates)
    oarr, okeep = _obs_array(obs)
    d = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    pout = np.zeros(max(1, sum(len(g.params) for g in gates)))  # ref_driver.cpp writes every param gradient
    dout = np.zeros(max(1, len(d)))
    npar = C.c_int()
    rc = L.ref_adjoint(n, arr, len(gates), len(obs), oarr, _p(d) if d.size else None, len(d), _p(pout),
                       C.byref(npar), _p(dout))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return pout[: npar.value], dout[: len(d)]


def ref_time_apply(n, gates, amps):
    """Applies gates with the reference apply_gate; returns (seconds, new amps)."""
    L = ref()
    arr, keep = gate_structs(gates)
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    sec = C.c_double()
    rc = L.ref_time_apply(n, arr, len(gates), _p(a), 1, C.byref(sec))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return sec.value, a


# ------------------------------------------------------ C restatement -----
def port_forward(n, gates, init=None, data=None):
    L = port()
    arr, keep = gate_structs(gates)
    rows = 0 if data is None or len(data) == 0 else len(data)
    slots = 0
    d = None
    if rows:
        d = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(rows, -1))
        slots = d.shape[1]
    out = np.zeros((max(rows, 1), 1 << n), dtype=np.complex128)
    ini = None if init is None else np.ascontiguousarray(init, dtype=np.complex128)
    rc = L.qo_forward(n, arr, len(gates), None if ini is None else _p(ini), None if d is None else _p(d), rows, slots,
                      _p(out))
    if rc:
        raise OracleError(rc, "qo_forward failed")
    return out


def port_apply_matrix(psi, n, m, wires, controls=(), zero_off_control=False):
    L = port()
    a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
    mm = np.ascontiguousarray(m, dtype=np.complex128)
    w = (C.c_int32 * len(wires))(*wires)
    c = (C.c_int32 * max(1, len(controls)))(*controls)
    rc = L.qo_apply_matrix(_p(a), n, _p(mm), len(wires), w, len(controls), c, int(zero_off_control))
    if rc:
        raise OracleError(rc, "qo_apply_matrix failed")
    return a


def port_expectation(n, amps, wires, basis):
    L = port()
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    w = (C.c_int32 * max(1, len(wires)))(*wires)
    out, im = C.c_double(), C.c_double()
    rc = L.qo_expectation(n, _p(a), len(wires), w, basis.encode(), C.byref(out), C.byref(im))
    if rc not in (0, -4):
        raise OracleError(rc, "qo_expectation failed")
    return out.value, im.value


def port_marginal(n, amps, wires):
    L = port()
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    w = (C.c_int32 * len(wires))(*wires)
    out = np.zeros(1 << len(wires))
    L.qo_marginal_probabilities(n, _p(a), len(wires), w, _p(out))
    return out


def port_rng(seed, label, kind, count, arg=0):
    L = port()
    st = C.create_string_buffer(int(L.qo_rng_sizeof()))
    L.qo_rng_init(st, C.c_uint64(seed), None if label is None else label.encode())
    out = np.zeros(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    L.qo_rng_draw(st, kind, C.c_uint64(arg), C.c_int64(count), _p(out))
    return out


def port_gate_matrix(g):
    L = port()
    keep = []
    s = gate_struct(g, keep)
    out = np.zeros(32)
    k = L.qo_gate_matrix(C.byref(s), _p(out))
    if k < 0:
        raise OracleError(k, "qo_gate_matrix failed")
    d = 1 << k
    return out[: 2 * d * d].view(np.complex128).reshape(d, d)


# ------------------------------------------------- mixed states (channels) ---
# Ops of a mixed-state run: a qsv Gate, or (channel_name, wire, parameter)
# with channel_name in CHANNEL_KINDS (channel.hpp:40-69).
CHANNEL_KINDS = {"bit_flip": 1, "phase_flip": 2, "depolarizing": 3, "amplitude_damping": 4, "phase_damping": 5}


def ref_mixed_run(n, ops, init=None):
    """to_mixed + apply_gate / apply_channel in order (reference library)."""
    L = ref()
    gates = [op for op in ops if not isinstance(op, tuple)]
    arr, keep = gate_structs(gates)
    kinds = (C.c_int32 * max(1, len(ops)))(*[0 if not isinstance(op, tuple) else CHANNEL_KINDS[op[0]] for op in ops])
    wires = (C.c_int32 * max(1, len(ops)))(*[op[1] if isinstance(op, tuple) else 0 for op in ops])
    params = np.array([op[2] if isinstance(op, tuple) else 0.0 for op in ops] or [0.0])
    dim = 1 << n
    out = np.zeros((dim, dim), dtype=np.complex128)
    ini = None if init is None else np.ascontiguousarray(init, dtype=np.complex128)
    rc = L.ref_mixed_run(n, None if ini is None else _p(ini), len(ops), kinds, wires, _p(params), arr, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


def ref_density_expectation(n, rho, obs):
    L = ref()
    r = np.ascontiguousarray(rho, dtype=np.complex128)
    arr, keep = _obs_array(obs)
    out = np.zeros(max(1, len(obs)))
    rc = L.ref_density_expectation(n, _p(r), len(obs), arr, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out[: len(obs)]


def ref_density_marginal(n, rho, wires):
    L = ref()
    r = np.ascontiguousarray(rho, dtype=np.complex128)
    w = (C.c_int32 * len(wires))(*wires)
    out = np.zeros(1 << len(wires))
    rc = L.ref_density_marginal(n, _p(r), len(wires), w, _p(out))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return out


_SQ = np.sqrt
_KX = np.array([[0, 1], [1, 0]], complex)
_KY = np.array([[0, -1j], [1j, 0]], complex)
_KZ = np.array([[1, 0], [0, -1]], complex)


def port_kraus(name, p):
    """channel.hpp:40-69 restated."""
    i2 = np.eye(2, dtype=complex)
    if name == "bit_flip":
        return [_SQ(1 - p) * i2, _SQ(p) * _KX]
    if name == "phase_flip":
        return [_SQ(1 - p) * i2, _SQ(p) * _KZ]
    if name == "depolarizing":
        return [_SQ(1 - 3 * p / 4) * i2, _SQ(p / 4) * _KX, _SQ(p / 4) * _KY, _SQ(p / 4) * _KZ]
    if name == "amplitude_damping":
        return [np.array([[1, 0], [0, _SQ(1 - p)]], complex), np.array([[0, _SQ(p)], [0, 0]], complex)]
    if name == "phase_damping":
        return [np.array([[1, 0], [0, _SQ(1 - p)]], complex), np.array([[0, 0], [0, _SQ(p)]], complex)]
    raise ValueError(name)


def _conjugate_columns_rows(rho, n, m, wires, controls=()):
    """state.hpp:159-172 / channel.hpp:80-92: M on every column, conj(M) on
    every row, with the strided kernel restatement."""
    t = rho.copy()
    for c in range(t.shape[1]):
        t[:, c] = port_apply_matrix(t[:, c], n, m, wires, controls)
    mc = np.conj(m)
    for r in range(t.shape[0]):
        t[r, :] = port_apply_matrix(t[r, :], n, mc, wires, controls)
    return t


def port_mixed_run(n, ops, init=None):
    """Restatement of to_mixed + apply_gate (mixed) + apply_channel."""
    dim = 1 << n
    psi = np.zeros(dim, complex) if init is None else np.asarray(init, complex)
    if init is None:
        psi[0] = 1
    rho = np.outer(psi, psi.conj())
    for op in ops:
        if isinstance(op, tuple):
            name, w, p = op
            rho = sum(_conjugate_columns_rows(rho, n, k, [w]) for k in port_kraus(name, p))
        else:
            rho = _conjugate_columns_rows(rho, n, port_gate_matrix(op), op.wires, op.controls)
    return rho


def port_density_expectation(n, rho, wires, basis):
    """circuit.hpp:264-281 restated: Paulis on every column, then the trace."""
    t = np.asarray(rho, complex).copy()
    pm = {"x": _KX, "y": _KY, "z": _KZ}
    for c in range(t.shape[1]):
        v = t[:, c]
        for w, b in zip(wires, basis):
            v = port_apply_matrix(v, n, pm[b], [w])
        t[:, c] = v
    return np.trace(t)


def port_density_marginal(n, rho, wires):
    """circuit.hpp:199-203 restated."""
    out = np.zeros(1 << len(wires))
    d = np.real(np.diag(rho))
    for idx in range(1 << n):
        o = 0
        for w in wires:
            o = (o << 1) | ((idx >> (n - 1 - w)) & 1)
        out[o] += d[idx]
    return out


# ------------------------------------- full size (threaded / digests) -----
def port_rng_normal(seed, label, count, offset=0, nthreads=0):
    """Rng(seed, label).normal() draws [offset, offset + count), counter-parallel
    on host threads (bit-identical to the sequential stream)."""
    import os

    L = port()
    out = np.empty(count, dtype=np.float64)
    rc = L.qo_rng_fill_normal(C.c_uint64(seed), None if label is None else label.encode(), C.c_uint64(offset),
                              C.c_uint64(count), _p(out), nthreads or os.cpu_count() or 1)
    if rc:  # the u1 == 0 rejection: replay sequentially
        seq = port_rng(seed, label, 2, offset + count)
        out[:] = seq[offset:]
    return out


def port_forward_mt(n, gates, psi, nthreads=0):
    """Circuit::forward (no data) of `psi` in place, threaded restatement."""
    import os

    L = port()
    arr, keep = gate_structs(gates)
    a = np.ascontiguousarray(psi, dtype=np.complex128)
    assert a.size == 1 << n
    rc = L.qo_forward_mt(n, arr, len(gates), _p(a), nthreads or os.cpu_count() or 1)
    if rc:
        raise OracleError(rc, "qo_forward_mt failed")
    return a


def port_digest(n, psi, nblocks=4096, nthreads=0):
    """(blocks[nblocks, 3], z[n + 2]) of a state (qo_digest)."""
    import os

    L = port()
    a = np.ascontiguousarray(psi, dtype=np.complex128)
    blocks = np.zeros((nblocks, 3))
    z = np.zeros(n + 2)
    rc = L.qo_digest(n, _p(a), nblocks, _p(blocks), _p(z), nthreads or os.cpu_count() or 1)
    if rc:
        raise OracleError(rc, "qo_digest failed")
    return blocks, z


def ref_forward_digest(n, gates, init_kind, seed, label, idx, nblocks=4096):
    """The reference's own apply_gate loop at full size, reduced to a digest:
    returns (blocks, z, samples at idx, seconds)."""
    L = ref()
    arr, keep = gate_structs(gates)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    blocks = np.zeros((nblocks, 3))
    z = np.zeros(n + 2)
    samples = np.zeros(len(idx), dtype=np.complex128)
    sec = C.c_double()
    rc = L.ref_forward_digest(n, arr, len(gates), init_kind, C.c_uint64(seed), None if label is None else label.encode(),
                              nblocks, _p(blocks), _p(z), len(idx), _p(idx), _p(samples), C.byref(sec))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return blocks, z, samples, sec.value


class RefState:
    """A reference QubitState kept across calls; apply() times
    quasar::qubit::apply_gate on it (bench.py --impl reference)."""

    def __init__(self, n, amps):
        L = ref()
        L.ref_state_new.restype = C.c_void_p
        L.ref_state_new.argtypes = [C.c_int, C.c_void_p]
        L.ref_state_free.argtypes = [C.c_void_p]
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        self.h = L.ref_state_new(n, _p(a))
        if not self.h:
            raise OracleError(1, L.ref_last_error().decode())

    def apply(self, gates) -> float:
        L = ref()
        arr, keep = gate_structs(gates)
        sec = C.c_double()
        rc = L.ref_state_apply_timed(C.c_void_p(self.h), arr, len(gates), C.byref(sec))
        if rc:
            raise OracleError(rc, L.ref_last_error().decode())
        return sec.value

    def close(self):
        if self.h:
            ref().ref_state_free(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_time_forward_z(n, gates, data=None, nthreads=1):
    """Circuit::forward + expectation() of every single-Z observable, timed in
    C++ (steady_clock); rows fanned over `nthreads` with quasar::parallel_for.
    Returns (seconds, z[rows, n])."""
    L = ref()
    arr, keep = gate_structs(gates)
    rows = 0 if data is None else len(data)
    d = None if data is None else np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(rows, -1))
    slots = 0 if d is None else d.shape[1]
    z = np.zeros((max(rows, 1), n))
    sec = C.c_double()
    rc = L.ref_time_forward_z(n, arr, len(gates), None if d is None else _p(d), rows, slots, nthreads, _p(z),
                              C.byref(sec))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return sec.value, z
