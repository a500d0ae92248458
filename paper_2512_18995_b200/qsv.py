"""Python mirror of the reference's qubit API over the qsv C ABI.

Names, argument meaning and errors follow quasar::qubit
(/root/reference/proj/include/quasar/qubit/{gate,state,circuit}.hpp) so the
parity tests read like the reference's own tests:

  Gate, make_gate, gate_matrix        gate.hpp:28-38, 89-154, 193-207
  QubitState.basis / from_amplitudes  state.hpp:34-51
  apply_gate                          state.hpp:149-157 (value semantics)
  Circuit (builders, forward)         circuit.hpp:39-163
  qft_circuit                         circuit.hpp:167-178
  expectation_one / expectation       circuit.hpp:248-282
  marginal_probabilities / measure    circuit.hpp:182-244
  Rng                                 rng.hpp:29-103
  InvalidInput / GuardError / TransportError   core.hpp:34-47

Everything numeric runs in libqsv.so on the GPU; this module only marshals.
There is no CPU fallback: without the library or a CUDA device the calls
raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libqsv.so"

C64, C128 = 1, 2
OK, ERR_INTERNAL, ERR_INVALID, ERR_GUARD, ERR_TRANSPORT = 0, 1, 2, 3, 4
ZERO_OFF_CONTROL = 1
HINT_DIAGONAL = 2      # structure hints: checked against the matrix, no effect on the path
HINT_PERMUTATION = 4
kPi = 3.141592653589793238462643383279502884


class QsvError(RuntimeError):
    """CUDA / internal failure (status 1)."""


class InvalidInput(ValueError):
    """quasar::invalid_input (status 2)."""


class GuardError(RuntimeError):
    """quasar::guard_error (status 3)."""


class TransportError(RuntimeError):
    """quasar::transport_error (status 4)."""


_ERRORS = {ERR_INTERNAL: QsvError, ERR_INVALID: InvalidInput, ERR_GUARD: GuardError, ERR_TRANSPORT: TransportError}


class qsv_gate(C.Structure):
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


class qsv_obs(C.Structure):
    _fields_ = [("nwires", C.c_int32), ("wires", C.POINTER(C.c_int32)), ("basis", C.c_char_p)]


class qsv_opts(C.Structure):
    _fields_ = [("fuse", C.c_int32), ("tile_bits", C.c_int32), ("low_bits", C.c_int32), ("use_graph", C.c_int32),
                ("no_fuse_1q", C.c_int32), ("no_phase_flush", C.c_int32), ("jit", C.c_int32), ("reg_slots", C.c_int32),
                ("no_relabel", C.c_int32), ("from_zero", C.c_int32), ("super_bits", C.c_int32),
                ("dense_blocks", C.c_int32), ("lazy_layout", C.c_int32)]


class qsv_plan_info(C.Structure):
    _fields_ = [("ngates", C.c_int32), ("npasses", C.c_int32), ("nswaps", C.c_int32), ("max_tile_bits", C.c_int32),
                ("bytes_per_exec", C.c_double), ("comm_bytes_per_exec", C.c_double), ("ntile_passes", C.c_int32),
                ("nblocks", C.c_int32)]


# every symbol include/qsv.h declares, with its ctypes signature
_P = C.c_void_p
_SIGS = {
    "qsv_last_error": (C.c_char_p, []),
    "qsv_version": (C.c_int, []),
    "qsv_device_count": (C.c_int, []),
    "qsv_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "qsv_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "qsv_ctx_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(_P)]),
    "qsv_ctx_destroy": (C.c_int, [_P]),
    "qsv_ctx_create_multi": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_P)]),
    "qsv_ctx_rank_ctx": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "qsv_run_on_ranks": (C.c_int, [_P, C.c_void_p, C.c_void_p]),
    "qsv_ctx_comm_stats": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "qsv_ctx_comm_reset": (C.c_int, [_P]),
    "qsv_measure": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int, C.c_uint64, C.c_char_p,
                              C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p]),
    "qsv_run_rows_expect_z": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(qsv_gate), C.c_int, C.c_void_p, C.c_int,
                                        C.c_int, C.POINTER(qsv_opts), C.c_void_p]),
    "qsv_ctx_sync": (C.c_int, [_P]),
    "qsv_ctx_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "qsv_ctx_rank": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "qsv_state_create": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "qsv_state_destroy": (C.c_int, [_P]),
    "qsv_state_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "qsv_state_set_basis": (C.c_int, [_P, C.c_uint64]),
    "qsv_state_upload": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_download": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_upload_raw": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_download_raw": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_upload_raw_async": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_download_raw_async": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "qsv_state_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "qsv_state_device_ptr": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "qsv_state_peer_memory": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "qsv_gate_matrix": (C.c_int, [C.POINTER(qsv_gate), C.c_void_p, C.POINTER(C.c_int)]),
    "qsv_apply_matrix": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int32), C.c_void_p,
                                   C.c_int]),
    "qsv_apply_gate": (C.c_int, [_P, C.POINTER(qsv_gate)]),
    "qsv_run_circuit": (C.c_int, [_P, C.POINTER(qsv_gate), C.c_int, C.c_void_p, C.c_int, C.c_int,
                                  C.POINTER(qsv_opts)]),
    "qsv_plan_create": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(qsv_gate), C.c_int, C.POINTER(qsv_opts),
                                  C.POINTER(_P)]),
    "qsv_plan_destroy": (C.c_int, [_P]),
    "qsv_plan_info_get": (C.c_int, [_P, C.POINTER(qsv_plan_info)]),
    "qsv_plan_execute": (C.c_int, [_P, _P, C.c_void_p, C.c_int, C.c_int]),
    "qsv_plan_profile": (C.c_int, [_P, _P, C.c_void_p]),
    "qsv_norm2": (C.c_int, [_P, C.c_void_p]),
    "qsv_expect_z_all": (C.c_int, [_P, C.c_void_p]),
    "qsv_expect_pauli": (C.c_int, [_P, C.c_int, C.POINTER(qsv_obs), C.c_void_p]),
    "qsv_marginal_probs": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_void_p]),
    "qsv_plan_execute_expect_z": (C.c_int, [_P, _P, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "qsv_density_expect_pauli": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_void_p]),
    "qsv_density_marginal_probs": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_void_p]),
    "qsv_rng_fill": (C.c_int, [C.c_uint64, C.c_char_p, C.c_int, C.c_uint64, C.c_void_p, C.c_int]),
    "qsv_rng_fill_at": (C.c_int, [C.c_uint64, C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int]),
    "qsv_plan_steps": (C.c_int, [_P, C.c_void_p, C.c_int]),
    "qsv_adjoint_gradients": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(qsv_gate), C.c_int, C.c_int,
                                        C.POINTER(qsv_obs), C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                        C.POINTER(C.c_int), C.c_void_p]),
    "qsv_plan_dry": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(qsv_gate), C.c_int, C.POINTER(qsv_opts),
                               C.POINTER(qsv_plan_info), C.c_int, C.c_char_p, C.c_size_t]),
}


def plan_dry(nqubit: int, gates, dtype: int = C128, world: int = 1, opts: dict | None = None,
             source_of_pass: int = -1) -> tuple[dict, str]:
    """Host-only planning (no GPU): plan statistics and, optionally, the
    generated CUDA source of one pass."""
    arr, keep = gate_array(gates)
    o = make_opts(opts)
    info = qsv_plan_info()
    cap = 8 << 20 if source_of_pass >= 0 or source_of_pass <= -3 else 0
    buf = C.create_string_buffer(cap) if cap else None
    check(lib().qsv_plan_dry(nqubit, dtype, world, arr, len(gates), C.byref(o), C.byref(info), source_of_pass, buf,
                             cap))
    return {f: getattr(info, f) for f, _ in qsv_plan_info._fields_}, (buf.value.decode() if buf else "")


def plan_schedule(nqubit: int, gates, dtype: int = C128, world: int = 1, opts: dict | None = None) -> dict:
    """Host-only: the executable step list (local passes with their gates on
    physical bits, global<->local swap steps) the engine would run on `world`
    ranks. Used to verify the distributed schedule on CPU."""
    import json

    arr, keep = gate_array(gates)
    o = make_opts(opts)
    info = qsv_plan_info()
    cap = 64 << 20
    buf = C.create_string_buffer(cap)
    check(lib().qsv_plan_dry(nqubit, dtype, world, arr, len(gates), C.byref(o), C.byref(info), -2, buf, cap))
    return json.loads(buf.value.decode())

_lib = None


def lib():
    """Loads libqsv.so (built in-tree by paper_2512_18995_b200/build.py)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise QsvError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        if "QSV_NCCL_LIB" not in os.environ:
            try:
                import nvidia.nccl  # torch's bundled NCCL
                cand = Path(nvidia.nccl.__path__[0]) / "lib" / "libnccl.so.2"
                if cand.exists():
                    os.environ["QSV_NCCL_LIB"] = str(cand)
            except Exception:
                pass
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != OK:
        msg = lib().qsv_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, QsvError)(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- context ---
class Context:
    """Owns one GPU's stream (and, when distributed, its NCCL communicator).

    Context(device)                       one GPU
    Context(device, rank, world, uid)     one rank of a one-process-per-GPU job
    Context.multi(devices)                one process driving len(devices) ranks
                                          (ncclCommInitAll; every call runs on
                                          all ranks -- dist::run_on_ranks)"""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
                 _handle=None, _owned: bool = True):
        h = C.c_void_p()
        if _handle is not None:
            h = _handle
        elif world == 1:
            check(lib().qsv_ctx_create(device, C.byref(h)))
        else:
            buf = C.create_string_buffer(unique_id, 128)
            check(lib().qsv_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        self.h = h
        self._owned = _owned
        self.device, self.rank, self.world = device, rank, world
        self.multi_ranks = 0

    @staticmethod
    def multi(devices) -> "Context":
        devs = [int(d) for d in devices]
        arr = (C.c_int * max(1, len(devs)))(*devs)
        h = C.c_void_p()
        check(lib().qsv_ctx_create_multi(len(devs), arr, C.byref(h)))
        c = Context(devs[0] if devs else 0, 0, len(devs), _handle=h)
        c.multi_ranks = len(devs)
        return c

    def rank_context(self, rank: int) -> "Context":
        """Rank `rank`'s own context inside a multi-device one (not owned)."""
        h = C.c_void_p()
        check(lib().qsv_ctx_rank_ctx(self.h, int(rank), C.byref(h)))
        return Context(self.device, int(rank), self.world, _handle=h, _owned=False)

    def comm_stats(self) -> dict:
        """Transport counters (messages, bytes sent; all-reduces apart)."""
        m, b, a = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().qsv_ctx_comm_stats(self.h, C.byref(m), C.byref(b), C.byref(a)))
        return {"messages": m.value, "bytes": b.value, "allreduces": a.value}

    def reset_counters(self):
        check(lib().qsv_ctx_comm_reset(self.h))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().qsv_nccl_unique_id(buf))
        return buf.raw

    def sync(self):
        check(lib().qsv_ctx_sync(self.h))

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib().qsv_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def close(self):
        if self.h and self._owned:
            lib().qsv_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_RANK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p)


def run_on_ranks(ctx: Context, fn) -> None:
    """dist::run_on_ranks (tests/test_dist.cpp:66-94): fn(rank_ctx, rank) on one
    host thread per rank of a multi-device context, all joined; the first
    failing rank's exception is re-raised."""
    errors: dict = {}

    def tramp(h, rank, _user):
        try:
            fn(Context(ctx.device, rank, ctx.world, _handle=C.c_void_p(h), _owned=False), rank)
            return OK
        except BaseException as e:  # noqa: BLE001 -- carried to the caller
            errors[rank] = e
            return ERR_INTERNAL

    cb = _RANK_FN(tramp)
    rc = lib().qsv_run_on_ranks(ctx.h, C.cast(cb, C.c_void_p), None)
    if errors:
        raise errors[min(errors)]
    check(rc)


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def set_default_context(ctx: Context | None):
    global _default_ctx
    _default_ctx = ctx


# ------------------------------------------------------------------ gates ---
@dataclass
class Gate:
    name: str
    wires: list
    controls: list = field(default_factory=list)
    params: list = field(default_factory=list)
    trainable: bool = False
    encode: bool = False
    custom: np.ndarray | None = None

    def num_params(self) -> int:
        return len(self.params)


def make_gate(name, wires, controls=(), params=(), trainable=False, encode=False, custom=None) -> Gate:
    """gate.hpp:193-207 (wires and controls must be disjoint)."""
    g = Gate(str(name), [int(w) for w in wires], [int(c) for c in controls], [float(p) for p in params],
             bool(trainable), bool(encode), None if custom is None else np.asarray(custom, dtype=np.complex128))
    for w in g.wires:
        if w in g.controls:
            raise InvalidInput("gate wires and controls must be disjoint")
    return g


def _to_c_gate(g: Gate, keep: list) -> qsv_gate:
    c = qsv_gate()
    c.name = g.name.encode()[:15]
    if len(g.wires) > 2:
        raise InvalidInput(f"gate {g.name}: 1 or 2 target wires supported")
    if len(g.controls) > 6:
        raise InvalidInput(f"gate {g.name}: at most 6 controls")
    if len(g.params) > 3:
        raise InvalidInput(f"gate {g.name}: at most 3 params")
    c.nwires = len(g.wires)
    for i, w in enumerate(g.wires):
        c.wires[i] = w
    c.ncontrols = len(g.controls)
    for i, w in enumerate(g.controls):
        c.controls[i] = w
    c.nparams = len(g.params)
    for i, p in enumerate(g.params):
        c.params[i] = p
    c.trainable = int(g.trainable)
    c.encode = int(g.encode)
    if g.custom is not None:
        m = np.ascontiguousarray(np.asarray(g.custom, dtype=np.complex128)).view(np.float64).ravel().copy()
        keep.append(m)
        c.custom = m.ctypes.data_as(C.POINTER(C.c_double))
    return c


def gate_array(gates: Sequence[Gate]):
    keep: list = []
    arr = (qsv_gate * max(1, len(gates)))()
    for i, g in enumerate(gates):
        arr[i] = _to_c_gate(g, keep)
    return arr, keep


def gate_matrix(g: Gate) -> np.ndarray:
    keep: list = []
    cg = _to_c_gate(g, keep)
    out = np.zeros(32, dtype=np.float64)
    k = C.c_int()
    check(lib().qsv_gate_matrix(C.byref(cg), _ptr(out), C.byref(k)))
    d = 1 << k.value
    return out[: 2 * d * d].view(np.complex128).reshape(d, d)


# ------------------------------------------------------------------ state ---
class QubitState:
    """Device-resident batch of pure states (state.hpp:29-91)."""

    def __init__(self, nqubit: int, batch: int = 1, dtype: int = C128, ctx: Context | None = None, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self.h = _handle
        else:
            h = C.c_void_p()
            check(lib().qsv_state_create(self.ctx.h, int(nqubit), int(batch), int(dtype), C.byref(h)))
            self.h = h
        n, b, d, g, la = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
        check(lib().qsv_state_info(self.h, C.byref(n), C.byref(b), C.byref(d), C.byref(g), C.byref(la)))
        self._n, self._batch, self.dtype, self.global_bits, self.local_amps = n.value, b.value, d.value, g.value, la.value
        self._mixed = None  # m when this engine state holds vec(rho) of m-qubit density matrices

    # reference constructors
    @staticmethod
    def basis(nqubit: int, index: int = 0, batch: int = 1, dtype: int = C128, ctx: Context | None = None):
        s = QubitState(nqubit, batch, dtype, ctx)
        if index:
            check(lib().qsv_state_set_basis(s.h, int(index)))
        return s

    @staticmethod
    def from_amplitudes(nqubit: int, amps, dtype: int = C128, ctx: Context | None = None, batch: int = 1,
                        check_norm: bool = True):
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        if a.size != (1 << nqubit) >> 0 and (ctx is None or ctx.world == 1):
            raise InvalidInput("QubitState: amplitude length mismatch")
        if check_norm and abs(float(np.vdot(a, a).real) - 1.0) >= 1e-10:
            raise InvalidInput("QubitState: not normalized")
        s = QubitState(nqubit, batch, dtype, ctx)
        for b in range(batch):
            s.upload(a, b)
        return s

    def nqubit(self) -> int:
        return self._mixed if self._mixed is not None else self._n

    def is_mixed(self) -> bool:
        return self._mixed is not None

    # ---- mixed states (state.hpp:53-62, 73-80; channel.hpp) ----
    @staticmethod
    def from_density(nqubit: int, rho, dtype: int = C128, ctx: Context | None = None) -> "QubitState":
        """state.hpp:53-62: shape, Hermitian within 1e-9, unit trace within 1e-10."""
        r = np.ascontiguousarray(rho, dtype=np.complex128)
        dim = 1 << nqubit
        if r.shape != (dim, dim):
            raise InvalidInput("QubitState: density shape mismatch")
        if np.max(np.abs(r - r.conj().T)) >= 1e-9:
            raise InvalidInput("QubitState: rho not Hermitian")
        if abs(np.trace(r).real - 1.0) >= 1e-10:
            raise InvalidInput("QubitState: trace != 1")
        s = QubitState(2 * nqubit, dtype=dtype, ctx=ctx)
        s.upload(r.reshape(-1))
        s._mixed = nqubit
        return s

    def to_mixed(self) -> "QubitState":
        """state.hpp:73-80: rows become |psi><psi| (vec(rho) on 2m engine
        qubits, built on the host: O(4^m) host memory)."""
        if self._mixed is not None:
            return self.clone()
        m = self._n
        if 2 * m > 34:
            raise InvalidInput("to_mixed: 2n engine qubits exceed one GPU")
        s = QubitState(2 * m, batch=self._batch, dtype=self.dtype, ctx=self.ctx)
        for b in range(self._batch):
            a = self.amplitudes(b)
            s.upload(np.outer(a, a.conj()).reshape(-1), b)
        s._mixed = m
        return s

    def density(self, b: int = 0) -> np.ndarray:
        if self._mixed is None:
            raise InvalidInput("QubitState: not a mixed state")
        out = np.empty(self.local_amps, dtype=np.complex128)
        check(lib().qsv_state_download(self.h, b, _ptr(out.view(np.float64)), self.local_amps))
        d = 1 << self._mixed
        return out.reshape(d, d)

    def batch(self) -> int:
        return self._batch

    def upload(self, amps, row: int = 0):
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        check(lib().qsv_state_upload(self.h, row, _ptr(a.view(np.float64)), a.size))

    def amplitudes(self, b: int = 0) -> np.ndarray:
        if self._mixed is not None:
            raise InvalidInput("QubitState: mixed state has no amplitudes (use density)")
        out = np.empty(self.local_amps, dtype=np.complex128)
        check(lib().qsv_state_download(self.h, b, _ptr(out.view(np.float64)), self.local_amps))
        return out

    def clone(self) -> "QubitState":
        h = C.c_void_p()
        check(lib().qsv_state_clone(self.h, C.byref(h)))
        out = QubitState(self._n, ctx=self.ctx, _handle=h)
        out._mixed = self._mixed
        return out

    def peer_memory(self) -> int:
        """Multi-GPU: 1 = qubit swaps fused into the passes (peer memory),
        -1 = NCCL swaps, 0 = not decided yet."""
        v = C.c_int(0)
        check(lib().qsv_state_peer_memory(self.h, C.byref(v)))
        return v.value

    def norm2(self) -> np.ndarray:
        out = np.zeros(self._batch)
        check(lib().qsv_norm2(self.h, _ptr(out)))
        return out

    def expect_z_all(self) -> np.ndarray:
        out = np.zeros(self._batch * self._n)
        check(lib().qsv_expect_z_all(self.h, _ptr(out)))
        return out.reshape(self._batch, self._n)

    def apply_matrix(self, m, wires, controls=(), zero_off_control=False, hints=0):
        """detail::apply_matrix_strided (state.hpp:111-143), in place. `hints`:
        HINT_DIAGONAL / HINT_PERMUTATION (verified against the matrix)."""
        m = np.ascontiguousarray(m, dtype=np.complex128)
        k = len(wires)
        if m.shape != (1 << k, 1 << k):
            raise InvalidInput("gate matrix shape mismatch")
        w = (C.c_int32 * max(1, k))(*wires)
        c = (C.c_int32 * max(1, len(controls)))(*controls)
        check(lib().qsv_apply_matrix(self.h, k, w, len(controls), c, _ptr(m.view(np.float64)),
                                     (ZERO_OFF_CONTROL if zero_off_control else 0) | hints))

    def close(self):
        if getattr(self, "h", None):
            lib().qsv_state_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def approx_unitary(u, tol: float = 1e-8) -> bool:
    """core.hpp:53-57."""
    u = np.asarray(u, dtype=np.complex128)
    if u.ndim != 2 or u.shape[0] != u.shape[1]:
        return False
    return float(np.max(np.abs(u.conj().T @ u - np.eye(u.shape[0])))) < tol


# --------------------------------------------------------------- channels ---
@dataclass
class Channel:
    """channel.hpp:22-27: a single-qubit channel as a Kraus set."""
    name: str
    wire: int
    kraus: list


def make_channel(name: str, wire: int, kraus) -> Channel:
    """channel.hpp:29-38: 2x2 Kraus operators, sum K^dagger K = I within 1e-10."""
    ks = [np.asarray(k, dtype=np.complex128) for k in kraus]
    acc = np.zeros((2, 2), dtype=np.complex128)
    for k in ks:
        if k.shape != (2, 2):
            raise InvalidInput("channel: Kraus operators must be 2x2")
        acc += k.conj().T @ k
    if np.max(np.abs(acc - np.eye(2))) >= 1e-10:
        raise InvalidInput("channel: Kraus set not trace preserving")
    return Channel(str(name), int(wire), ks)


_PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_PY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_PZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
_I2 = np.eye(2, dtype=np.complex128)


def bit_flip(wire: int, p: float) -> Channel:  # channel.hpp:40-43
    return make_channel("bit_flip", wire, [math.sqrt(1 - p) * _I2, math.sqrt(p) * _PX])


def phase_flip(wire: int, p: float) -> Channel:  # channel.hpp:45-48
    return make_channel("phase_flip", wire, [math.sqrt(1 - p) * _I2, math.sqrt(p) * _PZ])


def depolarizing(wire: int, p: float) -> Channel:  # channel.hpp:50-55
    return make_channel("depolarizing", wire, [math.sqrt(1 - 3.0 * p / 4.0) * _I2, math.sqrt(p / 4.0) * _PX,
                                               math.sqrt(p / 4.0) * _PY, math.sqrt(p / 4.0) * _PZ])


def amplitude_damping(wire: int, gamma: float) -> Channel:  # channel.hpp:57-62
    return make_channel("amplitude_damping", wire, [np.array([[1, 0], [0, math.sqrt(1 - gamma)]]),
                                                    np.array([[0, math.sqrt(gamma)], [0, 0]])])


def phase_damping(wire: int, lam: float) -> Channel:  # channel.hpp:64-69
    return make_channel("phase_damping", wire, [np.array([[1, 0], [0, math.sqrt(1 - lam)]]),
                                                np.array([[0, 0], [0, math.sqrt(lam)]])])


def density_trace(state: QubitState) -> np.ndarray:
    """Tr rho per batch row (the identity observable on the device)."""
    arr = (qsv_obs * 1)()
    arr[0].nwires = 0
    arr[0].wires = None
    arr[0].basis = b""
    out = np.zeros(state.batch())
    check(lib().qsv_density_expect_pauli(state.h, 1, arr, _ptr(out)))
    return out


def apply_channel(state: QubitState, ch: Channel) -> QubitState:
    """channel.hpp:73-100: rho' = sum_i K_i rho K_i^dagger, pure states
    promoted first. On the device this is ONE pass: the 4x4 superoperator
    sum_i K_i (x) conj(K_i) on the (row, column) wire pair of vec(rho)."""
    out = state.to_mixed()
    m = out.nqubit()
    if not 0 <= ch.wire < m:
        raise InvalidInput("target wire out of range")
    sop = sum(np.kron(k, k.conj()) for k in ch.kraus)
    out.apply_matrix(sop, [ch.wire, ch.wire + m])
    tr = density_trace(out)
    # channel.hpp:96 checks 1e-10 in double; a complex64 state carries ~1e-7
    if np.any(np.abs(tr - 1.0) >= (1e-10 if out.dtype == C128 else 1e-5)):
        raise InvalidInput("channel: trace not preserved")
    return out


def _conj_gate(g: Gate, m: int) -> Gate:
    """conj(U) of gate g acting on the column wires m + w of vec(rho)."""
    return Gate("custom", [w + m for w in g.wires], [c + m for c in g.controls], [], False, False,
                np.conj(gate_matrix(g)))


def _mixed_gates(gates, m: int) -> list:
    """The 2m-qubit circuit of U rho U^dagger (state.hpp:159-172): each gate on
    the row wires, then its conjugate on the column wires."""
    out = []
    for g in gates:
        if g.encode:
            raise InvalidInput("encoded batch runs expect a pure initial state")  # circuit.hpp:131
        out += [g, _conj_gate(g, m)]
    return out


def apply_gate(state: QubitState, g: Gate) -> QubitState:
    """Value semantics like state.hpp:149-157: returns a new state. A mixed
    state gets U on its row wires and conj(U) on its column wires."""
    if state.is_mixed():
        m = state.nqubit()
        if not approx_unitary(gate_matrix(g), 1e-10):
            raise InvalidInput(f"gate {g.name}: matrix not unitary")
        out = state.clone()
        for h in (g, _conj_gate(g, m)):
            keep: list = []
            cg = _to_c_gate(h, keep)
            check(lib().qsv_apply_gate(out.h, C.byref(cg)))
        return out
    out = state.clone()
    keep: list = []
    cg = _to_c_gate(g, keep)
    check(lib().qsv_apply_gate(out.h, C.byref(cg)))
    return out


# ---------------------------------------------------------------- circuit ---
@dataclass
class Observable:
    wires: list
    basis: str


class Circuit:
    """quasar::qubit::Circuit (circuit.hpp:39-163) executing on the GPU."""

    def __init__(self, nqubit: int):
        if not (1 <= nqubit <= 40):
            raise InvalidInput("Circuit: nqubit out of range")
        self._n = nqubit
        self._gates: list[Gate] = []
        self._obs: list[Observable] = []

    def nqubit(self):
        return self._n

    def gates(self):
        return self._gates

    def observables(self):
        return self._obs

    def add(self, g: Gate):
        for w in g.wires:
            if not (0 <= w < self._n):
                raise InvalidInput("gate wire out of range")
        for c in g.controls:
            if not (0 <= c < self._n):
                raise InvalidInput("control wire out of range")
        self._gates.append(g)

    def h(self, w): self.add(make_gate("h", [w]))
    def x(self, w, controls=()): self.add(make_gate("x", [w], controls))
    def y(self, w): self.add(make_gate("y", [w]))
    def z(self, w): self.add(make_gate("z", [w]))
    def cnot(self, c, t): self.add(make_gate("x", [t], [c]))
    def cz(self, c, t): self.add(make_gate("z", [t], [c]))
    def cp(self, c, t, theta): self.add(make_gate("p", [t], [c], [theta]))
    def swap(self, a, b): self.add(make_gate("swap", [a, b]))
    def rx(self, w, theta, trainable=False, encode=False): self.add(make_gate("rx", [w], [], [theta], trainable, encode))
    def ry(self, w, theta, trainable=False, encode=False): self.add(make_gate("ry", [w], [], [theta], trainable, encode))
    def rz(self, w, theta, trainable=False, encode=False): self.add(make_gate("rz", [w], [], [theta], trainable, encode))
    def cry(self, c, t, theta, trainable=False): self.add(make_gate("ry", [t], [c], [theta], trainable))
    def rxx(self, a, b, theta, trainable=False): self.add(make_gate("rxx", [a, b], [], [theta], trainable))
    def ryy(self, a, b, theta, trainable=False): self.add(make_gate("ryy", [a, b], [], [theta], trainable))
    def rzz(self, a, b, theta, trainable=False): self.add(make_gate("rzz", [a, b], [], [theta], trainable))

    def rylayer(self, encode=False, init=()):
        for w in range(self._n):
            self.ry(w, init[w] if len(init) else 0.0, not encode, encode)

    def cnot_ring(self):
        for w in range(self._n):
            self.cnot(w, (w + 1) % self._n)

    def observable(self, wires, basis: str):
        if len(wires) != len(basis):
            raise InvalidInput("observable: one basis letter per wire")
        for ch in basis:
            if ch not in "xyz":
                raise InvalidInput("observable: basis letter outside {x,y,z}")
        self._obs.append(Observable(list(wires), basis))

    def encode_slots(self) -> int:
        return sum(g.num_params() for g in self._gates if g.encode)

    def forward(self, init: QubitState | None = None, data=None, dtype: int = C128, opts: dict | None = None,
                ctx: Context | None = None) -> QubitState:
        """Circuit::forward (circuit.hpp:121-157): fused on the GPU."""
        slots = self.encode_slots()
        data = [] if data is None else data
        arr, keep = gate_array(self._gates)
        o = make_opts(opts)
        if init is None and "from_zero" not in (opts or {}):
            o.from_zero = 1  # starts from |0...0>: leading 1q gates become a synthesised product state
        if len(data) == 0:
            if slots != 0:
                raise InvalidInput("circuit has encode slots but no data given")
            s = init.clone() if init is not None else QubitState.basis(self._n, dtype=dtype, ctx=ctx)
            if s.is_mixed():  # the same fused passes on the 2m-qubit vec(rho)
                arr, keep = gate_array(_mixed_gates(self._gates, self._n))
                check(lib().qsv_run_circuit(s.h, arr, 2 * len(self._gates), None, 0, 0, C.byref(o)))
                return s
            check(lib().qsv_run_circuit(s.h, arr, len(self._gates), None, 0, 0, C.byref(o)))
            return s
        rows = [list(map(float, r)) for r in data]
        for r in rows:
            if len(r) != slots:
                raise InvalidInput(f"data length {len(r)} != encode slots {slots}")
        if init is not None and init.is_mixed():
            raise InvalidInput("encoded batch runs expect a pure initial state")  # circuit.hpp:131
        if init is not None and init.batch() != 1:
            raise InvalidInput("encoded runs broadcast a single initial state")
        dt = init.dtype if init is not None else dtype
        s = QubitState(self._n, batch=len(rows), dtype=dt, ctx=ctx or (init.ctx if init else None))
        if init is not None:
            a0 = init.amplitudes(0)
            for b in range(len(rows)):
                s.upload(a0, b)
        d = np.ascontiguousarray(np.asarray(rows, dtype=np.float64).reshape(len(rows), max(slots, 0)))
        check(lib().qsv_run_circuit(s.h, arr, len(self._gates), _ptr(d) if d.size else None, len(rows), slots,
                                    C.byref(o)))
        return s


def make_opts(opts: dict | None) -> qsv_opts:
    o = qsv_opts()
    o.fuse = 1
    for k, v in (opts or {}).items():
        setattr(o, k, int(v))
    return o


def run_rows_expect_z(cir: "Circuit", data, dtype: int = C64, ctx: Context | None = None,
                      opts: dict | None = None) -> np.ndarray:
    """Batched small circuits as independent units (cfg2): every data row a
    from-|0...0> forward of `cir`, then all <Z_w> -- rows x n. On a
    multi-device context the rows split over the devices with no
    communication (qsv_run_rows_expect_z)."""
    ctx = ctx or default_context()
    d = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    rows = d.shape[0]
    slots = d.shape[1] if d.ndim == 2 else 0
    arr, keep = gate_array(cir.gates())
    o = make_opts(opts)
    out = np.zeros(rows * cir.nqubit())
    check(lib().qsv_run_rows_expect_z(ctx.h, cir.nqubit(), dtype, arr, len(cir.gates()), _ptr(d) if slots else None,
                                      rows, slots, C.byref(o), _ptr(out)))
    return out.reshape(rows, cir.nqubit())


class Plan:
    """A planned circuit: planning hoisted out of the timed loop."""

    def __init__(self, nqubit: int, gates: Sequence[Gate], dtype: int = C128, opts: dict | None = None,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        arr, keep = gate_array(gates)
        o = make_opts(opts)
        h = C.c_void_p()
        check(lib().qsv_plan_create(self.ctx.h, nqubit, dtype, arr, len(gates), C.byref(o), C.byref(h)))
        self.h = h
        info = qsv_plan_info()
        check(lib().qsv_plan_info_get(self.h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in qsv_plan_info._fields_}

    def execute(self, state: QubitState, data=None):
        if data is None:
            check(lib().qsv_plan_execute(self.h, state.h, None, 0, 0))
        else:
            d = np.ascontiguousarray(data, dtype=np.float64)
            check(lib().qsv_plan_execute(self.h, state.h, _ptr(d), d.shape[0], d.shape[1]))

    def execute_expect_z(self, state: QubitState, data=None) -> np.ndarray:
        """forward + every <Z_w>: batch x n (qsv_plan_execute_expect_z)."""
        out = np.zeros(state.batch() * state.nqubit())
        if data is None:
            check(lib().qsv_plan_execute_expect_z(self.h, state.h, None, 0, 0, _ptr(out)))
        else:
            d = np.ascontiguousarray(data, dtype=np.float64)
            check(lib().qsv_plan_execute_expect_z(self.h, state.h, _ptr(d), d.shape[0], d.shape[1], _ptr(out)))
        return out.reshape(state.batch(), state.nqubit())

    def step_kinds(self) -> np.ndarray:
        """0 = local pass, 1 = global<->local qubit swap, in execution order."""
        n = lib().qsv_plan_steps(self.h, None, 0)
        k = np.zeros(max(1, n), dtype=np.int32)
        lib().qsv_plan_steps(self.h, _ptr(k), n)
        return k[:n]

    def profile(self, state: QubitState) -> np.ndarray:
        """One execution with CUDA events around every step; per-step ms."""
        n = lib().qsv_plan_steps(self.h, None, 0)
        out = np.zeros(max(1, n))
        check(lib().qsv_plan_profile(self.h, state.h, _ptr(out)))
        return out[:n]

    def close(self):
        if getattr(self, "h", None):
            lib().qsv_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def qft_circuit(nqubit: int) -> Circuit:
    """circuit.hpp:167-178 (no final swaps)."""
    cir = Circuit(nqubit)
    for n in range(nqubit):
        cir.h(n)
        k = 2
        for i in range(n, nqubit - 1):
            cir.cp(i + 1, n, kPi / math.pow(2.0, k - 1))
            k += 1
    return cir


# ------------------------------------------------------------ reductions ---
def expectation_one(state: QubitState, obs: Observable, batch_index: int = 0) -> float:
    return expectation_many(state, [obs])[batch_index][0]


def expectation_many(state: QubitState, obs: Sequence[Observable]) -> np.ndarray:
    arr = (qsv_obs * max(1, len(obs)))()
    keep = []
    for i, o in enumerate(obs):
        w = (C.c_int32 * max(1, len(o.wires)))(*o.wires)
        b = o.basis.encode()
        keep += [w, b]
        arr[i].nwires = len(o.wires)
        arr[i].wires = C.cast(w, C.POINTER(C.c_int32))
        arr[i].basis = b
    out = np.zeros(state.batch() * max(1, len(obs)))
    fn = lib().qsv_density_expect_pauli if state.is_mixed() else lib().qsv_expect_pauli
    check(fn(state.h, len(obs), arr, _ptr(out)))
    return out.reshape(state.batch(), max(1, len(obs)))[:, : len(obs)]


def expectation(state: QubitState, cir: Circuit, batch_index: int = 0) -> list:
    if not cir.observables():
        return []
    return list(expectation_many(state, cir.observables())[batch_index])


def marginal_probabilities(state: QubitState, wires, batch_index: int = 0) -> np.ndarray:
    if len(wires) == 0:
        raise InvalidInput("measure: empty wire list")
    k = len(wires)
    w = (C.c_int32 * k)(*wires)
    out = np.zeros(1 << k)
    if state.is_mixed():
        check(lib().qsv_density_marginal_probs(state.h, batch_index, k, w, _ptr(out)))
        return out
    check(lib().qsv_marginal_probs(state.h, batch_index, k, w, _ptr(out)))
    return out


@dataclass
class AdjointGradients:
    """adjoint.hpp:25-28."""
    param_grads: list
    data_grads: list


def adjoint_gradients(cir: Circuit, init: "QubitState | None" = None, data=(), dtype: int = C128,
                      ctx: Context | None = None) -> AdjointGradients:
    """quasar::qubit::adjoint_gradients (adjoint.hpp:52-110) on the GPU:
    gradient of the summed expectation of the circuit's observables."""
    ctx = ctx or default_context()
    arr, keep = gate_array(cir.gates())
    obs = cir.observables()
    oarr = (qsv_obs * max(1, len(obs)))()
    for i, o in enumerate(obs):
        w = (C.c_int32 * max(1, len(o.wires)))(*o.wires)
        b = o.basis.encode()
        keep += [w, b]
        oarr[i].nwires = len(o.wires)
        oarr[i].wires = C.cast(w, C.POINTER(C.c_int32))
        oarr[i].basis = b
    d = np.ascontiguousarray(np.asarray(list(data), dtype=np.float64))
    ini = None
    if init is not None:
        if init.is_mixed():
            raise InvalidInput("adjoint_gradients: pure states only")  # adjoint.hpp:54
        if init.batch() != 1:
            raise InvalidInput("adjoint_gradients: one batch row at a time")
        ini = np.ascontiguousarray(init.amplitudes(0)).view(np.float64)
    cap = sum(g.num_params() for g in cir.gates())
    pg = np.zeros(max(1, cap))
    dg = np.zeros(max(1, len(d)))
    npar = C.c_int()
    check(lib().qsv_adjoint_gradients(ctx.h, cir.nqubit(), dtype, arr, len(cir.gates()), len(obs), oarr,
                                      _ptr(ini) if ini is not None else None, _ptr(d) if d.size else None, len(d),
                                      _ptr(pg), cap, C.byref(npar), _ptr(dg)))
    return AdjointGradients(list(pg[: npar.value]), list(dg[: len(d)]))


def bits_to_string(outcome: int, k: int) -> str:
    return "".join("1" if (outcome >> (k - 1 - i)) & 1 else "0" for i in range(k))


def measure_counts(state: QubitState, shots: int, wires, rng: "Rng", batch_index: int = 0):
    """qsv_measure as arrays: (counts[2^k] uint64, probs[2^k]) -- the
    marginals on the device, the reference's seeded sampling in the library
    (identical histograms), continuing this Rng's stream. Pure states,
    1 <= k <= 26 wires."""
    if shots < 1:
        raise InvalidInput("measure: shots must be >= 1")
    k = len(wires)
    w = (C.c_int32 * max(1, k))(*wires)
    counts = np.zeros(1 << k, dtype=np.uint64)
    probs = np.zeros(1 << k)
    ctr = C.c_uint64(rng.counter)
    check(lib().qsv_measure(state.h, batch_index, k, w, int(shots), C.c_uint64(rng.seed0),
                            None if rng.label is None else rng.label.encode(), C.byref(ctr), _ptr(counts),
                            _ptr(probs)))
    rng.counter = ctr.value
    return counts, probs


def measure(state: QubitState, shots: int, wires, rng: "Rng", with_prob: bool = False, batch_index: int = 0):
    """circuit.hpp:217-244: CDF sampling over the device-computed marginals."""
    if shots < 1:
        raise InvalidInput("measure: shots must be >= 1")
    k = len(wires)
    if not state.is_mixed() and 1 <= k <= 26:
        counts, probs = measure_counts(state, shots, wires, rng, batch_index)
        out: dict = {}
        for i in np.nonzero(counts)[0]:
            out[bits_to_string(int(i), k)] = {"count": int(counts[i]), "probability": 0.0}
        if with_prob:
            for i, p in enumerate(probs):
                key = bits_to_string(i, k)
                if p <= 0 and key not in out:
                    continue
                out.setdefault(key, {"count": 0, "probability": 0.0})["probability"] = float(p)
        return dict(sorted(out.items()))
    probs = marginal_probabilities(state, wires, batch_index)
    cdf = np.cumsum(probs)
    # the reference accumulates sequentially; np.cumsum is sequential too
    acc = float(cdf[-1])
    out: dict = {}
    u = np.array([rng.uniform() for _ in range(shots)]) * acc
    idx = np.minimum(np.searchsorted(cdf, u, side="left"), len(probs) - 1)
    for i in idx:
        key = bits_to_string(int(i), k)
        out.setdefault(key, {"count": 0, "probability": 0.0})["count"] += 1
    if with_prob:
        for i, p in enumerate(probs):
            key = bits_to_string(i, k)
            if p <= 0 and key not in out:
                continue
            out.setdefault(key, {"count": 0, "probability": 0.0})["probability"] = float(p)
    return dict(sorted(out.items()))


# -------------------------------------------------------------------- Rng ---
_M64 = (1 << 64) - 1


def _mix(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & _M64
    return h


class Rng:
    """quasar::Rng (rng.hpp:29-103), sequential draws for circuit generation."""

    def __init__(self, seed: int = 0, stream: str | None = None):
        seed &= _M64
        self.seed0, self.label = seed, stream
        if stream is not None:
            seed ^= _fnv1a(stream)
        self.seed_eff = seed
        self.key = _mix(seed ^ 0x9E3779B97F4A7C15)
        self.counter = 0
        self.spare = 0.0
        self.have_spare = False

    def next_u64(self) -> int:
        self.counter += 1
        return _mix((self.key + 0x9E3779B97F4A7C15 * self.counter) & _M64)

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def normal(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        u1 = 0.0
        while u1 == 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        self.spare = r * math.sin(2.0 * 3.141592653589793 * u2)
        self.have_spare = True
        return r * math.cos(2.0 * 3.141592653589793 * u2)

    def next_below(self, n: int) -> int:
        return self.next_u64() % n if n else 0


def rng_fill(seed: int, label: str | None, kind: str, count: int, nthreads: int = 0, offset: int = 0) -> np.ndarray:
    """Bulk stream Rng(seed, label) draws through the library (multi-threaded,
    bit-identical to the sequential stream), starting `offset` draws in.
    kind: 'u64' | 'uniform' | 'normal'."""
    k = {"u64": 0, "uniform": 1, "normal": 2}[kind]
    out = np.empty(count, dtype=np.uint64 if k == 0 else np.float64)
    check(lib().qsv_rng_fill_at(seed, label.encode() if label is not None else None, k, offset, count, _ptr(out),
                                nthreads))
    return out
