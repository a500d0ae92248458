"""qsv: a B200-native state-vector engine for DeepQuantum's qubit hot path.

The compute lives in libqsv.so (hand-written sm_100a CUDA behind the C ABI in
include/qsv.h); `qsv` mirrors the reference's quasar::qubit API over it.
"""
from .qsv import (  # noqa: F401
    C64, C128, Circuit, Context, Gate, GuardError, InvalidInput, Observable, Plan, QsvError, QubitState, Rng,
    TransportError, apply_gate, Channel, make_channel, apply_channel, bit_flip, phase_flip, depolarizing,
    amplitude_damping, phase_damping, approx_unitary, density_trace, default_context, expectation, expectation_many, expectation_one, gate_matrix, lib,
    make_gate, marginal_probabilities, measure, qft_circuit, rng_fill, set_default_context,
)
