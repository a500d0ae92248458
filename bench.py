"""Benchmark: BASELINE.json metric "gate passes/sec and achieved HBM GB/s per
pass at n qubits" on config 3 -- the 30-qubit complex128 QFT (+ final swaps)
on the seeded, normalised Gaussian input state, one B200 (16 GiB state).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Arms
  default      the engine (libqsv.so, fused sm_100a tile passes) through the C
               ABI. A step = one full execution of the 480-gate circuit on the
               HBM-resident state. value = source gates applied per second
               (one "gate pass" = one reference gate applied to all 2^30
               amplitudes). Under torchrun (N > 1) the state is sharded over N
               GPUs (top log2 N qubits global, NCCL qubit swaps): strong scaling.
  reference    the reference's own CPU path (oracle/_ref: the unmodified
               quasar headers, quasar::qubit::apply_gate) on this host, a
               bounded sample of the same workload: each step applies one
               gate of the same circuit to the same 30-qubit state.

Timing: W warm-up steps, then K steps bracketed by barrier +
cudaStreamSynchronize, CUDA events on the engine's own stream, max over
ranks; the state (16 GiB) is far larger than L2 (126 MB), so no flush is
needed. Per-launch CUDA events inside the timed region give the dominant
kernel's average duration for the roofline.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_QUBITS = 30
METRIC = "gate passes/sec at n qubits (source gates applied to the full state per second)"
WORKLOAD = "cfg3: 30-qubit complex128 QFT + 15 final swaps on a seeded normalised Gaussian state"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # diagnostics only: every rank on device 0 (the multi-rank path through
    # tests/fake_nccl on a one-GPU box); never set for a measurement
    if os.environ.get("QSV_BENCH_SHARE_GPU") == "1":
        local = 0
    return rank, world, local


NOMINAL_HBM_GBS = 8000.0  # north_star's "~8 TB/s"


def config_dict(n):
    """The workload; identical in both arms (engine details go under "plan")."""
    return {"workload": WORKLOAD, "n_qubits": n, "gates": 480 if n == 30 else None, "dtype": "c128",
            "input": "seeded normalised Gaussian state Rng(0,'cfg3')",
            "l2": "state (16 GiB) >> L2 (126 MB); no flush needed"}


def cfg3_gate_list(n):
    """The cfg3 circuit built from the reference's own qft_circuit
    (circuit.hpp:167-178, through oracle/_ref) plus the 15 final swaps --
    no libqsv involved (the reference arm must not map it)."""
    from oracle import oracle as O

    gl = list(O.ref_qft_gates(n))
    for i in range(n // 2):
        g = O.RefGate()
        g.name = b"swap"
        g.nwires = 2
        g.wires[0], g.wires[1] = i, n - 1 - i
        gl.append(g)
    return gl


class _G:  # RefGate -> the attribute view oracle.gate_struct expects
    def __init__(self, r):
        self.name = r.name.decode()
        self.wires = [r.wires[i] for i in range(r.nwires)]
        self.controls = [r.controls[i] for i in range(r.ncontrols)]
        self.params = [r.params[i] for i in range(r.nparams)]
        self.trainable = bool(r.trainable)
        self.encode = bool(r.encode)
        self.custom = None


def stratified_sample(gl, k):
    """k gates of the circuit with its gate kinds in proportion (h / cp /
    swap = 30 / 435 / 15 of 480), evenly spread through the circuit within
    each kind, in circuit order."""
    kinds = {}
    for i, g in enumerate(gl):
        kinds.setdefault(g.name, []).append(i)
    total = len(gl)
    quota = {nm: max(1, round(k * len(ix) / total)) for nm, ix in kinds.items()}
    big = max(quota, key=lambda nm: len(kinds[nm]))
    quota[big] = max(1, k - sum(q for nm, q in quota.items() if nm != big))
    pick = []
    for nm, ix in kinds.items():
        q = quota[nm]
        pick += [ix[int((j + 0.5) * len(ix) / q)] for j in range(q)]
    return [gl[i] for i in sorted(pick)][:k] if len(pick) >= k else [gl[i] for i in sorted(pick)]


def reference_cpu_sample(n, nsteps, warmup):
    """The reference's CPU path on a bounded sample of cfg3 at full size:
    quasar::qubit::apply_gate (state.hpp:149-157; gate_matrix, unitarity
    check, full copy, strided sweep) on a reference QubitState holding the
    seeded 30-qubit input, one gate per step, `warmup` + `nsteps` gates drawn
    by stratified_sample. The input comes from the oracle's threaded Rng
    restatement (bit-identical to Rng(0,'cfg3')). Returns (per-step seconds,
    sample description)."""
    import gc

    from oracle import oracle as O

    psi = O.port_rng_normal(0, "cfg3", 2 << n).view(np.complex128)
    psi /= np.sqrt(float(np.dot(psi.view(np.float64), psi.view(np.float64))))
    st = O.RefState(n, psi)
    del psi
    gc.collect()
    gl = [_G(r) for r in cfg3_gate_list(n)]
    sample = stratified_sample(gl, warmup + nsteps)
    times = [st.apply([g]) for g in sample]
    st.close()
    mix = {}
    for g in sample[warmup:]:
        mix[g.name] = mix.get(g.name, 0) + 1
    desc = (f"{nsteps} gates of cfg3 at n={n} (kinds {mix}, spread through the circuit in proportion) after "
            f"{warmup} warm-up gates, one per step, via quasar::qubit::apply_gate on a reference QubitState "
            "(single-threaded: the reference qubit path never calls parallel_for)")
    return times[warmup:], desc


def swap_accounting(n, cir, world, nl, amp_bytes, fused):
    """Per execute on one GPU: (bytes sent by NCCL swap all-to-alls, bytes
    stored into peers by passes with swaps fused into them, our kernels
    launched for the NCCL swaps, step indices of the fusing passes).

    An NCCL swap step: per run of m disjoint bit pairs (dist.cu) (1 - 2^-m)
    of the local slice leaves, with one gather and one scatter kernel per
    chunk round of up to 256 MiB. A fusing pass (fused=True: the state has
    peer memory) sends the amplitudes whose destination rank -- set by the
    m local bits its global permutation maps to rank bits -- is another one:
    (1 - 2^-m) of the slice, with no extra kernel."""
    if world == 1:
        return 0.0, 0.0, 0, []
    from paper_2512_18995_b200 import qsv

    sched = qsv.plan_schedule(n, cir.gates(), world=world)
    nccl = peer = 0.0
    kernels = 0
    fusing = []
    fused_done = False
    for i, step in enumerate(sched["steps"]):
        if step["kind"] == "pass":
            if step["fused"] and fused_done:
                continue
            fused_done = fused and bool(step["gperm"])
            if fused_done:
                m = sum(1 for b in range(nl) if step["gperm"][b] >= nl)
                peer += (amp_bytes << nl) * (1.0 - 2.0 ** -m)
                fusing.append(i)
            continue
        if step["fused"] and fused_done:
            continue
        fused_done = False
        runs, cur = [], []
        for gb, lb in step["pairs"]:
            if any(gb == g or lb == l for g, l in cur):
                runs.append(cur)
                cur = []
            cur.append((gb, lb))
        runs.append(cur)
        for r in runs:
            m = len(r)
            nccl += (amp_bytes << nl) * (1.0 - 2.0 ** -m)
            nv = (1 << m) - 1
            block = (1 << nl) >> m
            chunk = max(1, min(block * nv, (256 << 20) // amp_bytes) // nv)
            kernels += 2 * -(-block // chunk)
    return nccl, peer, kernels, fusing


def run_reference(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, the
    unmodified quasar headers) on this host, never loading libqsv.so."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    if not O.REF_LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libquasar_ref.so not built"}))
        return 0
    n = args.qubits
    times, desc = reference_cpu_sample(n, args.steps, args.warmup)
    t = float(np.sum(times))
    value = args.steps / t
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded Rng(0,'cfg3') Gaussian state)",
        "impl": "reference", "config": config_dict(n), "sample": desc,
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": 1, "host_cores": os.cpu_count(),
                         "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def _median_events(fn, stream, reps, warm=1):
    """1 warm-up + `reps` timed repeats, each bracketed by CUDA events on the
    engine's stream; the median ms (the reference CLI's protocol,
    tools/main.cpp:493-504)."""
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out)), out


def run_aux(ctx, stream, hbm_peak, want_cpu):
    """The other BASELINE.json configs on this GPU (device-resident, reference
    protocol: 1 warm-up + 10 repeats, median), with the reference's CPU path
    timed beside cfg1 / cfg2 on this host. Returns (aux dict, kernel launches)."""
    import time as _t

    from paper_2512_18995_b200 import qsv
    from paper_2512_18995_b200 import workloads as W

    L = qsv.lib()
    aux = {"protocol": "1 warm-up + 10 repeats, median; CUDA events on the engine stream"}
    launches = 0
    # ---- cfg1: 20q c128, 10 layers rx/ry/rz + CNOT ladder, all <Z_i> ----
    cir = W.cfg1_circuit()
    p = qsv.Plan(20, cir.gates(), dtype=qsv.C128, opts={"from_zero": 1})
    pg = qsv.Plan(20, cir.gates(), dtype=qsv.C128, opts={"from_zero": 1, "use_graph": 1})
    st = qsv.QubitState(20, dtype=qsv.C128)
    ms, _ = _median_events(lambda: p.execute(st), stream, 10)
    msg, _ = _median_events(lambda: pg.execute(st), stream, 10)
    p.execute_expect_z(st)  # warm-up (first use prepares the variant)
    t0 = _t.perf_counter()
    zs = [p.execute_expect_z(st) for _ in range(10)]
    msz = (_t.perf_counter() - t0) / 10 * 1e3
    npass = p.info["npasses"]
    launches += 21 * (npass + 1) + 11 * 10 + 10 * (npass + 3)
    l2_bytes = npass * 2 * 16 * (1 << 20)
    c1 = {"workload": "cfg1: 20-qubit c128, 10 layers of rx/ry/rz on every qubit + CNOT ladder (619 gates), "
                      "from |0>, all <Z_i>",
          "passes": npass, "us_per_forward": 1e3 * ms, "us_per_forward_graph": 1e3 * msg,
          "us_per_forward_plus_z_host": 1e3 * msz, "gates_per_s": 619 / (ms / 1e3),
          "l2_GBps": l2_bytes / (ms / 1e3) / 1e9,
          "note": "16 MiB state: L2-resident, launch/L2 bound (SURVEY.md 8(d))"}
    if want_cpu:
        from oracle import oracle as O

        sec = [O.ref_time_forward_z(20, cir.gates())[0] for _ in range(4)]
        c1["cpu_reference"] = {"ms_per_forward_plus_z": 1e3 * float(np.median(sec[1:])), "cores": 1,
                               "protocol": "1 warm-up + 3 repeats, median (Circuit::forward + expectation)"}
        want = O.ref_time_forward_z(20, cir.gates())[1][0]
        c1["z_max_abs_err_vs_reference"] = float(np.max(np.abs(zs[-1][0] - want)))
    aux["cfg1"] = c1
    del st, p, pg
    # ---- cfg2: 4096 x 12q c64 batched VQC, <Z_i> per circuit ----
    cir, data = W.cfg2_circuit()
    p = qsv.Plan(12, cir.gates(), dtype=qsv.C64, opts={"from_zero": 1})
    st = qsv.QubitState(12, batch=4096, dtype=qsv.C64)
    ms, _ = _median_events(lambda: p.execute(st, data), stream, 10)
    p.execute_expect_z(st, data)  # warm-up (first use compiles the fused <Z> variant)
    t0 = _t.perf_counter()
    for _ in range(10):
        z = p.execute_expect_z(st, data)
    msz = (_t.perf_counter() - t0) / 10 * 1e3
    launches += 11 * (p.info["npasses"] + 2) + 10 * (p.info["npasses"] + 2)
    c2 = {"workload": "cfg2: 4096 circuits x 12 qubits c64, encoded Ry(x) + 6 x (U3 + ring CZ), <Z_i> per circuit",
          "passes": p.info["npasses"], "ms_forward": ms, "circuits_per_s_forward": 4096 / (ms / 1e3),
          "ms_forward_plus_all_z_on_host": msz, "circuits_per_s": 4096 / (msz / 1e3),
          "note": "one pass, a whole circuit per CTA tile; <Z_i> fused into its last register group"}
    if want_cpu:
        from oracle import oracle as O

        sub = 512
        sec1, z1 = O.ref_time_forward_z(12, cir.gates(), data[:sub], 1)
        hc = os.cpu_count() or 1
        secs = [O.ref_time_forward_z(12, cir.gates(), data, hc)[0] for _ in range(6)]
        c2["cpu_reference"] = {
            "circuits_per_s_1core": sub / sec1, "sample_1core": f"first {sub} of the 4096 rows, 1 run",
            "circuits_per_s_all_cores": 4096 / float(np.median(secs[1:])), "cores": hc,
            "protocol_all_cores": "4096 rows fanned with quasar::parallel_for, 1 warm-up + 5 repeats, median"}
        c2["z_max_abs_err_vs_reference"] = float(np.max(np.abs(z[:sub] - z1)))
    aux["cfg2"] = c2
    del st, p
    # ---- adjoint gradients (adjoint.hpp:52-110) on the cfg1
    # circuit with every rotation trainable (600 parameters, sum of <Z_i>) ----
    n_adj = 20
    acir = W.cfg1_circuit(n_adj, trainable=True)
    qsv.adjoint_gradients(acir)  # warm-up (plans, kernels)
    ta = []
    for _ in range(9):
        t0 = _t.perf_counter()
        ag = qsv.adjoint_gradients(acir)
        ta.append(_t.perf_counter() - t0)
    nparams_adj = len(ag.param_grads)
    launches += 6 * (len(acir.gates()) + 4)
    adj = {"workload": f"adjoint_gradients of the cfg1 circuit at {n_adj} qubits c128 with every rotation trainable "
                       f"({nparams_adj} parameters, gradient of sum <Z_i>)",
           "ms_per_gradient": 1e3 * float(np.median(ta)), "ms_min": 1e3 * float(np.min(ta)),
           "protocol": "1 warm-up + 9 repeats, median (and min), host wall clock "
           "(forward plan, reverse sweep, one gradient read-back)",
           "note": "one fused kernel per reverse-sweep gate: psi' = U^dag psi, every parameter's Re<lambda|dU psi'>, "
                   "lambda' = U^dag lambda"}
    if want_cpu:
        from oracle import oracle as O

        t0 = _t.perf_counter()
        want, _ = O.ref_adjoint(n_adj, acir.gates(), [(list(o.wires), o.basis) for o in acir.observables()])
        adj["cpu_reference"] = {"ms_per_gradient": 1e3 * (_t.perf_counter() - t0), "cores": 1,
                                "protocol": "1 run of quasar::qubit::adjoint_gradients (oracle/_ref)"}
        adj["max_abs_err_vs_reference"] = float(np.max(np.abs(np.asarray(ag.param_grads) - want)))
    adj["note"] = ("runs of single-qubit gates on one wire as one reverse-sweep kernel (the psi/lambda pair in "
                   "registers through the run), other gates one kernel each: psi' = U^dag psi, every parameter's "
                   "Re<lambda|dU psi'>, lambda' = U^dag lambda (DESIGN.md 4.1c)")
    aux["adjoint_20q"] = adj
    # ---- training loops: the same structure with NEW trainable values every
    # step: steps 0-1 compile (the values in, then the
    # device-bound form), later steps reuse the passes ----
    def loop_steps(make, call, steps=5):
        out = []
        for k in range(steps):
            c = make(k)
            t0 = _t.perf_counter()
            call(c)
            out.append(1e3 * (_t.perf_counter() - t0))
        return out

    lrng = np.random.default_rng(0)

    def adj_circ(_k):
        c = qsv.Circuit(n_adj)
        for _ in range(10):
            for q in range(n_adj):
                c.rx(q, lrng.uniform(0, 2 * np.pi), True)
                c.ry(q, lrng.uniform(0, 2 * np.pi), True)
                c.rz(q, lrng.uniform(0, 2 * np.pi), True)
        for q in range(n_adj - 1):
            c.cnot(q, q + 1)
        for q in range(n_adj):
            c.observable([q], "z")
        return c

    t_adj = loop_steps(adj_circ, lambda c: qsv.adjoint_gradients(c))
    t_fwd = loop_steps(adj_circ, lambda c: c.forward())
    d2 = lrng.uniform(-np.pi, np.pi, (4096, 12))

    def cfg2_circ(_k):
        c = qsv.Circuit(12)
        for q in range(12):
            c.add(qsv.make_gate("ry", [q], [], [0.0], False, True))
        for _ in range(6):
            for q in range(12):
                c.add(qsv.make_gate("u3", [q], [], list(lrng.uniform(0, 2 * np.pi, 3)), True))
            for q in range(12):
                c.cz(q, (q + 1) % 12)
        return c

    t_c2 = loop_steps(cfg2_circ, lambda c: qsv.run_rows_expect_z(c, d2))
    launches += 3 * 5 * 2 * len(adj_circ(0).gates())
    aux["training_loops"] = {
        "workload": "new trainable values every step, host wall clock per step: adjoint_gradients and "
                    "Circuit.forward of the cfg1-shaped circuit at 20q c128 (600 trainable rotations), and cfg2 "
                    "(4096 rows x 12q c64, new shared U3 angles) through run_rows_expect_z",
        "adjoint_20q_ms_per_step": [round(x, 2) for x in t_adj],
        "forward_20q_ms_per_step": [round(x, 2) for x in t_fwd],
        "cfg2_ms_per_step": [round(x, 2) for x in t_c2],
        "note": "steps 0-1 include code generation + NVRTC (values compiled in, then the device-bound form); "
                "from step 2 on no compile: the reference's own CPU path takes ~17 s per 20q gradient and "
                "~0.9 s per cfg2 step on 16 cores (aux.adjoint_20q / aux.cfg2)"}
    # ---- seeded measurement (circuit.hpp:217-244): marginals
    # over 20 wires of a 24-qubit state on the device, 10^6 shots sampled on
    # the host with the reference's Rng stream; the histogram must equal the
    # reference's own ----
    n_m, wires_m, shots_m = 24, list(range(20)), 1_000_000
    amps_m = W.cfg3_slice(0, 1 << n_m)
    amps_m /= np.sqrt(float(np.vdot(amps_m, amps_m).real))
    sm = qsv.QubitState.from_amplitudes(n_m, amps_m)
    qsv.measure_counts(sm, shots_m, wires_m, qsv.Rng(5, "bench-measure"))  # warm-up
    tm = []
    for _ in range(3):
        t0 = _t.perf_counter()
        got_m, _ = qsv.measure_counts(sm, shots_m, wires_m, qsv.Rng(5, "bench-measure"))
        tm.append(_t.perf_counter() - t0)
    launches += 4 * 2
    meas = {"workload": f"measure: {shots_m} shots over wires 0..19 of a 24-qubit c128 state (seeded Gaussian), "
                        "histogram as an array (qsv_measure)",
            "ms_per_call": 1e3 * float(np.median(tm)), "protocol": "1 warm-up + 3 repeats, median, host wall clock"}
    if want_cpu:
        from oracle import oracle as O

        t0 = _t.perf_counter()
        want_m = O.ref_measure(n_m, amps_m, shots_m, wires_m, 5, "bench-measure")
        meas["cpu_reference"] = {"ms_per_call": 1e3 * (_t.perf_counter() - t0), "cores": 1,
                                 "protocol": "1 run of quasar::qubit::measure (oracle/_ref)"}
        meas["histogram_identical_to_reference"] = bool(np.array_equal(got_m, want_m))
    aux["measure_24q"] = meas
    del sm
    # ---- density matrices and channels (state.hpp:159-172,
    # channel.hpp:73-100): 10 qubits (rho 1024 x 1024 as a 20-qubit vector),
    # 4 layers of ry on every wire, a depolarizing channel on every wire and a
    # CNOT ladder; value semantics like the reference (every op returns a new
    # state) ----
    n_d = 10
    rng_d = qsv.Rng(0, "bench-density")
    ops_d = []
    for _ in range(4):
        for q in range(n_d):
            ops_d.append(qsv.make_gate("ry", [q], [], [rng_d.uniform(0.0, 6.283185307179586)]))
            ops_d.append(("depolarizing", q, 0.01))
        for q in range(n_d - 1):
            ops_d.append(qsv.make_gate("x", [q + 1], [q]))

    def run_density():
        sd = qsv.QubitState.basis(n_d)
        for op in ops_d:
            sd = qsv.apply_channel(sd, qsv.depolarizing(op[1], op[2])) if isinstance(op, tuple) else \
                qsv.apply_gate(sd, op)
        return sd

    run_density()
    td = []
    for _ in range(3):
        t0 = _t.perf_counter()
        sd = run_density()
        sd.ctx.sync()
        td.append(_t.perf_counter() - t0)
    launches += 4 * 3 * len(ops_d)
    dens = {"workload": f"density matrix, {n_d} qubits c128: {len(ops_d)} ops (ry + depolarizing on every wire, "
                        "CNOT ladder) x 4 layers from |0><0|",
            "ms_per_run": 1e3 * float(np.median(td)), "protocol": "1 warm-up + 3 repeats, median, host wall clock"}
    if want_cpu:
        from oracle import oracle as O

        t0 = _t.perf_counter()
        want_d = O.ref_mixed_run(n_d, ops_d)
        dens["cpu_reference"] = {"ms_per_run": 1e3 * (_t.perf_counter() - t0), "cores": 1,
                                 "protocol": "1 run of to_mixed + apply_gate / apply_channel (oracle/_ref)"}
        dens["max_abs_err_vs_reference"] = float(np.max(np.abs(sd.density() - want_d)))
    aux["density_10q"] = dens
    # ---- cfg4 / cfg5 families at the largest single-GPU sizes ----
    for name, n, cir, dt, desc in (
            ("cfg4_32q", 32, W.cfg4_circuit(32), qsv.C128,
             "cfg4 family at 32 qubits c128 (64 GiB): 20 layers of U3 + brickwork CNOT (950 gates)"),
            ("cfg5_33q", 33, W.cfg5_circuit(33), qsv.C64,
             "cfg5 family at 33 qubits c64 (64 GiB): 16 layers of rx/ry/rz + random-pair CZ (1856 gates)")):
        tp = _t.perf_counter()
        p = qsv.Plan(n, cir.gates(), dtype=dt)
        plan_s = _t.perf_counter() - tp
        st = qsv.QubitState(n, dtype=dt)
        p.profile(st)  # warm-up
        runs = [p.profile(st) for _ in range(3)]
        per = np.array(runs)
        tot = float(np.median(per.sum(axis=1)))
        amp = 8 if dt == qsv.C64 else 16
        bpl = 2.0 * amp * (1 << n)
        avg = float(per.mean())
        aux[name] = {"workload": desc, "passes": p.info["npasses"], "ms_per_forward": tot,
                     "gates_per_s": p.info["ngates"] / (tot / 1e3), "plan_seconds": plan_s,
                     "avg_pass_GBps": bpl / (avg / 1e3) / 1e9, "frac_of_measured_hbm": bpl / (avg / 1e3) / 1e9 / hbm_peak,
                     "protocol": "1 warm-up + 3 repeats (each a full forward with per-pass events), median",
                     "per_pass_ms": [round(float(x), 4) for x in per.mean(axis=0)],
                     "hbm_floor_ms": p.info["npasses"] * bpl / (hbm_peak * 1e9) * 1e3,
                     "bound": ("FP64 pipe (ncu: 57-66 % busy, profiles/r02_ncu_cfg4f_28q_passenger.txt)" if dt == qsv.C128
                               else "FMA pipe / latency (ncu: FMA 40-52 %, profiles/r02_ncu_cfg5f_28q.txt)"),
                     "note": ("passes fuse more gates each than in round 1 (" +
                              ("32q cfg4: 17 passes vs 32" if dt == qsv.C128 else "33q cfg5: 18 passes vs 20") +
                              "), so per-pass GB/s is lower while the forward is faster; the passes are "
                              "compute-bound, the HBM fraction is not their roofline")}
        launches += 4 * p.info["npasses"]
        del st, p
    # ---- north_star (2)'s tensor-core blocks, measured where they are
    # genuinely dense (NOT a BASELINE config): a 30-qubit c64 brickwork of
    # Haar-random two-qubit unitaries, the fused FFMA passes against the
    # dense-block tensor-core passes (opts.dense_blocks) on the same circuit
    st = qsv.QubitState(30, dtype=qsv.C64)
    for name, cir, desc in (
            ("dense_local_30q", W.dense_local_circuit(30, 5, 20),
             "demonstration (not a BASELINE config): 30-qubit c64, 6 windows of 5 wires, each a 20-layer brickwork "
             "of Haar-random two-qubit unitaries (240 gates, ~40 dense gates per 5-qubit block)"),
            ("dense_brickwork_30q", W.dense_brickwork_circuit(30, 20),
             "demonstration (not a BASELINE config): 30-qubit c64 brickwork over all wires, 20 layers of "
             "Haar-random two-qubit unitaries (290 gates, ~4 per 5-qubit block)")):
        dz = {"workload": desc, "protocol": "1 warm-up + 3 repeats (per-pass events), median"}
        for key, opts in (("ffma_passes", {"dense_blocks": -1}), ("tensor_core_blocks", {"dense_blocks": 1})):
            p = qsv.Plan(30, cir.gates(), dtype=qsv.C64, opts=opts)
            p.profile(st)
            tot = float(np.median([p.profile(st).sum() for _ in range(3)]))
            dz[key] = {"ms_per_forward": tot, "passes": p.info["npasses"], "blocks": p.info["nblocks"]}
            launches += 4 * p.info["npasses"]
            del p
        auto = qsv.Plan(30, cir.gates(), dtype=qsv.C64)
        dz["auto_mode_uses"] = "tensor_core_blocks" if auto.info["nblocks"] else "ffma_passes"
        del auto
        aux[name] = dz
    del st
    return aux, launches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qsv")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-aux", action="store_true")
    ap.add_argument("--qubits", type=int, default=N_QUBITS, help="(diagnostics only) qubit count")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    from paper_2512_18995_b200 import build as B

    B.build()
    from paper_2512_18995_b200 import qsv
    from paper_2512_18995_b200 import workloads as W

    rank, world, local = dist_env()
    assert world == args.gpus or "WORLD_SIZE" not in os.environ, "--gpus must match the torchrun world size"
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        # NCCL's own init lines (ranks, devices, transports: NVLS / P2P) go to
        # stderr, so a scaling run records what the communicator saw
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo", init_method="env://")
        uid = [qsv.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = qsv.Context(local, rank, world, uid[0])
    else:
        ctx = qsv.Context(local)
    qsv.set_default_context(ctx)
    n = args.qubits
    cir = W.cfg3_circuit(n)
    g = int(np.log2(world))
    nl = n - g
    # this rank's slice of the seeded input (counter-based stream: no rank
    # generates more than its own 2^(n-g) amplitudes), normalised globally
    mine = W.cfg3_slice(rank << nl, 1 << nl)
    ss = float(np.dot(mine.view(np.float64), mine.view(np.float64)))
    if world > 1:
        t = torch.tensor([ss], dtype=torch.float64)
        torch.distributed.all_reduce(t)
        ss = float(t.item())
    mine /= np.sqrt(ss)
    plan = qsv.Plan(n, cir.gates(), dtype=qsv.C128, ctx=ctx)
    st = qsv.QubitState(n, dtype=qsv.C128, ctx=ctx)
    st.upload(mine)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        plan.execute(st)
    ctx.sync()
    barrier()
    npass = plan.info["npasses"]
    launch_ms = []
    with Clocks(local) as clk:
        ctx.sync()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            launch_ms.append(plan.profile(st))  # one execution, events around every launch
        e1.record(stream)
        e1.synchronize()
        ctx.sync()
        barrier()
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([t_ms], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_ms = float(t.item())
    ngates = plan.info["ngates"]
    value = args.steps * ngates / (t_ms / 1e3)

    # ---- roofline of the dominant kernel (the fused tile pass) ----
    kinds = plan.step_kinds()
    lm = np.array(launch_ms)[:, kinds == 0]  # steps x passes (qubit-swap steps excluded)
    amp_bytes = 16
    # qubit swaps (N > 1): bytes each GPU sends per execute over the swap
    # steps' time, against the measured 770 GB/s per-direction peer copy and
    # the nominal 900 GB/s (B200_PROFILING.md)
    nvlink = None
    fused = world > 1 and st.peer_memory() == 1
    nccl_sent, peer_sent, swap_kern, fusing = swap_accounting(n, cir, world, nl, amp_bytes, fused)
    if world > 1 and (nccl_sent or peer_sent):
        lmall = np.array(launch_ms)
        sw_ms = float(lmall[:, kinds == 1].sum(axis=1).mean()) if (kinds == 1).any() else 0.0
        fz_ms = float(lmall[:, fusing].sum(axis=1).mean()) if fusing else 0.0
        sent = nccl_sent + peer_sent
        t = sw_ms + fz_ms
        gbs = sent / (t / 1e3) / 1e9 if t > 0 else None
        nvlink = {"bytes_sent_per_gpu_per_step": sent, "nccl_swap_bytes": nccl_sent, "peer_store_bytes": peer_sent,
                  "swaps": "fused into the passes (peer-memory stores)" if fused else "NCCL all-to-all",
                  "swap_ms_per_step": sw_ms, "fusing_pass_ms_per_step": fz_ms,
                  # the fusing passes also do their gate math: a lower bound of the link rate
                  "achieved_GBps": gbs, "frac_of_measured_770": gbs / 770.0 if gbs else None,
                  "frac_of_nominal_900": gbs / 900.0 if gbs else None}
    bytes_per_launch = 2.0 * amp_bytes * (1 << nl)  # read + write of every local amplitude
    avg_launch_ms = float(lm.mean())
    hbm_peak, peak_kind = peaks()
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    traffic = None  # DRAM bytes per launch from the committed ncu --set full capture of this workload
    tp = ROOT / "profiles" / "r02_traffic_cfg3_30q_final.json"
    if tp.exists() and n == N_QUBITS and world == 1:
        traffic = json.loads(tp.read_text())["traffic_per_launch_bytes"]

    # ---- end to end through the C ABI with pinned host buffers ----
    # Every step uploads its input state from pinned host memory, executes
    # the plan and downloads the result (qsv_state_upload_raw_async /
    # execute / qsv_state_download_raw_async, all stream-ordered). Two states
    # on two contexts (two CUDA streams) alternate, so step i's download
    # overlaps step i+1's upload (PCIe is full duplex); every step still moves
    # its full input and output. A lane waits for its own previous step
    # (qsv_ctx_sync) before reusing its output buffer.
    e2e = None
    if args.e2e_steps > 0:
        if world > 1:
            uid2 = [qsv.Context.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(uid2, src=0)
            ctx2 = qsv.Context(local, rank, world, uid2[0])
        else:
            ctx2 = qsv.Context(local)
        plan2 = qsv.Plan(n, cir.gates(), dtype=qsv.C128, ctx=ctx2)
        st2 = qsv.QubitState(n, dtype=qsv.C128, ctx=ctx2)
        stream2 = torch.cuda.ExternalStream(ctx2.stream(), device=torch.device("cuda", local))
        host_in = torch.from_numpy(mine.view(np.float64)).pin_memory()
        host_out = [torch.empty_like(host_in).pin_memory(), torch.empty_like(host_in).pin_memory()]
        L = qsv.lib()
        cnt = 1 << nl
        lanes = [(plan, st, ctx), (plan2, st2, ctx2)]
        plan2.execute(st2)  # warm-up (kernel loading) of the second lane
        ctx.sync()
        ctx2.sync()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        stream2.wait_event(f0)
        for i in range(args.e2e_steps):
            p_i, s_i, c_i = lanes[i % 2]
            if i >= 2:
                c_i.sync()  # this lane's previous download has landed
            qsv.check(L.qsv_state_upload_raw_async(s_i.h, 0, host_in.data_ptr(), cnt))
            p_i.execute(s_i)
            qsv.check(L.qsv_state_download_raw_async(s_i.h, 0, host_out[i % 2].data_ptr(), cnt))
        done2 = torch.cuda.Event()
        done2.record(stream2)
        stream.wait_event(done2)
        f1.record(stream)
        f1.synchronize()
        barrier()
        e2e_ms = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": args.e2e_steps * ngates / (e2e_ms / 1e3), "unit": "gates/s",
               "h2d_bytes_per_step": cnt * 16, "d2h_bytes_per_step": cnt * 16,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "pipeline": "2 states on 2 streams: step i's download overlaps step i+1's upload"}
        del st2, plan2
        ctx2.close()

    cpu = None
    want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    aux = None
    aux_launches = 0
    if rank == 0 and world == 1 and not args.no_aux and n == N_QUBITS:
        del st
        aux, aux_launches = run_aux(ctx, stream, hbm_peak, want_cpu)
    if want_cpu:
        from oracle import oracle as O

        if O.REF_LIB.exists():
            times, desc = reference_cpu_sample(n, 4, 1)
            cpu = {"value": len(times) / float(np.sum(times)), "unit": "gates/s", "cores": 1,
                   "host_cores": os.cpu_count(), "kind": "reference", "sample": desc}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded Rng(0,'cfg3') Gaussian state, normalised in FP64)",
            "config": config_dict(n),
            "plan": {"passes_per_step": npass, "swaps_per_step": plan.info["nswaps"],
                     "parallelism": f"state sharded over {world} GPU(s)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "frac_nominal": achieved / NOMINAL_HBM_GBS, "peak_nominal": NOMINAL_HBM_GBS,
                         "traffic_source": "profiles/r02_traffic_cfg3_30q_final.json (ncu --set full dram__bytes_read+write per launch)",
                         "kernel": "qsv_pass (NVRTC-specialised fused tile pass)", "bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": avg_launch_ms,
                         "per_pass_ms": [round(float(x), 4) for x in lm.mean(axis=0)]},
            "gpu_launches": args.steps * (npass + swap_kern),
            "gpu_launches_aux": aux_launches,
            "nvlink": nvlink,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "aux": aux,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
