"""Benchmark: BASELINE.json metric "gate passes/sec and achieved HBM GB/s per
pass at n qubits" on config 3 -- the 30-qubit complex128 QFT (+ final swaps)
on the seeded, normalised Gaussian input state, one B200 (16 GiB state).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Arms
  default      the engine (libqsv.so, fused sm_100a tile passes) through the C
               ABI. A step = one full execution of the 495-gate circuit on the
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


def cpu_reference_sample(cir, n, psi, gates_per_step, steps):
    """The reference CPU path on a bounded sample: quasar::qubit::apply_gate
    over `gates_per_step` gates of the same circuit, `steps` times."""
    from oracle import oracle as O

    gl = cir.gates()
    times = []
    state = psi
    for s in range(steps):
        sample = [gl[(s * gates_per_step + j) % len(gl)] for j in range(gates_per_step)]
        sec, state = O.ref_time_apply(n, sample, state)
        times.append(sec)
    return times


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
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2512_18995_b200 import workloads as W

    if not O.REF_LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libquasar_ref.so not built"}))
        return 0
    n = N_QUBITS
    cir = W.cfg3_circuit(n)
    psi = W.cfg3_input(n)
    times = cpu_reference_sample(cir, n, psi, 1, args.warmup + args.steps)[args.warmup:]
    t = float(np.sum(times))
    value = args.steps / t
    line = {
        "metric": "gate passes/sec at n qubits (source gates applied to the full state per second)",
        "value": value, "unit": "gates/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded Rng(0,'cfg3') Gaussian state)",
        "impl": "reference",
        "config": {"workload": WORKLOAD, "n_qubits": n, "sample": "1 gate of the circuit per step, in order"},
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} gates of cfg3 at n=30 via quasar::qubit::apply_gate "
                                   "(single-threaded reference path; parallel_for is unused by it)"},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qsv")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    psi = mine  # full state when world == 1 (the CPU baseline samples it)
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

    # ---- roofline of the dominant kernel (tile_pass_kernel) ----
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
    tp = ROOT / "profiles" / "r01_traffic_cfg3_30q.json"
    if tp.exists() and n == N_QUBITS and world == 1:
        traffic = json.loads(tp.read_text())["traffic_per_launch_bytes"]

    # ---- end to end through the C ABI with pinned host buffers ----
    # Every step uploads its input state from pinned host memory, executes
    # the plan and downloads the result (qsv_state_upload_raw / execute /
    # qsv_state_download_raw). Two states on two contexts (two CUDA streams)
    # alternate, so step i's download overlaps step i+1's upload (PCIe is
    # full duplex); every step still moves its full input and output.
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
        host_out = torch.empty_like(host_in).pin_memory()
        L = qsv.lib()
        cnt = 1 << nl
        lanes = [(plan, st, stream), (plan2, st2, stream2)]
        plan2.execute(st2)  # warm-up (kernel loading) of the second lane
        ctx.sync()
        ctx2.sync()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        stream2.wait_event(f0)
        for i in range(args.e2e_steps):
            p_i, s_i, _ = lanes[i % 2]
            qsv.check(L.qsv_state_upload_raw(s_i.h, 0, host_in.data_ptr(), cnt))
            p_i.execute(s_i)
            if i >= 1:  # the previous step's result, while this step's upload streams in
                qsv.check(L.qsv_state_download_raw(lanes[(i - 1) % 2][1].h, 0, host_out.data_ptr(), cnt))
        last = lanes[(args.e2e_steps - 1) % 2]
        qsv.check(L.qsv_state_download_raw(last[1].h, 0, host_out.data_ptr(), cnt))
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
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        if O.REF_LIB.exists():
            times = cpu_reference_sample(cir, n, psi, 1, 2)
            cpu = {"value": 2 / float(np.sum(times)), "unit": "gates/s", "cores": 1, "kind": "reference",
                   "sample": "first 2 gates of cfg3 (h(0), cp(1,0)) at n=30 via quasar::qubit::apply_gate, "
                             "single thread"}
    if rank == 0:
        line = {
            "metric": "gate passes/sec at n qubits (source gates applied to the full state per second)",
            "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded Rng(0,'cfg3') Gaussian state, normalised in FP64)",
            "config": {"workload": WORKLOAD, "n_qubits": n, "gates": ngates, "passes_per_step": npass,
                       "swaps_per_step": plan.info["nswaps"], "parallelism": f"state sharded over {world} GPU(s)",
                       "l2": "state (16 GiB) >> L2 (126 MB); no flush needed"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "traffic_source": "profiles/r01_traffic_cfg3_30q.json (ncu dram__bytes_read+write per launch)",
                         "kernel": "qsv_pass (NVRTC-specialised fused tile pass)", "bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": avg_launch_ms,
                         "per_pass_ms": [round(float(x), 4) for x in lm.mean(axis=0)]},
            "gpu_launches": args.steps * (npass + swap_kern),
            "nvlink": nvlink,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
