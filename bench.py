#!/usr/bin/env python3
"""Benchmark of the hot path: one SGD training iteration (feed -> Net::forward ->
SoftmaxWithLoss -> Net::backward -> momentum-SGD update) of AlexNet at batch
256 per GPU (BASELINE.json configs[3], the largest single-GPU config; float ->
3xTF32 tensor cores).  The other configs are behind --workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload alexnet|cifar10_quick|lenet|resnet20] [--dtype f32|f64]

Prints ONE JSON line (rank 0).  N > 1: one rank per GPU (launched by
torch.distributed.run, or bench.py re-executes itself under it when WORLD_SIZE
is unset), NCCL gradient all-reduce (weak scaling: the per-GPU batch is fixed).

* value      images/s with the batch already resident in HBM (captured CUDA
             graph of the step), L2 flushed (256 MiB write) before every timed
             step, CUDA events on the compute stream, max over ranks.
* e2e        images/s through the public API with host buffers: each step copies
             that step's batch into pinned memory, replays the graph whose first
             node is the H2D copy and last node the D2H of the loss, and reads
             the loss; polegrad.FeedRing (two pinned slots) lets the host stage
             batch i+1 while step i runs.
* roofline   the dominant kernel (per-layer event profile of one eager step).
* cpu_baseline  the reference CPU implementation (oracle/_ref: unmodified
             reference core + reference-style conv/pool/loss extension, 1 thread)
             on a bounded sample.
--impl reference  times that CPU implementation on all host cores (independent
             replicas), same metric / config.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training images/sec (fwd+bwd+SGD) at 1/2/4/8 B200 vs CPU ref; ms/iter"
UNIT = "images/s"
# BASELINE.json configs; the default (headline) workload is configs[1].  ref_batch:
# images per reference-CPU step per process (bounded sample; CPU cost is linear in batch).
WORKLOADS = {
    "cifar10_quick": dict(batch=100, img=(3, 32, 32), classes=10, ref_batch=20, cpu_batch=100,
                          solver=dict(method="sgd", lr=0.001, momentum=0.9, weight_decay=0.004)),
    "lenet": dict(batch=64, img=(1, 28, 28), classes=10, ref_batch=64, cpu_batch=64,
                  solver=dict(method="sgd", lr=0.01, momentum=0.9, weight_decay=5e-4)),
    "alexnet": dict(batch=256, img=(3, 227, 227), classes=1000, ref_batch=1, cpu_batch=2,
                    solver=dict(method="sgd", lr=0.001, momentum=0.9, weight_decay=5e-4)),
    "resnet20": dict(batch=128, img=(3, 32, 32), classes=10, ref_batch=8, cpu_batch=16,
                     solver=dict(method="sgd", lr=0.1, momentum=0.9, weight_decay=1e-4)),
    # configs[2]: the reference's pg_softmax graph (4-10-2 + Softmax + MemoryLoss) at batch
    # 1024; the unit is Cart-Pole states per second (BASELINE.md §3 times the same
    # iteration on the unmodified reference Net: enqueue, forward, logits diff,
    # backward_from("logits"), plain SGD)
    "pg_mlp": dict(batch=1024, img=(4, 1, 1), classes=2, ref_batch=1024, cpu_batch=1024,
                   solver=dict(method="sgd", lr=0.001, momentum=0.0, weight_decay=0.0)),
}
DEFAULT_WORKLOAD = "alexnet"
WORKLOAD = DEFAULT_WORKLOAD
BATCH = WORKLOADS[WORKLOAD]["batch"]
SOLVER = WORKLOADS[WORKLOAD]["solver"]
IMG = WORKLOADS[WORKLOAD]["img"]
CLASSES = WORKLOADS[WORKLOAD]["classes"]
REF_SAMPLE_BATCH = WORKLOADS[WORKLOAD]["ref_batch"]  # images per reference step per process
DTYPE = "f32"


def select_workload(name: str) -> None:
    global WORKLOAD, BATCH, SOLVER, IMG, CLASSES, REF_SAMPLE_BATCH
    w = WORKLOADS[name]
    WORKLOAD, BATCH, SOLVER, IMG, CLASSES, REF_SAMPLE_BATCH = (name, w["batch"], w["solver"], w["img"],
                                                               w["classes"], w["ref_batch"])


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def model_text(batch: int) -> str:
    from paper_1810_02272_b200 import polegrad
    return polegrad.load_model(WORKLOAD, batch)


def config(n_gpus: int) -> dict:
    """The workload (identical on both arms)."""
    return {"workload": WORKLOAD, "per_gpu_batch": BATCH, "global_batch": BATCH * n_gpus,
            "input": "x".join(map(str, IMG)), "classes": CLASSES, "real": DTYPE,
            "solver": f"SGD lr={SOLVER['lr']:g} momentum={SOLVER['momentum']:g} "
                      f"weight_decay={SOLVER['weight_decay']:g}",
            "l2": "flushed (256 MiB device write) before every timed step",
            "parallelism": f"dp{n_gpus}" if n_gpus > 1 else "single"}


def dtype_label() -> str:
    if WORKLOAD == "pg_mlp":  # the fused MLP update: CUDA-core arithmetic, no tensor cores
        return "fp64 (CUDA cores, fused MLP update)" if DTYPE == "f64" else "fp32 (CUDA cores, fused MLP update)"
    if DTYPE == "f64":
        return "fp64 (SIMT DFMA)"
    return "fp32 (3xTF32 tensor cores)" if os.environ.get("CDNN_MATH", "tf32x3") == "tf32x3" else "fp32 (TF32)"


# --------------------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.path or not os.path.exists(self.path):
            return out
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return out
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        loaded = [s for s in sm if s > 500] or sm
        out.update(sm_mhz=statistics.median(loaded) if loaded else None, sm_max_mhz=max(mx) if mx else None,
                   reasons=sorted(reasons), samples=len(rows))
        return out


# --------------------------------------------------------------------------------------
class CtxView:
    """cudadnn calls on the net's own context (events, flush buffer, launch count)."""

    def __init__(self, ptr: int):
        from paper_1810_02272_b200 import cudadnn
        self.cd = cudadnn
        self.lib = cudadnn.load()
        self.ptr = C.c_void_p(ptr)

    def call(self, name, *args):
        self.cd.check(getattr(self.lib, name)(self.ptr, *args))

    def out_h(self, name, *args) -> int:
        h = C.c_uint64()
        self.call(name, *args, C.byref(h))
        return h.value

    def event(self) -> int:
        return self.out_h("cdnn_event_create")

    def record(self, ev):
        self.call("cdnn_event_record", ev, 0)

    def elapsed(self, a, b) -> float:
        v = C.c_float()
        self.call("cdnn_event_elapsed", a, b, C.byref(v))
        return v.value

    def launches(self) -> int:
        v = C.c_uint64()
        self.call("cdnn_launch_count", C.byref(v))
        return v.value


def layer_flops(net) -> dict:
    """Algorithmic FLOPs (2*M*N*K) of each contraction, forward and backward,
    from the net's own parameter and top shapes (in the bundled models each
    parameterised layer's top blob carries the layer's name)."""
    out = {}
    first = True
    for pname, wshape in net.param_info():
        if not pname.endswith(".weight"):
            continue
        lname = pname[: -len(".weight")]
        try:
            top = net.blob_shape(lname)
        except Exception:  # in-place layers (Scale) have no top of their own name
            continue
        if wshape[0] == 1 and wshape[1] == 1 and wshape[2] == 1:  # Scale (1,1,1,C): elementwise
            continue
        if wshape[0] == 1 and wshape[1] == 1:  # InnerProduct weight (1,1,O,K)
            f = 2.0 * top[0] * wshape[2] * wshape[3]
            out[lname] = {"fwd": f, "bwd": 2 * f}  # wgrad + dgrad (the reference always writes dX)
        else:  # Convolution weight (Co, C/g, kh, kw)
            n, co, p, q = top
            f = 2.0 * n * p * q * co * wshape[1] * wshape[2] * wshape[3]
            out[lname] = {"fwd": f, "bwd": f * (1 if first else 2)}  # no dgrad into the input data
        first = False
    return out


def peaks() -> dict:
    """Roofline denominators: HBM and bf16 from the driver's MEASURED_PEAKS.json; the
    dense TF32 (float path) and FP64 (double path) cuBLAS rates from
    profiles/r02_peaks.json, measured on a B200 of this pool by
    profiles/measure_peaks.py (MEASURED_PEAKS.json carries no TF32 / FP64 figure)."""
    out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out.update(hbm_gbs=float(d["hbm_gbs"]), bf16_tflops=float(d["bf16_tflops"]), source="measured")
    except Exception:
        pass
    try:
        m = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))
        out["tf32_tflops"] = float(m["tf32"]["burst_tflops"])
        out["fp64_tflops"] = float(m["fp64"]["burst_tflops"])
        out["tc_source"] = ("measured: torch.matmul 8192^3 burst on a B200 of this pool "
                            "(profiles/r02_peaks.json, profiles/measure_peaks.py)")
    except Exception:
        out["tf32_tflops"] = out["bf16_tflops"] / 2.0
        out["fp64_tflops"] = None
        out["tc_source"] = f"derived: bf16 {out['bf16_tflops']} / 2 ({out['source']})"
    return out


def ncu_traffic(kernel_key: str):
    """DRAM bytes (read + write) per launch of the dominant layer op, from the committed
    ncu capture of THIS workload, batch and dtype (profiles/ncu_summary.json, keyed
    '<workload>/b<batch>/<dtype>' -> '<layer>.<fwd|bwd>'); None when no capture exists."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d["traffic_bytes_per_launch"][f"{WORKLOAD}/b{BATCH}/{DTYPE}"].get(kernel_key)
    except Exception:
        return None


def host_cpu() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline_sample(iters: int = 2) -> dict:
    from oracle import pyoracle
    if not pyoracle.available("f32"):
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": "oracle/_ref not built on this host"}
    cb = WORKLOADS[WORKLOAD]["cpu_batch"]
    dt = ref_steps(cb, iters, 0, 2)
    unit = "states/s" if WORKLOAD == "pg_mlp" else UNIT
    what = ("the UNMODIFIED reference Net (pg_softmax graph, reference prototxt parser; enqueue, forward, "
            "logits diff, backward_from, SGD)" if WORKLOAD == "pg_mlp" else
            "unmodified reference core (kernels::gemm, InnerProduct, ReLU, solver) + reference-style "
            "Convolution/Pooling/SoftmaxWithLoss extension")
    return {"value": iters * cb / dt, "unit": unit, "cores": 1, "kind": "reference",
            "ms_per_step": 1000 * dt / iters, **host_cpu(),
            "sample": f"{iters} iterations of {WORKLOAD} at batch {cb} ({DTYPE}) on oracle/_ref: {what}, 1 thread"}


def ref_steps(nb: int, steps: int, warmup: int, seed: int) -> float:
    """Seconds for `steps` reference-CPU iterations of the workload at batch nb (after
    `warmup` untimed ones) on oracle/_ref."""
    from oracle import pyoracle
    text = model_text(nb)
    net = pyoracle.OracleNet(text, seed=1, dtype=DTYPE)
    solver = pyoracle.OracleSolver(net, **SOLVER)
    rng = np.random.default_rng(seed)
    if WORKLOAD == "pg_mlp":
        st, act, ret = pg_inputs(rng, 1, nb, np.float64)
        g = rng.uniform(-1, 1, (nb, 2))  # modulated log-prob gradients at the logits

        def one():
            net.set_batch(st[0])
            net.forward()
            net.set_blob("logits", g, diff=True)
            net.backward_from("logits")
            solver.apply()
    else:
        x = rng.uniform(-1, 1, (nb,) + IMG)
        y = np.floor(rng.uniform(0, 1, nb) * CLASSES)

        def one():
            net.set_batch(x, y)
            net.forward()
            net.backward()
            solver.apply()
    for _ in range(warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    return time.perf_counter() - t0


# --------------------------------------------------------------------------------------
def run_b200(args) -> None:
    import torch.distributed as dist  # plumbing only (rendezvous, barrier, max-over-ranks)
    from paper_1810_02272_b200 import cudadnn, polegrad

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE")
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    text = model_text(BATCH)
    if args.dp_transport == "host":  # validation runs may put several ranks on one GPU
        local = local % max(1, cudadnn.device_count())
    net = polegrad.Net(text, seed=1, dtype=DTYPE, device=local)
    solver = polegrad.Solver(net, **SOLVER)
    cx = CtxView(net.context_ptr())
    par = None
    if world > 1 and args.dp_transport == "host":
        # validation of the N > 1 path where NCCL cannot run (several ranks on one GPU):
        # the product's Parallel with its host transport over gloo (eager steps only)
        import torch

        def transport(op, arr, offset):
            t = torch.from_numpy(arr)
            if op == 0:
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
            else:
                dist.broadcast(t, src=0)

        par = polegrad.Parallel.host(net, world, rank, transport)
        par.broadcast()
        solver.set_parallel(par)
        args.no_graph = True
    elif world > 1:
        uid = [polegrad.Parallel.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        par = polegrad.Parallel(net, world, rank, uid[0])
        par.broadcast()
        solver.set_parallel(par)
    nccl_ranks = par.info() if par else None
    if nccl_ranks:
        log(f"rank {rank}: the Parallel communicator reports {nccl_ranks['nranks']} ranks (this one {nccl_ranks['rank']}), "
            f"{nccl_ranks['buckets']} gradient buckets")
        if nccl_ranks["nranks"] != world:
            raise RuntimeError(f"NCCL communicator has {nccl_ranks['nranks']} ranks, WORLD_SIZE {world}")

    npd = polegrad.NP_DTYPE[DTYPE]
    rng = np.random.default_rng(2 + rank)
    nb = min(3, max(args.steps, 1))  # distinct host batches, cycled
    host_x = rng.uniform(-1, 1, (nb, BATCH) + IMG).astype(npd)
    host_y = np.floor(rng.uniform(0, 1, (nb, BATCH)) * CLASSES).astype(npd)

    # eager step: allocates workspaces / tensor maps, counts kernel launches per step
    net.set_batch(host_x[0], host_y[0])
    l0 = cx.launches()
    net.forward()
    net.backward()
    solver.apply()
    net.sync()
    launches_per_step = cx.launches() - l0

    # per-layer device-time profile of one eager step (kernel shares)
    nl = len(net.layer_names())
    fwd = (C.c_float * nl)()
    bwd = (C.c_float * nl)()
    for _ in range(2):  # the first pass creates the sequential-backward workspaces
        net.set_batch(host_x[0], host_y[0])
        polegrad._check(net.lib, net.lib.pg_net_profile(net.ptr, fwd, bwd, nl))
        net.sync()
        solver.apply()  # consume the profiled gradients
    names = net.layer_names()
    prof = {names[i]: {"fwd_ms": float(fwd[i]), "bwd_ms": float(bwd[i])} for i in range(nl)}

    # graphs: resident-input step (value) and host-buffer step (e2e)
    use_graph = not args.no_graph
    pin_x = cudadnn.PinnedBuffer((BATCH,) + IMG, npd)
    pin_y = cudadnn.PinnedBuffer((BATCH,), npd)
    pin_loss = cudadnn.PinnedBuffer((1,), npd)
    g_res = g_e2e = None
    if use_graph:
        try:
            net.set_batch(host_x[0], host_y[0])
            g_res = polegrad.StepGraph(net, solver, 0, 0, 0)
            g_e2e = polegrad.StepGraph(net, solver, pin_x.ptr, pin_y.ptr, pin_loss.ptr)
        except Exception as e:  # fall back to eager steps (reported in config)
            log(f"graph capture failed ({e}); eager steps")
            use_graph = False

    def step_resident():
        if use_graph:
            g_res.replay()
        else:
            polegrad._check(net.lib, net.lib.pg_net_forward(net.ptr))
            polegrad._check(net.lib, net.lib.pg_net_backward(net.ptr))
            solver.apply()

    # L2 flush buffer (256 MiB > 126 MB L2), written by our fill kernel
    flush_elems = 64 << 20
    flush = cx.out_h("cdnn_alloc", flush_elems, cudadnn.F32)

    def flush_l2():
        cx.call("cdnn_fill", flush, flush_elems, 0.0, 0)

    # make the resident batch current
    net.set_batch(host_x[0], host_y[0])
    for _ in range(args.warmup):
        if not use_graph:
            net.set_batch(host_x[0], host_y[0])
        step_resident()
    net.sync()

    evs = [(cx.event(), cx.event()) for _ in range(args.steps)]
    barrier()
    net.sync()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush_l2()
            cx.record(evs[i][0])
            if not use_graph:
                net.set_batch(host_x[0], host_y[0])
            step_resident()
            cx.record(evs[i][1])
        net.sync()
        barrier()
        total_ms = sum(cx.elapsed(a, b) for a, b in evs)
    clocks = clk.summary()
    total_ms = max_over_ranks(total_ms)
    value = world * BATCH * args.steps / (total_ms / 1000.0)

    # ---- e2e: host buffers through the public API (H2D in, loss D2H out, every step)
    # Graph path: polegrad.FeedRing (pinned-memory feed ring):
    # push_pinned() enqueues batch i+1's H2D from page-locked host memory on the
    # ring's copy stream while step i runs; each slot's captured step starts with a
    # device copy of its staged batch and ends with the loss D2H; pop_loss() reads
    # every step's loss.
    e_start, e_end = cx.event(), cx.event()
    if use_graph:
        ring = polegrad.FeedRing(net, solver, 2)
        # the step inputs sit in page-locked host memory (three batches cycled);
        # push_pinned enqueues each step's H2D straight from them
        npin = min(3, nb)
        pins = []
        for j in range(npin):
            px, py = cudadnn.PinnedBuffer((BATCH,) + IMG, npd), cudadnn.PinnedBuffer((BATCH,), npd)
            px.array[...] = host_x[j]
            py.array[...] = host_y[j]
            pins.append((px, py))

        def run_ring(n, sink):
            inflight = 0
            for i in range(n):
                if inflight == 2:
                    sink.append(ring.pop_loss())
                    inflight -= 1
                px, py = pins[i % npin]
                ring.push_pinned(px, py)
                inflight += 1
            while inflight:
                sink.append(ring.pop_loss())
                inflight -= 1

        def run_ring_pageable(n, sink):
            # the caller's pageable numpy batches: FeedRing.push copies each into the
            # ring's page-locked slot (host memcpy) before enqueueing its H2D
            inflight = 0
            for i in range(n):
                if inflight == 2:
                    sink.append(ring.pop_loss())
                    inflight -= 1
                ring.push(host_x[i % nb], host_y[i % nb])
                inflight += 1
            while inflight:
                sink.append(ring.pop_loss())
                inflight -= 1

        run_ring(max(2, args.warmup), [])
        net.sync()
        barrier()
        net.sync()
        losses = []
        t0 = time.perf_counter()
        cx.record(e_start)
        run_ring(args.steps, losses)
        cx.record(e_end)
        net.sync()
        wall_ms_pinned = 1000 * (time.perf_counter() - t0)
        # same through pageable host arrays (the host memcpy into the pinned slot included)
        p_start, p_end = cx.event(), cx.event()
        barrier()
        net.sync()
        cx.record(p_start)
        run_ring_pageable(args.steps, losses)
        cx.record(p_end)
        net.sync()
        pageable_ms = max_over_ranks(cx.elapsed(p_start, p_end))
    else:
        for i in range(min(args.warmup, nb)):
            pin_x.array[...] = host_x[i]
            pin_y.array[...] = host_y[i]
            net.set_batch_ptr(pin_x.ptr, pin_y.ptr)
            polegrad._check(net.lib, net.lib.pg_net_forward(net.ptr))
            polegrad._check(net.lib, net.lib.pg_net_backward(net.ptr))
            solver.apply()
            net.sync()
        barrier()
        net.sync()
        t0 = time.perf_counter()
        cx.record(e_start)
        losses = []
        for i in range(args.steps):
            pin_x.array[...] = host_x[i % nb]
            pin_y.array[...] = host_y[i % nb]
            net.set_batch_ptr(pin_x.ptr, pin_y.ptr)
            polegrad._check(net.lib, net.lib.pg_net_forward(net.ptr))
            losses.append(net.loss())
            polegrad._check(net.lib, net.lib.pg_net_backward(net.ptr))
            solver.apply()
            net.sync()
        cx.record(e_end)
        net.sync()
    e2e_ms = max_over_ranks(cx.elapsed(e_start, e_end))
    wall_ms = max_over_ranks(wall_ms_pinned if use_graph else 1000 * (time.perf_counter() - t0))
    if not use_graph:
        pageable_ms = None
    e2e = world * BATCH * args.steps / (e2e_ms / 1000.0)
    if not all(np.isfinite(losses)):
        raise RuntimeError("non-finite loss")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant layer op (largest per-layer device time)
    flops = layer_flops(net)
    pk = peaks()
    math3 = DTYPE == "f32" and os.environ.get("CDNN_MATH", "tf32x3") == "tf32x3"
    tc_peak = pk["tf32_tflops"] if DTYPE == "f32" else pk["fp64_tflops"]
    ops = []
    for lname, t in prof.items():
        for phase in ("fwd", "bwd"):
            ms = t[f"{phase}_ms"]
            f = flops.get(lname, {}).get(phase)
            ops.append((ms, lname, phase, f))
    ops.sort(reverse=True)
    dom_ms, dom_layer, dom_phase, dom_f = ops[0]
    prof_total = sum(o[0] for o in ops)
    kernel_key = f"{dom_layer}.{dom_phase}"
    if dom_f and tc_peak:
        achieved = dom_f / (dom_ms / 1000.0) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(tc_peak, 1), "unit": "TFLOP/s",
                "frac": round(achieved / tc_peak, 5), "traffic": ncu_traffic(kernel_key),
                "kernel": f"{dom_layer} {dom_phase} ("
                          + ("implicit-GEMM tcgen05, " + ("3xTF32" if math3 else "TF32") if DTYPE == "f32"
                             else "SIMT FP64") + ")",
                "flops_per_launch": dom_f, "ms_per_launch": round(dom_ms, 5),
                "share_of_step": round(dom_ms / prof_total, 4),
                "peak_note": ("dense TF32 " if DTYPE == "f32" else "dense FP64 ") + pk["tc_source"]}
        if math3:
            # 3xTF32 issues three TF32 products per multiply-add (hi*hi, hi*lo, lo*hi):
            # the tensor-core work behind the algorithmic FLOPs, against the same peak
            roof["mma_frac"] = round(3 * achieved / tc_peak, 5)
    else:
        roof = {"bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": None,
                "traffic": ncu_traffic(kernel_key), "kernel": f"{dom_layer} {dom_phase}",
                "ms_per_launch": round(dom_ms, 5), "share_of_step": round(dom_ms / prof_total, 4)}

    cpu = cpu_baseline_sample(args.cpu_iters) if not args.no_cpu_baseline else None
    esz = 8 if DTYPE == "f64" else 4
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(), "data": "synthetic",
        "config": config(world),
        "step": "cuda-graph" if use_graph else "eager",
        "e2e": {"value": round(e2e, 1), "unit": UNIT, "ms_per_step": round(e2e_ms / args.steps, 5),
                "wall_ms_per_step": round(wall_ms / args.steps, 5),
                "h2d_bytes_per_step": int(BATCH * np.prod(IMG) * esz + BATCH * esz), "d2h_bytes_per_step": esz,
                "host_copy": "each step's batch H2D from page-locked host memory (FeedRing.push_pinned) and its "
                             "loss D2H, inside the timed region",
                "pageable": None if pageable_ms is None else {
                    "value": round(world * BATCH * args.steps / (pageable_ms / 1000.0), 1),
                    "ms_per_step": round(pageable_ms / args.steps, 5),
                    "how": "FeedRing.push from pageable numpy arrays: the host memcpy into the ring's pinned "
                           "slot, the H2D and the loss D2H every step, overlapped with the step in flight"}},
        "gpu_launches": int(launches_per_step * args.steps),
        "launches_per_step": int(launches_per_step),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "nccl_ranks": nccl_ranks,
        "layer_profile_ms": prof,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------------------------
def pg_inputs(rng, n, batch, npd):
    """Cart-Pole-shaped states (acceptance.cpp:518-522 ranges), sampled actions and
    normalised returns (the modulated-gradient inputs of trainer.cpp:94-109)."""
    lo = np.array([-2.0, -3.0, -0.3, -3.0])
    st = (lo + (-2 * lo) * rng.uniform(0, 1, (n, batch, 4))).astype(npd).reshape(n, batch, 4, 1, 1)
    act = np.floor(rng.uniform(0, 1, (n, batch)) * 2).astype(npd)
    ret = rng.standard_normal((n, batch)).astype(npd)
    return st, act, ret


def run_pg_b200(args) -> None:
    """configs[2]: one policy-gradient update of the whole episode batch on the device:
    states in, forward, device-side modulated log-prob gradients at the logits
    (Net::pg_backward), backward_from, SGD.  Launch / latency
    bound (0.33 MFLOP); eager steps (the actions / returns H2D is part of the step)."""
    from paper_1810_02272_b200 import cudadnn, polegrad
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and int(os.environ.get("RANK", "0")) != 0:
        return  # the 288-byte gradient does not shard usefully: replicas only, rank 0 reports
    local = int(os.environ.get("LOCAL_RANK", "0"))
    npd = polegrad.NP_DTYPE[DTYPE]
    net = polegrad.Net(model_text(BATCH), seed=1, dtype=DTYPE, device=local)
    solver = polegrad.Solver(net, **SOLVER)
    cx = CtxView(net.context_ptr())
    rng = np.random.default_rng(2)
    nb = 3
    st, act, ret = pg_inputs(rng, nb, BATCH, npd)
    pins = []
    for j in range(nb):
        px = cudadnn.PinnedBuffer((BATCH, 4, 1, 1), npd)
        px.array[...] = st[j]
        pins.append(px)
    prob = cudadnn.PinnedBuffer((BATCH, 2), npd)

    def step(i, readback):
        # the MemoryData feed is consumed by every forward (reference FIFO semantics): the
        # episode's states are staged every step (pinned H2D)
        net.set_batch_ptr(pins[i % nb].ptr, None)
        polegrad._check(net.lib, net.lib.pg_net_forward(net.ptr))
        net.pg_backward(act[i % nb], ret[i % nb])
        solver.apply()
        if readback:  # the policy's probabilities back to the host (action sampling)
            polegrad._check(net.lib, net.lib.pg_blob_get(net.ptr, b"prob", 0, C.c_void_p(prob.ptr)))

    l0 = cx.launches()
    step(0, False)
    net.sync()
    eager_launches = cx.launches() - l0
    for i in range(args.warmup):
        step(i, False)
    net.sync()
    # the whole update captured once: H2D(states, actions, returns) -> forward -> pg diff ->
    # backward_from -> SGD -> D2H(probabilities); replayed per episode batch
    gs, ga, gr = (cudadnn.PinnedBuffer(shape, npd) for shape in ((BATCH, 4, 1, 1), (BATCH,), (BATCH,)))
    gs.array[...] = st[0]
    ga.array[...] = act[0]
    gr.array[...] = ret[0]
    lg = cx.launches()
    graph = polegrad.PGStepGraph(net, solver, gs, ga, gr, BATCH, prob)
    launches = cx.launches() - lg  # kernels per replay (1 when the update is the fused MLP kernel)
    for _ in range(args.warmup):
        graph.replay()
    net.sync()
    out = {}
    for key in ("value", "e2e"):
        a, b = cx.event(), cx.event()
        net.sync()
        t0 = time.perf_counter()
        with ClockSampler(local) as clk:
            cx.record(a)
            for i in range(args.steps):
                if key == "e2e":  # the caller's next episode (host arrays) into the pinned inputs
                    gs.array[...] = st[i % nb]
                    ga.array[...] = act[i % nb]
                    gr.array[...] = ret[i % nb]
                graph.replay()
                if key == "e2e":
                    net.sync()  # the probabilities are needed on the host before the next episode
            cx.record(b)
            net.sync()
        out[key] = (cx.elapsed(a, b), 1000 * (time.perf_counter() - t0))
        if key == "value":
            clocks = clk.summary()
    value = BATCH * args.steps / (out["value"][0] / 1000.0)
    e2e = BATCH * args.steps / (out["e2e"][0] / 1000.0)
    cpu = cpu_baseline_sample(args.cpu_iters * 50) if not args.no_cpu_baseline else None
    esz = 8 if DTYPE == "f64" else 4
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "states/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(out["value"][0] / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(), "data": "synthetic",
        "config": config(1),
        "step": ("cuda-graph of ONE kernel (cdnn_mlp_pg_step: forward, softmax gradient, backward, solver) "
                 if graph.fused else "cuda-graph of the layer-by-layer update ")
                + "(launch-bound: 0.33 MFLOP per step; the 24 KB of inputs H2D and the 8 KB of probabilities D2H "
                  "are inside the graph)",
        "eager_launches_per_step": int(eager_launches),
        "e2e": {"value": round(e2e, 1), "unit": "states/s", "ms_per_step": round(out["e2e"][0] / args.steps, 5),
                "wall_ms_per_step": round(out["e2e"][1] / args.steps, 5),
                "h2d_bytes_per_step": int(BATCH * 4 * esz + 2 * BATCH * esz),
                "d2h_bytes_per_step": int(BATCH * 2 * esz)},
        "gpu_launches": int(launches * args.steps), "launches_per_step": int(launches),
        "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                     "kernel": "launch-bound (BASELINE.md §5: ideal 0.04 us)"},
        "cpu_baseline": cpu, "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
def ref_batch_per_process(procs: int) -> int:
    """Images per reference step per host process: the bench batch split over the
    host cores, capped by the workload's bounded-sample size (AlexNet: one image per
    core per step, ~1.6 s; a whole batch-256 step would take ~7 min per core)."""
    return max(1, min(-(-BATCH // procs), REF_SAMPLE_BATCH))


def _ref_worker(args_tuple):
    steps, warmup, seed, nb = args_tuple
    return ref_steps(nb, steps, warmup, seed)


def run_reference(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import pyoracle
    if not pyoracle.available(DTYPE):
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref/liboracle_{DTYPE}.so not built"}))
        return
    pyoracle.load(DTYPE)  # mapped in this (parent) process too, before the workers fork
    import multiprocessing as mp
    procs = max(1, os.cpu_count() or 1)
    nb = ref_batch_per_process(procs)
    steps = max(args.steps, 1)
    with mp.get_context("fork").Pool(procs) as pool:
        times = pool.map(_ref_worker, [(steps, args.warmup, 2 + i, nb) for i in range(procs)])
    t = max(times)
    value = procs * nb * steps / t
    sample = (f"{procs} single-threaded processes (one per host core: the reference has no threads), each step "
              f"{procs} x {nb} = {procs * nb} images of the batch-{BATCH} {WORKLOAD} step"
              + (" (the whole bench batch)" if procs * nb >= BATCH else " (bounded sample; CPU cost is linear in batch)")
              + f", {args.warmup} warm-up + {steps} timed SGD iterations, slowest process timed; oracle/_ref: "
              f"unmodified reference core + reference-style conv/pool/loss extension, {DTYPE}")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "states/s" if WORKLOAD == "pg_mlp" else UNIT,
        "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": round(1000 * t / steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic", "impl": "reference",
        "config": config(world),
        "cpu_baseline": {"value": round(value, 3), "unit": "states/s" if WORKLOAD == "pg_mlp" else UNIT,
                         "cores": procs, "kind": "reference",
                         "sample": sample, **host_cpu()},
        "e2e": {"value": round(value, 3), "unit": "states/s" if WORKLOAD == "pg_mlp" else UNIT,
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def respawn_under_torchrun(args) -> None:
    """`bench.py --gpus N` without a launcher: re-execute under torch.distributed.run,
    one rank per GPU, so N > 1 never silently measures one rank."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("launching", " ".join(cmd))
    os.execv(sys.executable, cmd)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-graph", action="store_true", help="eager steps instead of the captured CUDA graph")
    ap.add_argument("--dp-transport", choices=["nccl", "host"], default="nccl",
                    help="N > 1 gradient exchange: NCCL (product), or the Parallel host transport over gloo "
                         "(validation of the multi-rank path with several ranks on one GPU; eager steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD,
                    help="BASELINE.json config to run (default: AlexNet b256, configs[3])")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32",
                    help="the library's real type (f32: 3xTF32 tensor cores; f64: SIMT FP64)")
    args = ap.parse_args()
    select_workload(args.workload)
    global DTYPE
    DTYPE = args.dtype
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(args)
    if args.warmup < 3 and args.impl == "b200":
        log("note: timing rules ask for >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    elif WORKLOAD == "pg_mlp":
        run_pg_b200(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
