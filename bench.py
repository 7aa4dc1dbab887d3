#!/usr/bin/env python
"""Benchmark of the merged-CG hot path (BASELINE.json metric: CG DoF*iterations/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one fixed-iteration merged Jacobi-PCG solve (`--iters`, default 200)
of the Q5 Poisson problem on a Cartesian mesh (BASELINE.json configs[1], top rung
116^3 cells ~ 1.96e8 DoFs at N=1; configs[4] weak scaling 80^3 cells per GPU for
N>1).  Inputs are seeded synthetic data (uniform[-1,1] RHS, seed 0), stated in
the JSON line.  `value` times K solves with b and x resident in HBM; `e2e` times
the same K solves through the public API `solve("combined_pcg", op, b_host, ...)`
with pinned host buffers (H2D of b and D2H of x inside the timed region).

N > 1: one process per GPU (torchrun; `--gpus N` without torchrun re-launches itself
under it), z-slabs of BASELINE configs[4]: `--scaling weak` (default) 80^3 cells per
GPU, `--scaling strong` 160^3 cells in total.

`--impl reference` times the CPU implementation of the same path (the oracle
port of the pure-Python reference; `oracle/_ref` cannot exist because the
reference has no compiled sources) on the host cores on a bounded sample of the
SAME mesh: a few merged-PCG iterations instead of the full count.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
for _p in (ROOT, ROOT / "oracle"):
    if str(_p) not in sys.path:
        sys.path.insert(0, str(_p))

import numpy as np  # noqa: E402

METRIC = "merged Jacobi-PCG throughput (n_dofs x CG iterations / s)"
UNIT = "DoF*it/s"
BYTES_PER_DOF_IT = 64.0  # r,p,v read+write, Minv read, x every 2nd iteration, fp64


def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_problem(cells, p, deform=0.0, components=1):
    from paper_2205_08909_b200 import dofs, mesh as pmesh
    mesh = pmesh.build_cartesian_mesh(cells)
    if deform:
        mesh = pmesh.deform_mesh(mesh, deform)
    h = dofs.distribute_dofs(mesh, p, components, constrain_boundary=True)
    plan = dofs.make_batches(mesh, dofs.batch_size(p, components, 8), "morton")
    return mesh, h, plan


def seeded_rhs(h, out=None):
    b = np.random.default_rng(0).uniform(-1.0, 1.0, h.n_dofs)
    b[h.constrained_dofs] = 0.0
    if out is not None:
        out[:] = b
        return out
    return b


class CpuPort:
    """The oracle port of the reference's merged Jacobi-PCG on the host cores: the C/pthreads
    restatement (oracle/mfcg_oracle.c) when it builds, else the NumPy one.  Set up once,
    timed per call."""

    def __init__(self, cells, p):
        import mfcg_oracle as orc
        self.orc = orc
        mesh, h, plan = build_problem(cells, p)
        self.n_dofs = h.n_dofs
        self.b = seeded_rhs(h)
        self.prob = orc.Problem(tuple(cells), mesh.extents, 0.0, p, p + 1, h.cell_index_blocks,
                                h.constrained_dofs, h.n_dofs)
        self.minv = orc.inverse_diagonal_affine(self.prob)  # closed form, pinned to inverse_diagonal in tests
        self.cp = None
        self.cores = 1
        self.note = "NumPy restatement (oracle/mfcg_oracle.py)"
        try:
            import mfcg_oracle_c as oc
            if oc.available():
                self.cp = oc.CProblem(self.prob)
                self.cores = oc.max_threads()
                self.note = "C/pthreads restatement (oracle/mfcg_oracle.c)"
                self.cp.apply(self.b)
        except ImportError:
            pass

    def seconds(self, iters):
        t0 = time.perf_counter()
        if self.cp is not None:
            self.cp.combined_pcg(self.b, self.minv, iters)
        else:
            self.orc.combined_pcg(lambda v: self.orc.apply(self.prob, v), self.b, self.minv,
                                  fixed_iterations=iters)
        return time.perf_counter() - t0


def reference_package_config1():
    """the reference package itself (pure Python / NumPy, sequential) on BASELINE
    configs[0] -- 8^3 cells Q4, 100 fixed iterations -- when /root/reference is present (the authoring container);
    the GPU box has no copy of it, and the entry says so."""
    src = Path("/root/reference/pkg/src")
    if not src.exists():
        return {"available": False, "note": "/root/reference does not exist on this box; measured in the authoring "
                                            "container: profiles/r02_reference_package_config1.json"}
    sys.path.insert(0, str(src))
    from mfcg.dofs import batch_size, distribute_dofs, make_batches
    from mfcg.mesh import GeometryVariant, build_cartesian_mesh
    from mfcg.operator import MatrixFreeOperator, OperatorSpec
    from mfcg.solvers import SolverConfig, solve
    mesh = build_cartesian_mesh((8, 8, 8))
    h = distribute_dofs(mesh, 4, 1, constrain_boundary=True)
    plan = make_batches(mesh, batch_size(4, 1, 8), "morton")
    op = MatrixFreeOperator(OperatorSpec("laplace", 1, 4, 5, GeometryVariant.AFFINE, "gauss"), mesh, h, plan)
    minv = op.compute_diagonal()
    b = np.random.default_rng(0).uniform(-1, 1, h.n_dofs)
    b[h.constrained_dofs] = 0.0
    out = {"available": True, "config": "BASELINE configs[0]: 8^3 cells Q4, 35937 DoFs, 100 fixed iterations, one core"}
    for variant in ("pcg", "combined_pcg"):
        best = 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            res = solve(variant, op, b, minv=minv, config=SolverConfig(fixed_iterations=100))
            best = min(best, time.perf_counter() - t0)
        out[variant] = {"seconds": best, "DoF_it_per_s": h.n_dofs * 100 / best, "residual": res.residual}
    return out


def run_reference(args, rank):
    """The reference arm: the CPU port of the reference's merged Jacobi-PCG on the host cores, on the
    SAME mesh as the GPU arm (BASELINE configs[1] top rung at N = 1), for `--ref-iters` iterations per
    step instead of the GPU arm's `--iters` (DoF*it/s does not depend on the iteration count)."""
    if rank != 0:
        return
    cells = tuple(args.ref_cells_xyz) if args.ref_cells_xyz else workload_cells(args, 1)
    t0 = time.perf_counter()
    port = CpuPort(cells, args.degree)
    setup = time.perf_counter() - t0
    times = [port.seconds(args.ref_iters) for _ in range(args.warmup + args.steps)][args.warmup:]
    total = sum(times)
    value = port.n_dofs * args.ref_iters * len(times) / total
    sample = (f"{cells[0]}x{cells[1]}x{cells[2]} cells Q{args.degree} ({port.n_dofs} DoFs), {args.ref_iters} merged-PCG "
              f"iterations per step of the same seeded problem; {port.note}; {port.cores} threads; "
              f"setup {setup:.0f} s (not timed)")
    cfg = workload_config(args, 1, cells=cells, iters=args.ref_iters)
    cfg["bounded_sample"] = (f"{args.ref_iters} iterations per step instead of {args.iters}: same mesh, same "
                             f"operator, same right-hand side")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (uniform[-1,1] RHS, seed 0)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": port.cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "reference_package_config1": reference_package_config1(),
    }
    print(json.dumps(line))


def workload_cells(args, n_gpus):
    if args.cells:
        return tuple(args.cells)
    if n_gpus == 1:
        return (116, 116, 116)
    if args.scaling == "strong":
        return (160, 160, 160)
    return (80, 80, 80 * n_gpus)


def workload_config(args, n_gpus, cells=None, iters=None):
    cells = tuple(cells) if cells else workload_cells(args, n_gpus)
    iters = iters or args.iters
    n_dofs = int(np.prod([c * args.degree + 1 for c in cells])) * args.components
    if args.cells:
        which = "custom"
    elif n_gpus == 1:
        which = "BASELINE configs[1] top rung"
    elif args.scaling == "strong":
        which = "BASELINE configs[4] strong scaling, 160^3 cells in z-slabs"
    else:
        which = "BASELINE configs[4] weak scaling, 80^3 cells per GPU in z-slabs"
    return {"workload": f"Q{args.degree} {'Poisson' if args.components == 1 else '3-component Laplace (BP4 type)'}, Cartesian {cells[0]}x{cells[1]}x{cells[2]} cells, "
                        f"{n_dofs} DoFs, fp64, Jacobi, seeded uniform[-1,1] RHS, {iters} merged-CG "
                        f"iterations per step ({which})",
            "cells": list(cells), "degree": args.degree, "n_dofs": n_dofs, "iterations_per_step": iters,
            "variant": args.variant, "geometry": args.geometry, "deformation": args.deform, "l2": "inputs larger than L2 (each vector >> 126 MB); no flush needed",
            "parallelism": "1 GPU" if n_gpus == 1 else f"z-slabs x{n_gpus}"}


def run_slabs(args, rank, local_rank, world):
    """N > 1: BASELINE configs[4] weak scaling -- 80^3 cells per GPU stacked in z, one process per
    GPU, shared lattice planes exchanged with ncclSend/ncclRecv, seven sums per iteration through
    one ncclAllReduce.  No data-path collective beyond those two."""
    import torch
    import torch.distributed as dist
    from paper_2205_08909_b200 import _lib, dofs, mesh as pmesh, slabs
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    from paper_2205_08909_b200.solvers import SolverConfig
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line only
    dist.init_process_group("nccl", rank=rank, world_size=world)
    p = args.degree
    cells = workload_cells(args, world)
    gmesh = pmesh.build_cartesian_mesh(cells)
    z0, nzg = slabs.slab_layers(cells[2], world)[rank]
    nc = args.components
    slab = slabs.build_slab(gmesh, p, z0, nzg, components=nc)
    plan = dofs.make_batches(slab.mesh, dofs.batch_size(p, nc, 8), "morton")
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(slabs.new_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    slabs.init_comm(local_rank, bytes(uid.cpu().numpy().tobytes()), rank, world)
    op = MatrixFreeOperator(OperatorSpec("laplace", nc, p, p + 1, pmesh.GeometryVariant.AFFINE), slab.mesh,
                            slab.handler, plan, device=local_rank, precision=args.precision,
                            brick=tuple(args.brick), slab_z0=z0, global_cells_z=cells[2])
    group = slabs.SlabGroup([op])
    n_local = slab.handler.n_dofs
    n_global = int(np.prod([c * p + 1 for c in cells])) * nc
    # seeded RHS of the global problem in lattice order, restricted to the slab
    rng = np.random.default_rng(0)
    NX, NY = cells[0] * p + 1, cells[1] * p + 1
    plane = NX * NY
    rng.uniform(-1.0, 1.0, z0 * p * plane)                      # skip the lower slabs' part of the stream
    vals = rng.uniform(-1.0, 1.0, (nzg * p + 1) * plane)
    b = vals[slab.global_nodes - z0 * p * plane]
    if nc > 1:  # interleaved components: the node's value scaled per component
        b = (b[:, None] * (1.0 - 0.5 * np.arange(nc))[None, :]).ravel()
    b[slab.handler.constrained_dofs] = 0.0
    b_host = torch.from_numpy(b).pin_memory()
    b_dev = b_host.cuda()
    x_dev = torch.empty_like(b_dev)
    cfg = SolverConfig(fixed_iterations=args.iters)
    lib_stream = torch.cuda.ExternalStream(_lib.stream_handle(local_rank))

    def step():
        return group.solve(args.variant, [b_dev.data_ptr()], cfg, location=1, xs=[x_dev.data_ptr()])[0]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches = 0
    e0.record(lib_stream)
    for _ in range(args.steps):
        res = step()
        launches += res.device_stats["kernel_launches"]
    e1.record(lib_stream)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    clocks = sampler.stop()
    # end to end through SlabGroup.solve with HOST buffers: every step copies the rank's part of b from pinned
    # host memory and x back (inside the library call); wall clock between barriers, max over ranks
    x_host = torch.empty(n_local, dtype=torch.float64).pin_memory()
    group.solve(args.variant, [b_host.numpy()], cfg, outs=[x_host.numpy()])
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        group.solve(args.variant, [b_host.numpy()], cfg, outs=[x_host.numpy()])
    torch.cuda.synchronize()
    dist.barrier()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    if rank == 0:
        value = n_global * args.iters * args.steps / (ms_total * 1e-3)
        peak, peak_src = measured_peak()
        info = op.info()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (uniform[-1,1] RHS, seed 0, constrained entries zeroed)",
            "config": workload_config(args, world),
            "roofline": {"bound": "hbm", "kernel": "whole merged iteration, all GPUs",
                         "achieved": value * BYTES_PER_DOF_IT / 1e9, "peak": peak * world, "unit": "GB/s",
                         "frac": value * BYTES_PER_DOF_IT / 1e9 / (peak * world), "peak_source": peak_src,
                         "traffic": None},
            "cpu_baseline": None,
            "e2e": {"value": n_global * args.iters * args.steps / t_e2e, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * n_local * world, "d2h_bytes_per_step": 8 * n_local * world,
                    "ms_per_step": 1e3 * t_e2e / args.steps,
                    "timer": "host wall clock between barriers around K SlabGroup.solve calls with pinned host "
                             "buffers, max over ranks"},
            "gpu_launches": int(launches), "clocks": clocks,
            "extra": {"final_relative_residual": res.residual, "dofs_per_gpu": n_local,
                      "plane_bytes_per_exchange": 8 * plane * nc, "bricks_per_gpu": info["n_bricks"],
                      "timer": "CUDA events on each rank's library stream, max over ranks"},
        }
        print(json.dumps(line))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, nargs=3, default=None)
    ap.add_argument("--degree", type=int, default=5)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--variant", default="combined_pcg")
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--brick", type=int, nargs=3, default=(0, 0, 0))
    ap.add_argument("--geometry", default="affine",
                    choices=["affine", "final_tensor_load", "inverse_jacobian_load", "quadratic_compute"])
    ap.add_argument("--deform", type=float, default=0.0)
    ap.add_argument("--components", type=int, default=1, choices=[1, 3],
                    help="3: vector Laplacian of the BP4 type (SURVEY.md 8f row 3); single GPU only")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = 80^3 cells per GPU, strong = 160^3 cells in total (BASELINE configs[4])")
    ap.add_argument("--ref-cells-xyz", type=int, nargs=3, default=None,
                    help="reference arm / cpu_baseline mesh (default: the GPU arm's mesh)")
    ap.add_argument("--ref-iters", type=int, default=2,
                    help="merged-PCG iterations per step of the CPU port (bounded sample of the same workload)")
    ap.add_argument("--cpu-baseline-cells", type=int, default=48,
                    help="edge of the cube the cpu_baseline leg of the GPU arm times (bounded sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the N > 1 code path (slab group, NCCL communicator, all-reduce) with one rank: a "
                         "one-GPU check of everything but the cross-rank transfers")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a B200: the hot path has no CPU fallback")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: re-launch under it, one rank per GPU
        if torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but only {torch.cuda.device_count()} GPU(s) are visible")
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / transport lines on stderr
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                   "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]])
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE {world}")
    torch.cuda.set_device(local_rank)
    if world > 1 or args.force_slabs:
        if world == 1:  # stand-alone rendezvous for the one-rank check
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        run_slabs(args, rank, local_rank, world)
        return
    from paper_2205_08909_b200 import _lib
    from paper_2205_08909_b200.mesh import GeometryVariant
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    from paper_2205_08909_b200.solvers import SolverConfig, solve, solve_device

    p = args.degree
    cells = workload_cells(args, 1)
    t_setup = time.perf_counter()
    mesh, h, plan = build_problem(cells, p, args.deform, args.components)
    op = MatrixFreeOperator(OperatorSpec("laplace", args.components, p, p + 1, GeometryVariant(args.geometry)), mesh, h, plan,
                            device=local_rank, precision=args.precision, brick=tuple(args.brick))
    info = op.info()
    n = h.n_dofs
    minv = op.compute_diagonal()
    b_host = torch.empty(n, dtype=torch.float64).pin_memory()
    x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    seeded_rhs(h, b_host.numpy())
    b_dev = b_host.cuda()
    x_dev = torch.empty_like(b_dev)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    cfg = SolverConfig(fixed_iterations=args.iters)
    lib_stream = torch.cuda.ExternalStream(_lib.stream_handle(local_rank))

    def step_dev(timed=False):
        return solve_device(args.variant, op, b_dev.data_ptr(), x_dev.data_ptr(), minv=minv, config=cfg,
                            time_kernels=timed)

    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches = 0
    e0.record(lib_stream)
    for _ in range(args.steps):
        res = step_dev()
        launches += res.device_stats["kernel_launches"]
    e1.record(lib_stream)
    torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    clocks = sampler.stop()
    value = n * args.iters * args.steps / (ms_total * 1e-3)
    residual = res.residual

    # dominant kernel, timed per launch with CUDA events on the library stream
    rt = step_dev(timed=True)
    op_ms = rt.device_stats["operator_ms"] / max(rt.device_stats["operator_launches"], 1)
    nc = args.components                        # one brick-kernel launch per component field
    n_int, n_sh = info["n_interior"], n // nc - info["n_interior"]
    w = 8 if args.precision == "fp64" else 4
    kernel_bytes = 8 * w * n_int + 2 * w * n_sh  # interior: the full 8 scalars; shared: read p, add to v
    kernel_bytes += info["geometry_bytes"]      # stored geometry streamed once per operator application
    kernel_bytes *= nc
    peak, peak_src = measured_peak()
    achieved = kernel_bytes / (op_ms * 1e-3) / 1e9
    it_ms = rt.device_stats["solve_ms"] / args.iters
    roofline = {
        "bound": "hbm", "kernel": (f"k_brick2<{p},{'double' if w == 8 else 'float'}> (persistent, cp.async.bulk fed)" if info["threads"] == 512
                                   else f"k_brick<{p},{'double' if w == 8 else 'float'},merged>"),
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
        "traffic": None, "algorithmic_bytes_per_launch": kernel_bytes, "kernel_ms": op_ms,
        "iteration_ms": it_ms, "kernel_share_of_step": op_ms / it_ms,
        "iteration_frac": (8 * w * n + nc * info["geometry_bytes"]) / (it_ms * 1e-3) / 1e9 / peak,
        "whole_solve_frac": value * 8 * w / 1e9 / peak,
    }
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            # ncu capture of the same kernel at the bench workload (116^3 cells; tools/gpu_traffic116.sh); DRAM bytes
            # per DoF are size independent above L2, so other sizes scale the per-DoF figure
            tj = json.loads(prof.read_text())
            if args.geometry == "affine" and args.degree == 5 and args.precision == "fp64" and nc == 1:
                roofline["traffic"] = tj["bytes_per_dof"] * n
                roofline["traffic_source"] = ("from_profile (not measured in this run): profiles/traffic.json, " + tj["source"]
                                              + f"; {tj['workload']}, bytes per DoF scaled by n_dofs")
        except Exception:
            pass

    # end to end through the public API: pinned host b in, pinned host x out, every step
    for _ in range(1):
        solve(args.variant, op, b_host.numpy(), minv=minv, config=cfg, out=x_host.numpy())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_launches = 0
    for _ in range(args.steps):
        r2 = solve(args.variant, op, b_host.numpy(), minv=minv, config=cfg, out=x_host.numpy())
        e2e_launches += r2.device_stats["kernel_launches"]
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t0
    e2e = {"value": n * args.iters * args.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n + 32 * args.iters, "ms_per_step": 1e3 * t_e2e / args.steps,
           "timer": "host wall clock around K public-API solves, synchronised both sides"}

    cpu = None
    if not args.no_cpu_baseline:
        nref = args.cpu_baseline_cells
        port = CpuPort((nref, nref, nref), p)
        its = max(args.ref_iters, 20)
        secs = port.seconds(its)
        cpu = {"value": port.n_dofs * its / secs, "unit": UNIT, "cores": port.cores, "kind": "port",
               "sample": f"{nref}^3 cells Q{p} ({port.n_dofs} DoFs), {its} merged-PCG iterations in {secs:.1f} s "
                         f"(bounded sample of the same problem family; `--impl reference` times the full mesh); "
                         f"{port.note}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if w == 8 else "f32",
        "data": "synthetic (uniform[-1,1] RHS, seed 0, constrained entries zeroed)",
        "config": workload_config(args, 1), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches), "clocks": clocks,
        "extra": {"final_relative_residual": residual, "bricks": info["n_bricks"], "brick": info["brick"],
                  "interior_fraction": n_int / n, "setup_seconds": t_setup,
                  "timer": "CUDA events on the library stream around K device-resident solves"},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
