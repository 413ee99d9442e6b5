"""Benchmark of the recursive corrective-motion pipeline on B200 (driver contract).

Default workload (BASELINE.json configs[3], the north star's target scene,
SURVEY.md §8d cfg3): two corotational 5-tet blocks of 50 x 50 x 30 nodes at
1 cm (450 000 DoF; the literal 50x50x20 gives 300 000), lower
block E=1e4 on a ground plane, upper block E=2e3 sliding at 0.5 m/s, nu=0.4,
mu=0.4, ~7 500 contact groups (upper vertices vs lower triangles, lower
vertices vs upper triangles, lower vertices vs ground), 10 forced fast-scheme
iterations, PGS 30 sweeps / tol 1e-6 (reference default budget, §9 #14).

One STEP = one whole Simulation.step() of that scene (GPU detection,
corotational assembly + supernodal Cholesky of both bodies, free motion,
W_g = sum_o S_o A_o^-1 S_o^T, 10 x [relinearise, W = D W_g D^T, violation,
PGS, proximity update], mechanical correction, integration, signed gaps).
The upper block starts half a cell off the lower grid and 1 mm above it; the
simulation is pre-rolled CFG3_PREROLL steps (block sliding, contacts
established) and every timed step replays the next step from that state
(consecutive steps do not reach a steady state: see Cfg3Workload).

Reported: value = ms per step (device-timed, inputs resident; the step's
working set of ~32 GB exceeds L2 many times over), ms per Newton iteration,
per-phase medians, e2e through the public API with host buffers (the same
step with the state uploaded from pinned memory and read back every step), the roofline of the dominant kernel (PGS: HBM bytes
of W per sweep) plus the factor and W_g fp64 tensor-core rooflines, and the
CPU baseline: the reference package itself on a bounded, extrapolated sample
(bench_reference.py, run in a separate process that never loads this repo's
library).

``--impl reference`` runs the reference arm (bench_reference.py): the
unmodified reference package on the host cores, plus one MEASURED (not
extrapolated) whole cfg1 step of the reference.  ``--workload cfg1|cfg4``
select BASELINE configs[1] / configs[4].  ``--gpus N`` (N > 1) re-launches
itself under torch.distributed.run with N ranks (one per GPU; fails loudly
if fewer GPUs are visible).
"""

from __future__ import annotations

import argparse
import contextlib
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

H = workloads.H
N_CONTACTS = workloads.CFG1_CONTACTS
N_REDRAW = workloads.CFG1_REDRAWS
CFG3_NXZ, CFG3_NZ = workloads.CFG3_NXZ, workloads.CFG3_NY
CFG3_PREROLL = 2
CFG3_SHIFT, CFG3_GAP = 0.005, 0.001  # upper block half a cell off the lower grid, 1 mm above it
# contact groups and PGS sweeps per Newton iteration of the GPU arm at the timed
# steps (B200 runs of this bench); the reference arm runs before the GPU arm, so
# its PGS extrapolation takes them from here (the GPU arm's own cpu_baseline
# passes the values it just measured)
CFG3_GROUPS = 7500
CFG3_SWEEPS_PER_ITER = 16.1  # profiles/r02_bench_cfg3.json: 161 sweeps over 10 iterations at the timed step
CFG4_COPIES = workloads.CFG4_COPIES
CFG4_PREROLL = 12
METRIC_CFG3 = ("ms per full time step (cfg3 450k-DoF two-body scene); also ms per Newton constraint-update "
               "iteration")
METRIC_CFG1 = "ms per full step (cfg1 compliance-update pipeline); also ms per Newton constraint-update iteration"
METRIC_CFG4 = "scene-steps per second (cfg4: 1024 independent cfg0 beam copies, 5 corrective iterations)"


# ----------------------------------------------------------------------------
# workload construction (GPU arm)
# ----------------------------------------------------------------------------

def make_inputs():
    return workloads.cfg1_inputs()


def make_pairs(cn, inp):
    nodes, tris = inp["nodes"], inp["tris"]
    pairs = []
    for i in range(N_CONTACTS):
        tri = tris[inp["tri_idx"][i]]
        w = inp["weights"][i]
        p = w @ nodes[tri]
        pairs.append(cn.ProximityPair(
            object_a=0, object_b=1,
            attach_a=cn.Attachment(cn.AttachKind.BARYCENTRIC, 0, triangle=tri.copy(), weights=w.copy()),
            attach_b=cn.Attachment(cn.AttachKind.WORLD, 1, world_point=p.copy()),
            p_a=p.copy(), p_b=p.copy(), ref_normal=np.array([0.0, 1.0, 0.0]), signed_distance=0.0,
            vertex_id=i, element_id=int(inp["tri_idx"][i])))
    return pairs


def make_cfg3_config(cn, nxz=CFG3_NXZ, ny=CFG3_NZ, material="corotational", shift=0.0, gap=0.0):
    (ln, lt), (un, ut) = workloads.cfg3_meshes(nxz, ny, shift, gap)
    objs = [cn.SoftSpec(name="lower", mesh=cn.TetMesh(ln, lt), young=1e4, poisson=0.4, density=1000.0,
                        material=material),
            cn.SoftSpec(name="upper", mesh=cn.TetMesh(un, ut), young=2e3, poisson=0.4, density=1000.0,
                        velocity=(0.5, 0.0, 0.0), material=material),
            cn.PlaneSpec(name="ground", normal=(0.0, 1.0, 0.0), offset=0.0)]
    return cn.SceneConfig(objects=objs, h=H, threshold=0.005,
                          pgs=cn.PgsConfig(max_iterations=30, tolerance=1e-6, friction=0.4),
                          newton=cn.NewtonConfig(scheme="fast", max_iterations=10, penetration_tol=-1.0,
                                                 rotation_tol=-1.0),
                          output=cn.OutputConfig(snapshots=False, metrics=False))


class GpuWorkload:
    """cfg1: factorisation + W_g once, then 10 frame re-draws (rebuild W, dx)."""

    def __init__(self, inp):
        import torch

        import paper_2306_06946_b200 as cn
        from paper_2306_06946_b200 import _lib

        self.cn, self.torch, self._lib = cn, torch, _lib
        self.inp = inp
        # the reference material (linear): the reference runs cfg1 as-is
        self.body = cn.SoftBody(cn.TetMesh(inp["nodes"], inp["tets"]), young=5e3, poisson=0.45, density=1000.0,
                                rayleigh_mass=0.0, rayleigh_stiffness=0.0, material="linear")
        self.state = self.body.initial_state()
        self.pairs = make_pairs(cn, inp)
        self.S = cn.build_signed_mapping(self.pairs, 0, self.body.n_dofs, self.body.fixed_mask)
        A, _ = self.body.assemble(self.state, H, (0.0, -9.81, 0.0))
        self.F = cn.Factorization(A)
        dev = torch.device("cuda")
        self.Ds = [torch.as_tensor(D, device=dev) for D in inp["Ds"]]
        self.lams = [torch.as_tensor(l, device=dev) for l in inp["lams"]]
        m = 3 * N_CONTACTS
        self.W = torch.empty((m, m), dtype=torch.float64, device=dev)
        self.t = torch.empty(m, dtype=torch.float64, device=dev)
        self.dx = torch.empty((N_REDRAW, self.body.n_dofs), dtype=torch.float64, device=dev)
        self.rhs = torch.empty(self.body.n_dofs, dtype=torch.float64, device=dev)
        self.wg = None
        self.q_host = torch.as_tensor(inp["nodes"].reshape(-1).copy()).pin_memory()
        self.dx_host = torch.empty((N_REDRAW, self.body.n_dofs), dtype=torch.float64).pin_memory()
        self.phase_events = None

    def step(self, q=None, record=False):
        """One full step: assemble, refactor, W_g, 10 x (W_k, dx_k)."""
        cn, torch, _lib = self.cn, self.torch, self._lib
        st = self.state if q is None else cn.MechanicalState(q, self.state.v)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if record else None
        if record:
            ev[0].record()
        A, _ = self.body.assemble(st, H, (0.0, -9.81, 0.0))
        if record:
            ev[1].record()
        self.F.refactor_async(A.values)
        if record:
            ev[2].record()
        self.wg = cn.assemble_Wg({0: self.S}, {0: self.F})
        if record:
            ev[3].record()
        m = N_CONTACTS
        stream = _lib.stream()
        for k in range(N_REDRAW):
            D = self.Ds[k]
            _lib.call("cnb_rebuild_w", m, D.data_ptr(), self.wg.wg.data_ptr(), 3 * m, self.W.data_ptr(), 3 * m, stream)
            _lib.call("cnb_apply_dt", m, D.data_ptr(), self.lams[k].data_ptr(), self.t.data_ptr(), None, stream)
            self.S.rmatvec(self.t, out=self.rhs, alpha=H)
            self.F.solve_device(self.rhs.reshape(1, -1), out=self.dx[k].reshape(1, -1))
        if record:
            ev[4].record()
            self.phase_events = ev
        return self.dx

    def step_e2e(self):
        """Public-API step with host buffers: H2D of the positions, D2H of every dx."""
        q = self.q_host.to("cuda", non_blocking=True)
        dx = self.step(q=q)
        self.dx_host.copy_(dx, non_blocking=True)
        return self.dx_host

    def phase_ms(self):
        ev = self.phase_events
        self.torch.cuda.synchronize()
        names = ["assemble", "factor", "build_wg", "newton_iters"]
        return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}


class Cfg3Workload:
    """cfg3 through the public Simulation API.

    The scene is run CFG3_PREROLL steps (the upper block sliding, contacts
    established), and every timed step replays the next step from that state:
    consecutive steps are not a steady state here, since the BASELINE scene
    degenerates after a few steps (the E = 2 kPa upper block collapses under its
    own weight while sliding; the reference algorithm does the same at reduced
    size), with the contact count growing 2x and PGS capped."""

    name = "cfg3"

    def __init__(self, preroll=CFG3_PREROLL):
        import torch

        import paper_2306_06946_b200 as cn

        self.cn, self.torch = cn, torch
        self.config = make_cfg3_config(cn, shift=CFG3_SHIFT, gap=CFG3_GAP)
        self.sim = cn.Simulation(self.config)
        self.preroll_reports = [self.sim.step() for _ in range(preroll)]
        objs = self.sim.dynamic_objects
        self.q0 = {o.oid: o.state.q.clone() for o in objs}
        self.v0 = {o.oid: o.state.v.clone() for o in objs}
        self.snap = (self.sim.time, self.sim.step_index)
        self.q_host = {o.oid: o.state.q.cpu().pin_memory() for o in objs}
        self.v_host = {o.oid: o.state.v.cpu().pin_memory() for o in objs}
        self.q_out = {o.oid: torch.empty(o.state.q.shape, dtype=torch.float64).pin_memory() for o in objs}
        self.v_out = {o.oid: torch.empty(o.state.v.shape, dtype=torch.float64).pin_memory() for o in objs}
        self.last = None

    def _restore(self, q, v):
        for o in self.sim.dynamic_objects:
            o.state = self.cn.MechanicalState(q[o.oid], v[o.oid])
        self.sim.time, self.sim.step_index = self.snap

    def step(self):
        self._restore({k: t.clone() for k, t in self.q0.items()}, {k: t.clone() for k, t in self.v0.items()})
        self.last = self.sim.step()
        return self.last

    def step_e2e(self):
        """The same step with the state uploaded from pinned host memory and the
        new state read back."""
        torch = self.torch
        self._restore({k: t.to("cuda", non_blocking=True) for k, t in self.q_host.items()},
                      {k: t.to("cuda", non_blocking=True) for k, t in self.v_host.items()})
        rep = self.sim.step()
        for o in self.sim.dynamic_objects:
            self.q_out[o.oid].copy_(o.state.q, non_blocking=True)
            self.v_out[o.oid].copy_(o.state.v, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return rep

    def phases(self, rep):
        return {"detect": rep.t_detect * 1e3, "assemble_factor": rep.t_assemble * 1e3, "free": rep.t_free * 1e3,
                "constraints": rep.t_constraints * 1e3, "build_wg": rep.t_build_wg * 1e3,
                "rebuild_w": rep.t_rebuild_w * 1e3, "pgs": rep.t_pgs * 1e3, "prox_update": rep.t_correction * 1e3,
                "final_correction": rep.t_final_correction * 1e3}

    @property
    def h2d_bytes(self):
        return int(sum(t.numel() for t in self.q_host.values()) * 16)

    @property
    def d2h_bytes(self):
        return int(sum(t.numel() for t in self.q_out.values()) * 16)

    def kernel_rooflines(self, dmma, hbm):
        """Factor and W_g at the timed step's state, timed alone with CUDA events."""
        torch = self.torch
        from paper_2306_06946_b200.wg import object_compliance

        self._restore({k: t.clone() for k, t in self.q0.items()}, {k: t.clone() for k, t in self.v0.items()})
        out = {}
        fac_ms, fac_fl = 0.0, 0.0
        for o in self.sim.dynamic_objects:
            A, _ = o.body.assemble(o.state, self.config.h, self.config.gravity)
            F = o.factorization
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            F.refactor_async(A.values)
            e1.record()
            torch.cuda.synchronize()
            fac_ms += e0.elapsed_time(e1)
            fac_fl += F.flops
        ach = fac_fl / (fac_ms * 1e-3) / 1e12
        out["factor"] = {"kernel": "supernodal Cholesky (2 bodies)", "bound": "tensor", "achieved": round(ach, 3),
                         "peak": round(dmma, 2), "unit": "TFLOP/s", "frac": round(ach / dmma, 4),
                         "algorithmic_gflop": round(fac_fl / 1e9, 1), "ms": round(fac_ms, 3)}
        ctx = self.sim.prepare_step(build_wg=False)[0]
        st = {}
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for oid in sorted(ctx.S_by_object):
            object_compliance(ctx.S_by_object[oid], ctx.F_by_object[oid], 3 * len(ctx.pairs), stats=st, shard=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        fl = st.get("fwd_flops", 0.0) + st.get("gram_flops", 0.0)
        ach = fl / (ms * 1e-3) / 1e12
        out["build_wg"] = {"kernel": "W_g: sparse-RHS forward solve + Gram (2 bodies)", "bound": "tensor",
                           "achieved": round(ach, 3), "peak": round(dmma, 2), "unit": "TFLOP/s",
                           "frac": round(ach / dmma, 4), "algorithmic_gflop": round(fl / 1e9, 1), "ms": round(ms, 3),
                           "fwd_gflop": round(st.get("fwd_flops", 0.0) / 1e9, 1),
                           "gram_gflop": round(st.get("gram_flops", 0.0) / 1e9, 1)}
        return out

    def config_json(self, world, steps):
        return {"workload": "cfg3: two corotational 5-tet blocks 50x50x30 nodes (450000 DoF), ground plane, "
                            "10 fast-scheme iterations, PGS 30 sweeps tol 1e-6",
                "dofs": self.sim.total_dofs(), "contacts": self.last.c_groups if self.last else None,
                "newton_iterations": 10, "pgs_budget": "30 sweeps, tol 1e-6",
                "upper_block_placement": f"shifted {CFG3_SHIFT} m in x and z, {CFG3_GAP} m above the lower block "
                                         "(no coincident nodes across the interface)",
                "timed_steps": f"step {CFG3_PREROLL} of the running simulation (upper block sliding), replayed from "
                               f"its start state every timed step",
                "preroll": [{"pairs": r.c_groups, "sweeps": r.pgs_iterations_total, "pen_after": r.pen_after}
                            for r in self.preroll_reports],
                "parallelism": (f"dp{world}: factor replicated, W_g right-hand-side columns split per rank "
                                f"(forward solve + Gram rows), NCCL all-gathers of Y and C; Newton loop replicated"
                                if world > 1 else "single"),
                "l2": "working set ~32 GB per step >> 126 MB L2 (no flush needed)"}


# ----------------------------------------------------------------------------
# measurement helpers
# ----------------------------------------------------------------------------

def flush_l2(torch, buf):
    buf.add_(1.0)  # 512 MiB read+write > 126 MB L2


@contextlib.contextmanager
def _no_gc():
    """Timed regions run with Python's cyclic collector paused (collected just
    before): a collection pause inside one step is host jitter, not the path."""
    gc.collect()
    gc.disable()
    try:
        yield
    finally:
        gc.enable()


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        if os.environ.get("CNB_BENCH_NO_CLOCKS") == "1":  # diagnostic: timing without the sampler
            return self
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
            # nvidia-smi's start-up (NVML initialisation) stays outside the timed
            # region: wait for its first sample
            t_end = time.time() + 3.0
            while time.time() < t_end and self.proc.poll() is None and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self, gpu_index=0):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.proc is None or not os.path.exists(self.path):
            return out
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(gpu_index):
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower() == "active":
                    reasons.add(nm)
        if sm:
            out["sm_mhz"] = statistics.median(sm)
            out["sm_max_mhz"] = mx
            out["reasons"] = sorted(reasons)
            out["samples"] = len(sm)
        return out


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def dmma_peak_tflops(torch, _lib):
    """fp64 MMA (DMMA) peak of this GPU, measured with the library's microbenchmark."""
    import ctypes

    out = (ctypes.c_double * 1)()
    _lib.call("cnb_bench_dmma", 4096, out, _lib.stream())
    return float(out[0])


def _max_over_ranks(torch, world, *vals):
    if world == 1:
        return vals
    t = torch.tensor(vals, device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return tuple(float(x) for x in t)


def reference_subprocess(workload, extra=()):
    """Run the reference arm in a fresh interpreter (it never loads this repo's
    library) and return its JSON line, or an error dict."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
           "--steps", "1", "--warmup", "0", "--quick", *extra]
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        for line in reversed(res.stdout.strip().splitlines()):
            if line.startswith("{"):
                return json.loads(line)
        return {"error": (res.stderr or res.stdout)[-400:]}
    except Exception as exc:  # the baseline is reported, never required
        return {"error": repr(exc)}


# ----------------------------------------------------------------------------
# GPU arm: cfg1
# ----------------------------------------------------------------------------

def run_gpu_cfg1(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    wl = GpuWorkload(make_inputs())
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        wl.step(record=True)
        flush_l2(torch, flush)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    phases = []
    with ClockSampler() as clk, _no_gc():
        torch.cuda.synchronize()
        launches0 = _lib.lib().cnb_launch_count()
        for i in range(args.steps):
            starts[i].record()
            wl.step(record=True)
            ends[i].record()
            phases.append(wl.phase_ms())
            flush_l2(torch, flush)
        torch.cuda.synchronize()
        launches = _lib.lib().cnb_launch_count() - launches0
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    for _ in range(max(1, args.warmup // 2)):
        wl.step_e2e()
    torch.cuda.synchronize()
    with _no_gc():
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wl.step_e2e()
            torch.cuda.current_stream().synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    roof = roofline_cfg1(wl, torch, _lib, phases)
    total_ms, e2e_ms = _max_over_ranks(torch, world, total_ms, e2e_ms)
    ms_step = total_ms / args.steps
    med = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    return {
        "metric": METRIC_CFG1,
        "value": round(ms_step, 4), "unit": "ms/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1], workloads.cfg1_inputs)",
        "config": {"workload": "cfg1: 40x10x10-node 5-tet grid (12000 DoF, reference linear material), "
                               "500 barycentric contacts, 10 frame re-draws", "dofs": wl.body.n_dofs,
                   "contacts": N_CONTACTS, "redraws": N_REDRAW,
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": "flushed between steps (512 MiB write)"},
        "ms_per_newton_iter": round(med["newton_iters"] / N_REDRAW, 5),
        "phases_ms_median": {k: round(v, 4) for k, v in med.items()},
        "factor": {"nnz_L": wl.F.nnz_L, "supernodes": wl.F.n_supernodes, "levels": wl.F.n_levels,
                   "gflop": round(wl.F.flops / 1e9, 3)},
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms/step", "h2d_bytes_per_step": int(wl.q_host.numel() * 8),
                "d2h_bytes_per_step": int(wl.dx_host.numel() * 8)},
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk.summary(int(os.environ.get("LOCAL_RANK", 0))),
    }


def roofline_cfg1(wl, torch, _lib, phases):
    """Dominant phase of the cfg1 step against its bound."""
    med = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    peaks, src = measured_peaks()
    dom = max(med, key=med.get)
    dmma = dmma_peak_tflops(torch, _lib)
    dsrc = "fp64 DMMA microbenchmark measured in this run (not in MEASURED_PEAKS.json)"
    if dom == "build_wg":
        st = {}
        from paper_2306_06946_b200.wg import object_compliance

        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        object_compliance(wl.S, wl.F, 3 * N_CONTACTS, stats=st, shard=False)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        flops = st["fwd_flops"] + st["gram_flops"]
        ach = flops / (ms * 1e-3) / 1e12
        return {"kernel": "W_g build (panel_mma_kernel sparse forward + gram_kernel)", "bound": "tensor",
                "achieved": round(ach, 3), "peak": round(dmma, 2), "unit": "TFLOP/s", "frac": round(ach / dmma, 4),
                "traffic": None, "peak_source": dsrc, "algorithmic_gflop": round(flops / 1e9, 4), "ms": round(ms, 4)}
    if dom == "factor":
        ach = wl.F.flops / (med["factor"] * 1e-3) / 1e12
        return {"kernel": "numeric Cholesky (extend-add/potrf/trsm/syrk)", "bound": "tensor",
                "achieved": round(ach, 3), "peak": round(dmma, 2), "unit": "TFLOP/s", "frac": round(ach / dmma, 4),
                "traffic": None, "peak_source": dsrc, "algorithmic_gflop": round(wl.F.flops / 1e9, 4),
                "ms": round(med["factor"], 4)}
    if dom == "newton_iters":
        m = 3 * N_CONTACTS
        bytes_it = 16.0 * m * m + 24.0 * wl.F.nnz_L + 8.0 * 4 * wl.body.n_dofs
        ms_it = med["newton_iters"] / N_REDRAW
        ach = bytes_it / (ms_it * 1e-3) / 1e9
        return {"kernel": "Newton iteration (rebuild W + S^T t + solve)", "bound": "hbm", "achieved": round(ach, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None,
                "peak_source": src, "algorithmic_bytes": bytes_it, "ms": round(ms_it, 5)}
    bytes_as = 1440.0 * wl.body.mesh.n_tets
    ach = bytes_as / (med["assemble"] * 1e-3) / 1e9
    return {"kernel": "FE assembly", "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None, "peak_source": src,
            "ms": round(med["assemble"], 4)}


# ----------------------------------------------------------------------------
# GPU arm: cfg3 (default)
# ----------------------------------------------------------------------------

def pgs_ncu_traffic_per_sweep():
    """dram__bytes_read + dram__bytes_write of the largest pgs_pipe_kernel launch of a
    cfg3 step from the committed ncu --set full capture (profiles/
    r02_ncu_dmma_and_pgs_kernels.txt), per W pass: that launch ran the 30-sweep cap
    (7 301 groups) and forms delta_end without a pass, so 30 passes."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_dmma_and_pgs_kernels.txt")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        vals, inside = {}, False
        for line in open(path):
            if line.startswith("== "):
                inside = line.startswith("== pgs_pipe_kernel")
            elif inside and " = " in line:
                k, rest = line.strip().split(" = ", 1)
                parts = rest.split()
                if len(parts) >= 2 and parts[1] in scale:
                    vals[k] = float(parts[0]) * scale[parts[1]]
        return round((vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) / 30.0, 0)
    except (OSError, KeyError, ValueError):
        return None


def run_gpu_cfg3(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    wl = Cfg3Workload()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    reps = []
    with ClockSampler() as clk, _no_gc():
        torch.cuda.synchronize()
        launches0 = _lib.lib().cnb_launch_count()
        for i in range(args.steps):
            starts[i].record()
            reps.append(wl.step())
            ends[i].record()
        torch.cuda.synchronize()
        launches = _lib.lib().cnb_launch_count() - launches0
    if world > 1:
        torch.distributed.barrier()
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    total_ms = sum(step_ms)
    # e2e: the same step through pinned host buffers
    torch.cuda.synchronize()
    with _no_gc():
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wl.step_e2e()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    total_ms, e2e_ms = _max_over_ranks(torch, world, total_ms, e2e_ms)
    ms_step = total_ms / args.steps
    ph = [wl.phases(r) for r in reps]
    med = {k: round(statistics.median(p_[k] for p_ in ph), 3) for k in ph[0]}
    iters = reps[-1].newton_iterations
    newton_ms = statistics.median((r.t_rebuild_w + r.t_pgs + r.t_correction) * 1e3 / max(r.newton_iterations, 1)
                                  for r in reps)
    # dominant kernel: PGS (HBM: W read once per sweep, plus the delta_end pass per iteration)
    peaks, src = measured_peaks()
    groups = [r.c_groups for r in reps]
    sweeps = [r.pgs_iterations_total for r in reps]
    pgs_s = sum(r.t_pgs for r in reps)
    # one pass over W per sweep; delta_end needs none (formed from the proximity update)
    passes = sum(sweeps)
    bytes_pass = [8.0 * (3 * g) ** 2 for g in groups]
    alg = sum(b * s for b, s in zip(bytes_pass, sweeps))
    ach = alg / pgs_s / 1e9
    roof = {"kernel": "pgs_pipe_kernel (exact-order projected Gauss-Seidel, dense W, lookahead-2 pipeline)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": pgs_ncu_traffic_per_sweep(),
            "traffic_unit": "bytes per W pass (ncu --set full dram read+write)", "peak_source": src,
            "algorithmic_bytes_per_pass": bytes_pass[-1],
            "passes": "one W pass per sweep (delta_end is formed from the proximity update, no pass)",
            "passes_per_step_mean": round(passes / len(reps), 2),
            "ms_per_pass": round(pgs_s * 1e3 / max(passes, 1), 4)}
    dmma = dmma_peak_tflops(torch, _lib)
    others = wl.kernel_rooflines(dmma, peaks["hbm_gbs"])
    c = 3 * groups[-1]
    rb_s = reps[-1].t_rebuild_w / max(iters, 1)
    others["rebuild_w"] = {"kernel": "rebuild_w_kernel (W = D W_g D^T, bit-exact order)", "bound": "hbm",
                           "achieved": round(16.0 * c * c / rb_s / 1e9, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": round(16.0 * c * c / rb_s / 1e9 / peaks["hbm_gbs"], 4),
                           "ms": round(rb_s * 1e3, 4)}
    line = {
        "metric": METRIC_CFG3,
        "value": round(ms_step, 3), "unit": "ms/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded meshes of BASELINE configs[3], workloads.cfg3_meshes)",
        "config": wl.config_json(world, args.steps),
        "ms_per_newton_iter": round(newton_ms, 4),
        "step_ms_each": [round(x, 2) for x in step_ms],
        "phases_ms_median": med,
        "contacts": groups, "pgs_sweeps_per_step": sweeps,
        "pgs_sweeps_per_iter_mean": round(sum(sweeps) / sum(r.newton_iterations for r in reps), 2),
        "factor": {"nnz_L": [o.factorization.nnz_L for o in wl.sim.dynamic_objects],
                   "gflop": [round(o.factorization.flops / 1e9, 1) for o in wl.sim.dynamic_objects]},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms/step", "h2d_bytes_per_step": wl.h2d_bytes,
                "d2h_bytes_per_step": wl.d2h_bytes},
        "roofline": roof,
        "rooflines_other": others,
        "gpu_launches": int(launches),
        "clocks": clk.summary(int(os.environ.get("LOCAL_RANK", 0))),
    }
    if rank == 0 and not args.no_cfg1_pair:
        # the GPU side of the measured cfg1 pair (the reference arm times the reference's whole cfg1 step)
        sub = argparse.Namespace(steps=5, warmup=3)
        c1 = run_gpu_cfg1(sub, rank, 1) if world == 1 else None
        if c1:
            line["cfg1_pair"] = {"gpu_ms_per_step": c1["value"], "gpu_e2e_ms_per_step": c1["e2e"]["value"],
                                 "gpu_ms_per_newton_iter": c1["ms_per_newton_iter"],
                                 "reference": "bench.py --impl reference reports cfg1_measured (whole reference "
                                              "cfg1 step, timed, not extrapolated)"}
    return line


# ----------------------------------------------------------------------------
# GPU arm: cfg4 (batched independent scenes)
# ----------------------------------------------------------------------------

def cfg4_copy_range(rank, world, total=CFG4_COPIES):
    per = (total + world - 1) // world
    a = min(total, rank * per)
    return a, min(total, a + per)


class Cfg4Workload:
    """1024 copies of the cfg0 beam, this rank's share."""

    def __init__(self, rank, world, total=CFG4_COPIES):
        import torch

        from paper_2306_06946_b200.batch import BatchedPlaneScenes, cfg4_draws
        from paper_2306_06946_b200.mesh import five_tet_grid

        self.first, last = cfg4_copy_range(rank, world, total)
        self.ns = last - self.first
        self.mesh = five_tet_grid(workloads.CFG0_SHAPE, 0.01)
        tilts, mus, jit = cfg4_draws(self.first, self.ns, self.mesh.nodes.size)
        self.B = BatchedPlaneScenes(self.mesh, tilts, mus, jit, threshold=0.005, clearance=0.02,
                                    newton_iterations=5, pgs_tolerance=1e-10, pgs_max_iterations=1000)
        n = self.B.n
        self.q_host = torch.empty((self.ns, n), dtype=torch.float64).pin_memory()
        self.v_host = torch.empty((self.ns, n), dtype=torch.float64).pin_memory()
        self.pairs = 0

    def step(self):
        self.pairs = self.B.step()
        return self.pairs

    def snapshot(self):
        self.q_host.copy_(self.B.Q)
        self.v_host.copy_(self.B.V)

    def step_e2e(self):
        """Public API with host buffers: state uploaded from pinned memory, one time
        step of every copy, the new state read back into the same host buffers (the
        next step's input)."""
        import torch

        B = self.B
        B.Q.copy_(self.q_host, non_blocking=True)
        B.V.copy_(self.v_host, non_blocking=True)
        self.pairs = B.step()
        self.q_host.copy_(B.Q, non_blocking=True)
        self.v_host.copy_(B.V, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    @property
    def h2d_bytes(self):
        return int(2 * self.q_host.numel() * 8)

    @property
    def d2h_bytes(self):
        return int(2 * self.q_host.numel() * 8)


def cfg4_ncu_traffic_last_launch():
    p = os.path.join(ROOT, "profiles", "r01_cfg4_pgs_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh)["launches"][-1]["dram_bytes"]
    except (OSError, KeyError, IndexError, ValueError):
        return None


class _PgsBatchTimer:
    """CUDA events around the batched PGS launches of a step (wrapping the library
    call so the step code stays the product path)."""

    def __init__(self, torch):
        self.torch = torch
        self.recs = []
        self.cur = []

    def __enter__(self):
        from paper_2306_06946_b200 import _lib

        self._orig = _lib.call
        torch = self.torch
        cur = self.cur = []

        def call(name, *a):
            if name == "cnb_pgs_batched":
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r = self._orig(name, *a)
                e1.record()
                cur.append((e0, e1))
                return r
            return self._orig(name, *a)

        _lib.call = call
        import paper_2306_06946_b200.batch as bmod

        bmod._lib.call = call
        return self

    def __exit__(self, *a):
        from paper_2306_06946_b200 import _lib

        _lib.call = self._orig
        self.recs.append(self.cur)

    def pgs_ms_last_iter(self):
        self.torch.cuda.synchronize()
        if not self.recs or not self.recs[-1]:
            return 0.0
        e0, e1 = self.recs[-1][-1]
        return e0.elapsed_time(e1)

    def phases(self):
        self.torch.cuda.synchronize()
        per = [sum(a.elapsed_time(b) for a, b in r) for r in self.recs if r]
        return {"pgs_ms_per_step_median": round(statistics.median(per), 3) if per else 0.0}


def run_gpu_cfg4(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    wl = Cfg4Workload(rank, world)
    for _ in range(max(CFG4_PREROLL - args.warmup, 0) + args.warmup):
        wl.step()
    wl.B.check()
    wl.snapshot()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    pairs = []
    prof = _PgsBatchTimer(torch)
    with ClockSampler() as clk, _no_gc():
        torch.cuda.synchronize()
        launches0 = _lib.lib().cnb_launch_count()
        for i in range(args.steps):
            starts[i].record()
            with prof:
                pairs.append(wl.step())
            ends[i].record()
        torch.cuda.synchronize()
        launches = _lib.lib().cnb_launch_count() - launches0
    wl.B.check()
    sweeps = int(wl.B.last["iters"][:, 0].sum()) if wl.B.last else 0
    if world > 1:
        torch.distributed.barrier()
    total_ms = sum(s_.elapsed_time(e_) for s_, e_ in zip(starts, ends))
    torch.cuda.synchronize()
    with _no_gc():
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wl.step_e2e()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    total_ms, e2e_ms = _max_over_ranks(torch, world, total_ms, e2e_ms)
    ms_step = total_ms / args.steps
    peaks, src = measured_peaks()
    P = wl.B.last["pairs"] if wl.B.last else None
    it_h = wl.B.last["iters"].cpu().numpy() if wl.B.last else np.zeros((0, 2), dtype=np.int32)
    cnt = P["cnt"] if P is not None else np.zeros(0)
    pgs_bytes = float(sum(8.0 * (3 * c) ** 2 * int(k) for c, k in zip(cnt, it_h[:, 0])))
    pgs_ms = prof.pgs_ms_last_iter()
    ach = pgs_bytes / (pgs_ms * 1e-3) / 1e9 if pgs_ms > 0 else 0.0
    roof = {"kernel": "pgs_copy_kernel (one CTA per copy, exact-order projected Gauss-Seidel, dense W)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": cfg4_ncu_traffic_last_launch(), "peak_source": src,
            "traffic_unit": "dram bytes of the last Newton iteration's launch (profiles/r01_cfg4_pgs_traffic.json)",
            "algorithmic_bytes_per_launch": pgs_bytes, "ms_per_launch": round(pgs_ms, 4),
            "launch": "last Newton iteration of the last timed step"}
    return {
        "metric": METRIC_CFG4,
        "value": round(CFG4_COPIES * args.steps / (total_ms * 1e-3), 1), "unit": "scene-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded per-copy tilt, mu, jitter: np.random.default_rng([4, i]))",
        "config": {"workload": "cfg4: 1024 copies of the cfg0 beam (20x4x4-node 5-tet grid, 960 DoF, linear, "
                               "E=5e3 nu=0.45), plane tilt U(0,20) deg, mu U(0.2,0.8), threshold 0.005, 5 forced "
                               "fast-scheme iterations, PGS tol 1e-10 / 1000 sweeps",
                   "copies": CFG4_COPIES, "copies_per_rank": wl.ns,
                   "timed_steps": f"{CFG4_PREROLL}..{CFG4_PREROLL + args.steps - 1}",
                   "parallelism": f"scene-parallel over {world} GPU(s), no data-path collective",
                   "l2": "not flushed; per-step working set (W of all copies ~0.5 GB) exceeds L2"},
        "step_ms_each": [round(s_.elapsed_time(e_), 2) for s_, e_ in zip(starts, ends)],
        "contacts_per_copy_mean": round(float(np.mean(cnt)) if len(cnt) else 0.0, 1),
        "contacts_total": int(pairs[-1]) if pairs else 0,
        "pgs_sweeps_last_iter_max": int(it_h[:, 0].max()) if len(it_h) else 0,
        "pgs_sweeps_last_iter_total": sweeps,
        "phases_ms": prof.phases(),
        "e2e": {"value": round(wl.ns * world / (e2e_ms * 1e-3), 1), "unit": "scene-steps/s",
                "h2d_bytes_per_step": wl.h2d_bytes, "d2h_bytes_per_step": wl.d2h_bytes},
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk.summary(int(os.environ.get("LOCAL_RANK", 0))),
    }


# ----------------------------------------------------------------------------
# reference arm (bench_reference.py: the reference package only)
# ----------------------------------------------------------------------------

def _ref_common(args, metric, unit, workload, data):
    return {"metric": metric, "unit": unit, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": unit != "ms/step", "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": data, "config": {"workload": workload}, "impl": "reference"}


def run_reference(args):
    import bench_reference as br

    host = br.host_info()
    if args.workload == "cfg4":
        steps = max(1, min(args.steps, 3))
        v, procs, secs = br.cfg4_throughput(steps=steps)
        line = _ref_common(args, METRIC_CFG4, "scene-steps/s", "cfg4: 1024 copies of the cfg0 beam, sampled on "
                           "the host cores", "synthetic (seeded per-copy tilt, mu, jitter)")
        sample = (f"reference Simulation per process, {procs} processes x 1 thread, copy i in process i, pre-rolled "
                  f"{br.CFG4_PREROLL} steps then {steps} timed step(s); throughput = sum 1/t_step")
        line.update(value=round(v, 3), ms_per_step=round(CFG4_COPIES / v * 1e3, 1),
                    cpu_baseline={"value": round(v, 3), "unit": "scene-steps/s", "cores": procs,
                                  "kind": "reference", "sample": sample,
                                  "s_per_step_median": round(statistics.median(secs), 3), **host},
                    e2e={"value": round(v, 3), "unit": "scene-steps/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        return line
    if args.workload == "cfg1":
        line = _ref_common(args, METRIC_CFG1, "ms/step", "cfg1: 40x10x10-node 5-tet grid (12000 DoF), 500 "
                           "barycentric contacts, 10 frame re-draws", "synthetic (seeded, BASELINE configs[1])")
        if args.quick:
            s, redraw = br.cfg1_quick_step()
            sample = "whole cfg1 step with one of the 10 identical re-draws timed and counted 10 times"
            it = redraw
        else:
            s, ph = br.cfg1_full_step()
            sample = "one whole cfg1 step, timed end to end (not extrapolated)"
            it = ph["newton_iter_s"]
            line["phases_s"] = {k: round(v, 4) for k, v in ph.items()}
        line.update(value=round(s * 1e3, 2), ms_per_step=round(s * 1e3, 2), ms_per_newton_iter=round(it * 1e3, 2),
                    steps_run=1,
                    cpu_baseline={"value": round(s * 1e3, 2), "unit": "ms/step", "cores": host["blas_threads"],
                                  "kind": "reference", "sample": sample, **host},
                    e2e={"value": round(s * 1e3, 2), "unit": "ms/step", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        return line
    groups = args.groups or CFG3_GROUPS
    sweeps = args.sweeps or CFG3_SWEEPS_PER_ITER
    sampler = br.Cfg3Sampler(groups=groups, sweeps_per_iter=sweeps)
    for _ in range(min(args.warmup, 1)):
        sampler.step()
    vals, its, det = [], [], None
    for _ in range(max(1, args.steps)):
        v, det = sampler.step()
        vals.append(v)
        its.append(det["newton_iter_s"])
    v = statistics.median(vals)
    line = _ref_common(args, METRIC_CFG3, "ms/step", "cfg3: two 5-tet blocks 50x50x30 nodes (450000 DoF), ground "
                       "plane, 10 fast-scheme iterations, PGS 30 sweeps tol 1e-6 (reference: linear material)",
                       "synthetic (seeded meshes of BASELINE configs[3])")
    line.update(value=round(v * 1e3, 1), ms_per_step=round(v * 1e3, 1),
                ms_per_newton_iter=round(statistics.median(its) * 1e3, 1), extrapolated=True,
                same_config=False,
                same_config_note="the reference has only the linear material (factorised once per simulation); "
                                 "the GPU arm runs the corotational material and refactorises every step",
                cpu_baseline={"value": round(v * 1e3, 1), "unit": "ms/step", "cores": host["blas_threads"],
                              "kind": "reference", "extrapolated": True, "sample": br.sample_description(sampler),
                              "detail_s": {k: (round(x, 4) if isinstance(x, float) else x) for k, x in det.items()},
                              "setup_s": round(sampler.setup_s, 2), **host},
                e2e={"value": round(v * 1e3, 1), "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    if not args.quick:
        # the measured pair: one whole reference cfg1 step, as-is and with BLAS for the rebuild
        s, ph = br.cfg1_full_step()
        sb, phb = br.cfg1_full_step(blas_rebuild=True)
        line["cfg1_measured"] = {
            "ms_per_step": round(s * 1e3, 1), "ms_per_newton_iter": round(ph["newton_iter_s"] * 1e3, 2),
            "phases_s": {k: round(x, 4) for k, x in ph.items()}, "extrapolated": False, "same_config": True,
            "note": "one whole BASELINE configs[1] step of the unmodified reference (linear material, as the GPU "
                    "arm's cfg1), timed end to end",
            "reference_plus_blas_gemm_ms_per_step": round(sb * 1e3, 1),
            "reference_plus_blas_gemm_note": "NOT the reference: the same step with W_k = D W_g D^T by numpy BLAS"}
    return line


# ----------------------------------------------------------------------------
# driver
# ----------------------------------------------------------------------------

def spawn_ranks(args):
    """--gpus N without a launcher: re-run under torch.distributed.run, one rank per GPU."""
    import socket

    try:
        import torch

        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if args.impl == "ours" and have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible; one rank per GPU "
                         "is required (ranks are never stacked on one GPU)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg1", "cfg4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg1-pair", action="store_true", help="cfg3: skip the GPU side of the cfg1 pair")
    ap.add_argument("--quick", action="store_true", help="reference arm: cpu_baseline-sized sample only")
    ap.add_argument("--groups", type=int, default=0, help="reference arm, cfg3: contact groups")
    ap.add_argument("--sweeps", type=float, default=0.0, help="reference arm, cfg3: PGS sweeps per iteration")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    import torch

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    line = {"cfg3": run_gpu_cfg3, "cfg4": run_gpu_cfg4}.get(args.workload, run_gpu_cfg1)(args, rank, world)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            extra = []
            if args.workload == "cfg3":
                extra = ["--groups", str(line["contacts"][-1]), "--sweeps", str(line["pgs_sweeps_per_iter_mean"])]
            ref = reference_subprocess(args.workload, extra)
            cb = ref.get("cpu_baseline") if isinstance(ref, dict) else None
            line["cpu_baseline"] = cb if cb else {"value": None, "error": ref.get("error", "no output")}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
