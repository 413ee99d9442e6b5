"""Benchmark of the recursive corrective-motion pipeline on B200 (driver contract).

Default workload (BASELINE.json configs[3], the north star's target scene,
SURVEY.md §8d cfg3): two corotational 5-tet blocks of 50 x 50 x 30 nodes at
1 cm (450 000 DoF; the literal 50x50x20 gives 300 000), lower
block E=1e4 on a ground plane, upper block E=2e3 sliding at 0.5 m/s, nu=0.4,
mu=0.4, ~7 500 contact groups (upper vertices vs lower triangles, lower
vertices vs upper triangles, lower vertices vs ground), 10 forced fast-scheme
iterations, PGS 30 sweeps / tol 1e-6 (reference default budget, §9 #14).

One STEP = one whole Simulation.step() of that scene from its initial state
(GPU detection, corotational assembly + supernodal Cholesky of both bodies,
free motion, W_g = sum_o S_o A_o^-1 S_o^T, 10 x [relinearise, W = D W_g D^T,
violation, PGS, proximity update], mechanical correction, integration,
signed gaps).  Every timed step restarts from the same initial state so all
steps see the same contact set (the scene's later steps differ only in data).

Reported: value = ms per step (device-timed, inputs resident, the step's own
working set of ~32 GB exceeds L2 many times over), ms per Newton iteration,
per-phase medians, e2e through the public API with host buffers (state
uploaded from pinned memory, final state read back every step), the roofline
of the dominant kernel (PGS: HBM bytes of W per sweep) plus the factor and
W_g fp64 tensor-core rooflines, CPU baseline (oracle port of the reference,
sampled + extrapolated, see cpu_reference_sample_cfg3).

``--workload cfg1`` runs BASELINE configs[1] (isolated compliance-update
bench).  N>1 (torchrun): every rank runs the scene, the W_g Gram tiles are
split round-robin across ranks and summed with one NCCL all-reduce
(DESIGN.md §7); value = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H = 0.01
SHAPE = (40, 10, 10)
N_CONTACTS = 500
N_REDRAW = 10


# ----------------------------------------------------------------------------
# workload (host inputs, shared by both arms)
# ----------------------------------------------------------------------------

def make_inputs():
    from paper_2306_06946_b200.mesh import five_tet_grid, surface_triangles

    mesh = five_tet_grid(SHAPE, 0.01)
    tris = surface_triangles(mesh)
    rng = np.random.default_rng(1)
    tri_idx = rng.integers(0, len(tris), N_CONTACTS)
    weights = rng.dirichlet((1.0, 1.0, 1.0), N_CONTACTS)
    rng = np.random.default_rng(2)
    frames = np.zeros((N_CONTACTS, 3, 3))
    for i in range(N_CONTACTS):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        t1 = np.cross(n, rng.standard_normal(3))
        t1 /= np.linalg.norm(t1)
        frames[i] = np.stack([n, t1, np.cross(n, t1)])
    rng = np.random.default_rng(3)
    Ds = []
    cur = frames
    ang = np.deg2rad(5.0)
    for _ in range(N_REDRAW):
        ax = rng.standard_normal((N_CONTACTS, 3))
        ax /= np.linalg.norm(ax, axis=1, keepdims=True)
        K = np.zeros((N_CONTACTS, 3, 3))
        K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -ax[:, 2], ax[:, 1], -ax[:, 0]
        K = K - K.transpose(0, 2, 1)
        R = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * (K @ K)
        # rows of a frame are the directions: rotate each row vector
        cur = np.einsum("gij,gkj->gki", R, cur)
        Ds.append(cur.copy())
    lams = [np.random.default_rng(4 + k).uniform(0.0, 1.0, 3 * N_CONTACTS) for k in range(N_REDRAW)]
    return dict(mesh=mesh, tris=tris, tri_idx=tri_idx, weights=weights, Ds=Ds, lams=lams)


def make_pairs(cn, inp):
    mesh, tris = inp["mesh"], inp["tris"]
    pairs = []
    for i in range(N_CONTACTS):
        tri = tris[inp["tri_idx"][i]]
        w = inp["weights"][i]
        p = w @ mesh.nodes[tri]
        pairs.append(cn.ProximityPair(
            object_a=0, object_b=1,
            attach_a=cn.Attachment(cn.AttachKind.BARYCENTRIC, 0, triangle=tri.copy(), weights=w.copy()),
            attach_b=cn.Attachment(cn.AttachKind.WORLD, 1, world_point=p.copy()),
            p_a=p.copy(), p_b=p.copy(), ref_normal=np.array([0.0, 1.0, 0.0]), signed_distance=0.0,
            vertex_id=i, element_id=int(inp["tri_idx"][i])))
    return pairs


# cfg3 (BASELINE configs[3]): two corotational 5-tet blocks, 50 x 50 x CFG3_NZ
# nodes at 1 cm (CFG3_NZ = 30 -> 450 000 DoF, the north star's "450k-DoF"
# figure; 50x50x20 as literally written gives 300 000), the
# lower block (E=1e4) on a ground plane, the upper block (E=2e3) resting on it
# and sliding at 0.5 m/s, nu=0.4, mu=0.4, 10 forced fast-scheme iterations,
# PGS 30 sweeps / tol 1e-6 (the reference default budget).
# Contacts: upper vertices vs lower triangles, lower vertices vs upper
# triangles, lower vertices vs the ground.
CFG3_NXZ = 50
CFG3_NZ = 30


def make_cfg3_config(cn, nxz=CFG3_NXZ, ny=CFG3_NZ):
    from paper_2306_06946_b200.mesh import five_tet_grid

    lower = five_tet_grid((nxz, ny, nxz), 0.01)
    top = float(lower.nodes[:, 1].max())
    upper = five_tet_grid((nxz, ny, nxz), 0.01, (0.0, top, 0.0))
    objs = [cn.SoftSpec(name="lower", mesh=lower, young=1e4, poisson=0.4, density=1000.0, material="corotational"),
            cn.SoftSpec(name="upper", mesh=upper, young=2e3, poisson=0.4, density=1000.0, velocity=(0.5, 0.0, 0.0),
                        material="corotational"),
            cn.PlaneSpec(name="ground", normal=(0.0, 1.0, 0.0), offset=0.0)]
    return cn.SceneConfig(objects=objs, h=H, threshold=0.005,
                          pgs=cn.PgsConfig(max_iterations=30, tolerance=1e-6, friction=0.4),
                          newton=cn.NewtonConfig(scheme="fast", max_iterations=10, penetration_tol=-1.0,
                                                 rotation_tol=-1.0),
                          output=cn.OutputConfig(snapshots=False, metrics=False))


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

class GpuWorkload:
    def __init__(self, inp):
        import torch

        import paper_2306_06946_b200 as cn
        from paper_2306_06946_b200 import _lib

        self.cn, self.torch, self._lib = cn, torch, _lib
        self.inp = inp
        mesh = inp["mesh"]
        self.body = cn.SoftBody(mesh, young=5e3, poisson=0.45, density=1000.0, rayleigh_mass=0.0,
                                rayleigh_stiffness=0.0, material="corotational")
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
        # host-side (pinned) copies for the e2e leg
        self.q_host = torch.as_tensor(mesh.nodes.reshape(-1).copy()).pin_memory()
        self.dx_host = torch.empty((N_REDRAW, self.body.n_dofs), dtype=torch.float64).pin_memory()
        self.phase_events = None

    def step(self, q=None, record=False):
        """One full step; q: device positions (defaults to the resident state)."""
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
        torch = self.torch
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
    """cfg3 through the public Simulation API, every step from the initial state."""

    name = "cfg3"

    def __init__(self):
        import torch

        import paper_2306_06946_b200 as cn

        self.cn, self.torch = cn, torch
        self.config = make_cfg3_config(cn)
        self.sim = cn.Simulation(self.config)
        self.q0 = {o.oid: o.state.q.clone() for o in self.sim.dynamic_objects}
        self.v0 = {o.oid: o.state.v.clone() for o in self.sim.dynamic_objects}
        self.t0, self.k0 = self.sim.time, self.sim.step_index
        # e2e host buffers (pinned)
        self.q_host = {k: v.cpu().pin_memory() for k, v in self.q0.items()}
        self.v_host = {k: v.cpu().pin_memory() for k, v in self.v0.items()}
        self.q_out = {k: torch.empty_like(v, device="cpu").pin_memory() for k, v in self.q0.items()}
        self.v_out = {k: torch.empty_like(v, device="cpu").pin_memory() for k, v in self.v0.items()}
        self.last = None

    def _reset(self, q=None, v=None):
        cn = self.cn
        for o in self.sim.dynamic_objects:
            qq = (q or self.q0)[o.oid]
            vv = (v or self.v0)[o.oid]
            o.state = cn.MechanicalState(qq.clone() if q is None else qq, vv.clone() if v is None else vv)
        self.sim.time, self.sim.step_index = self.t0, self.k0

    def step(self):
        self._reset()
        self.last = self.sim.step()
        return self.last

    def step_e2e(self):
        torch = self.torch
        q = {k: t.to("cuda", non_blocking=True) for k, t in self.q_host.items()}
        v = {k: t.to("cuda", non_blocking=True) for k, t in self.v_host.items()}
        self._reset(q, v)
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

    def newton_iters(self, rep):
        return rep.newton_iterations

    @property
    def h2d_bytes(self):
        return int(sum(t.numel() for t in self.q_host.values()) * 16)

    @property
    def d2h_bytes(self):
        return int(sum(t.numel() for t in self.q_out.values()) * 16)

    def kernel_rooflines(self, dmma, hbm, rep):
        """Factor and W_g of the current state, timed alone with CUDA events."""
        torch, cn = self.torch, self.cn
        from paper_2306_06946_b200.wg import object_compliance

        self._reset()
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
            object_compliance(ctx.S_by_object[oid], ctx.F_by_object[oid], 3 * len(ctx.pairs), stats=st)
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

    def config_json(self, world):
        return {"workload": "cfg3: two corotational 5-tet blocks 50x50x30 nodes (450000 DoF), ground plane, "
                            "10 fast-scheme iterations, PGS 30 sweeps tol 1e-6",
                "dofs": self.sim.total_dofs(), "contacts": self.last.c_groups if self.last else None,
                "newton_iterations": 10, "pgs_budget": "30 sweeps, tol 1e-6",
                "parallelism": (f"dp{world}: scene replicated, W_g Gram tiles sharded round-robin + NCCL all-reduce"
                                if world > 1 else "single"),
                "l2": "working set ~32 GB per step >> 126 MB L2 (no flush needed)"}


def flush_l2(torch, buf):
    buf.add_(1.0)  # 512 MiB read+write > 126 MB L2


class ClockSampler:
    def __init__(self):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
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
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def dmma_peak_tflops(torch, _lib):
    """fp64 MMA (DMMA) peak of this GPU, measured with the library's microbenchmark."""
    import ctypes

    out = (ctypes.c_double * 1)()
    _lib.call("cnb_bench_dmma", 4096, out, _lib.stream())
    return float(out[0])


def run_gpu_cfg1(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    inp = make_inputs()
    wl = GpuWorkload(inp)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        wl.step(record=True)
        flush_l2(torch, flush)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # device-timed steps (L2 flushed between steps, outside the events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    phases = []
    kstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps * N_REDRAW)]
    with ClockSampler() as clk:
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
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    # e2e: public API with host buffers
    for _ in range(max(1, args.warmup // 2)):
        wl.step_e2e()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.step_e2e()
        torch.cuda.current_stream().synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    # dominant kernel roofline
    roof = roofline(args, wl, torch, _lib, phases)
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    ms_step = total_ms / args.steps
    med = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    line = {
        "metric": "ms per full step (cfg1 compliance-update pipeline); also ms per Newton constraint-update iteration",
        "value": round(ms_step, 4), "unit": "ms/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1])",
        "config": {"workload": "cfg1: 40x10x10-node 5-tet corotational grid (12000 DoF), 500 barycentric contacts, "
                               "10 frame re-draws", "dofs": wl.body.n_dofs, "contacts": N_CONTACTS,
                   "redraws": N_REDRAW, "parallelism": (f"dp{world}: factor replicated, W_g Gram tiles sharded round-robin + NCCL all-reduce, "
                                   "Newton iterations replicated") if world > 1 else "single",
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
    return line


def run_gpu_cfg3(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    wl = Cfg3Workload()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    reps = []
    with ClockSampler() as clk:
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
    total_ms = sum(s_.elapsed_time(e_) for s_, e_ in zip(starts, ends))
    # e2e: public API with host buffers (pinned H2D of every body's q, v; D2H of the result)
    wl.step_e2e()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.step_e2e()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    ms_step = total_ms / args.steps
    ph = [wl.phases(r) for r in reps]
    med = {k: round(statistics.median(p_[k] for p_ in ph), 3) for k in ph[0]}
    iters = reps[-1].newton_iterations
    newton_ms = statistics.median((r.t_rebuild_w + r.t_pgs + r.t_correction) * 1e3 for r in reps)
    # dominant kernel: PGS (HBM: W read once per sweep)
    peaks, src = measured_peaks()
    c = 3 * reps[-1].c_groups
    sweeps = reps[-1].pgs_iterations_total
    pgs_s = reps[-1].t_pgs
    bytes_sweep = 8.0 * c * c
    ach = sweeps * bytes_sweep / pgs_s / 1e9
    roof = {"kernel": "pgs_pipe_kernel (exact-order projected Gauss-Seidel, dense W, lookahead-2 pipeline)", "bound": "hbm",
            "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
            "traffic": pgs_ncu_traffic_per_sweep(), "traffic_unit": "bytes per sweep (ncu --set full dram read+write)", "peak_source": src, "algorithmic_bytes_per_sweep": bytes_sweep, "sweeps_per_step": sweeps,
            "ms_per_sweep": round(pgs_s * 1e3 / max(sweeps, 1), 4)}
    dmma = dmma_peak_tflops(torch, _lib)
    others = wl.kernel_rooflines(dmma, peaks["hbm_gbs"], reps[-1])
    rb_s = reps[-1].t_rebuild_w / max(iters, 1)
    others["rebuild_w"] = {"kernel": "rebuild_w_kernel (W = D W_g D^T, bit-exact order)", "bound": "hbm",
                           "achieved": round(16.0 * c * c / rb_s / 1e9, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": round(16.0 * c * c / rb_s / 1e9 / peaks["hbm_gbs"], 4),
                           "ms": round(rb_s * 1e3, 4)}
    line = {
        "metric": "ms per full time step (cfg3 450k-DoF two-body scene); also ms per Newton constraint-update "
                  "iteration",
        "value": round(ms_step, 3), "unit": "ms/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded meshes of BASELINE configs[3])",
        "config": wl.config_json(world),
        "ms_per_newton_iter": round(newton_ms / max(iters, 1), 4),
        "phases_ms_median": med,
        "contacts": reps[-1].c_groups, "pgs_sweeps_per_step": sweeps,
        "factor": {"nnz_L": [o.factorization.nnz_L for o in wl.sim.dynamic_objects],
                   "gflop": [round(o.factorization.flops / 1e9, 1) for o in wl.sim.dynamic_objects]},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms/step", "h2d_bytes_per_step": wl.h2d_bytes,
                "d2h_bytes_per_step": wl.d2h_bytes},
        "roofline": roof,
        "rooflines_other": others,
        "gpu_launches": int(launches),
        "clocks": clk.summary(int(os.environ.get("LOCAL_RANK", 0))),
    }
    return line


# ----------------------------------------------------------------------------
# cfg4: batched independent scenes (BASELINE configs[4])
# ----------------------------------------------------------------------------

CFG4_COPIES = 1024
CFG4_PREROLL = 12  # steps before the timed region: copies start 2 cm above their planes, contact from step ~7


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
        self.mesh = five_tet_grid((20, 4, 4), 0.01)
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


def run_gpu_cfg4(args, rank, world):
    import torch

    from paper_2306_06946_b200 import _lib

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    wl = Cfg4Workload(rank, world)
    for _ in range(max(CFG4_PREROLL - args.warmup, 0) + args.warmup):
        wl.step()
    wl.B.check()
    wl.snapshot()  # state at the start of the timed region: e2e replays the same steps from it
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    pairs, iters = [], []
    prof = _PgsBatchTimer(torch)
    with ClockSampler() as clk:
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
    # e2e: the same steps again from the snapshot, state round-tripping through host memory
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.step_e2e()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    ms_step = total_ms / args.steps
    total = CFG4_COPIES
    peaks, src = measured_peaks()
    # dominant kernel: batched PGS, W of every copy read once per sweep (8 c_s^2 bytes)
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
    line = {
        "metric": "scene-steps per second (cfg4: 1024 independent cfg0 beam copies, 5 corrective iterations)",
        "value": round(total * args.steps / (total_ms * 1e-3), 1), "unit": "scene-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded per-copy tilt, mu, jitter: np.random.default_rng([4, i]))",
        "config": {"workload": "cfg4: 1024 copies of the cfg0 beam (20x4x4-node 5-tet grid, 960 DoF, linear, "
                               "E=5e3 nu=0.45), plane tilt U(0,20) deg, mu U(0.2,0.8), threshold 0.005, 5 forced "
                               "fast-scheme iterations, PGS tol 1e-10 / 1000 sweeps",
                   "copies": total, "copies_per_rank": wl.ns, "timed_steps": f"{CFG4_PREROLL}..{CFG4_PREROLL + args.steps - 1}",
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
    return line


def cfg4_ncu_traffic_last_launch():
    """DRAM read+write bytes of the last batched PGS launch of a cfg4 step, from the
    committed ncu launch list (tools/gpu_ncu_cfg4.sh)."""
    p = os.path.join(ROOT, "profiles", "r01_cfg4_pgs_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh)["launches"][-1]["dram_bytes"]
    except (OSError, KeyError, IndexError, ValueError):
        return None


class _PgsBatchTimer:
    """CUDA events around the batched PGS launches of a step (monkey-patched onto the
    library call so the step code stays the product path)."""

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


def _cfg4_cpu_worker(arg):
    """One process: the oracle port of the reference advancing copy i, pre-rolled to
    the timed region, then ``steps`` timed steps.  Returns seconds per step."""
    i, steps, preroll = arg
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cn_oracle as orc

    from paper_2306_06946_b200.batch import cfg4_draws, placement, plane_normals
    from paper_2306_06946_b200.mesh import five_tet_grid

    mesh = five_tet_grid((20, 4, 4), 0.01)
    tilts, mus, jit = cfg4_draws(i, 1, mesh.nodes.size)
    nrm = plane_normals(tilts)[0]
    rest = placement(mesh.nodes, plane_normals(tilts), 0.02)[0]
    body = orc.Body(rest, mesh.tets, young=5e3, poisson=0.45, density=1000.0)
    sc = orc.Scene([body], [dict(normal=nrm, offset=0.0)], threshold=0.005, mu=float(mus[0]), pgs_iter=1000,
                   pgs_tol=1e-10, newton_iter=5, penetration_tol=-1.0, rotation_tol=-1.0)
    sc.q[0] = sc.q[0] + jit[0]
    for _ in range(preroll):
        sc.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        sc.step()
    return (time.perf_counter() - t0) / steps


def cpu_reference_cfg4(steps=1, procs=None, preroll=CFG4_PREROLL):
    """Oracle port on all host cores, one process per core (one copy each), SURVEY §8d:
    scene-steps/s = sum over processes of 1 / (seconds per step)."""
    import multiprocessing as mp

    procs = procs or (os.cpu_count() or 1)
    env_keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in env_keys}
    for k in env_keys:
        os.environ[k] = "1"
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            secs = pool.map(_cfg4_cpu_worker, [(i, steps, preroll) for i in range(procs)])
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return sum(1.0 / s for s in secs), procs, secs


def run_reference_cfg4(args):
    steps = max(1, min(args.steps, 3))
    v, procs, secs = cpu_reference_cfg4(steps=steps)
    sample = (f"oracle port of the reference, {procs} processes x 1 thread, copy i = process i (cfg4 draws), "
              f"pre-rolled {CFG4_PREROLL} steps, then {steps} timed step(s) each; throughput = sum 1/t_step")
    return {"metric": "scene-steps per second (cfg4: 1024 independent cfg0 beam copies, 5 corrective iterations)",
            "value": round(v, 3), "unit": "scene-steps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(CFG4_COPIES / v * 1e3, 1), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per-copy tilt, mu, jitter: np.random.default_rng([4, i]))",
            "config": {"workload": "cfg4: 1024 copies of the cfg0 beam, sampled on the host cores"},
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 3), "unit": "scene-steps/s", "cores": procs, "kind": "port",
                             "sample": sample, "s_per_step_median": round(statistics.median(secs), 3)},
            "e2e": {"value": round(v, 3), "unit": "scene-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def pgs_ncu_traffic_per_sweep():
    """dram__bytes_read + dram__bytes_write of one pgs_pipe_kernel launch from the
    committed ncu --set full capture (profiles/), per W pass (30 sweeps + the
    delta_end pass at G = 7500, the cfg3 size)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_ncu_pgs_pipe_kernel.txt")
    try:
        vals = {}
        for line in open(path):
            if " = " in line and "[" in line:
                k, rest = line.split(" [", 1)
                unit, v = rest.split("] = ")
                scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, None)
                if scale:
                    vals[k] = float(v) * scale
        return round((vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) / 31.0, 0)
    except (OSError, KeyError, ValueError):
        return None


def roofline(args, wl, torch, _lib, phases):
    """Dominant kernel = the phase with the largest median share; report its
    algorithmic throughput against the relevant peak."""
    med = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    peaks, src = measured_peaks()
    dom = max(med, key=med.get)
    dmma = dmma_peak_tflops(torch, _lib)
    if dom == "build_wg":
        st = {}
        from paper_2306_06946_b200.wg import object_compliance

        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        object_compliance(wl.S, wl.F, 3 * N_CONTACTS, stats=st)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        flops = st["fwd_flops"] + st["gram_flops"]
        ach = flops / (ms * 1e-3) / 1e12
        return {"kernel": "W_g build (fwd_kernel sparse + gram_kernel)", "bound": "tensor", "achieved": round(ach, 3),
                "peak": round(dmma, 2), "unit": "TFLOP/s", "frac": round(ach / dmma, 4), "traffic": None,
                "peak_source": "fp64 DMMA microbenchmark measured in this run (not in MEASURED_PEAKS.json)",
                "algorithmic_gflop": round(flops / 1e9, 4), "ms": round(ms, 4)}
    if dom == "factor":
        flops = wl.F.flops
        ach = flops / (med["factor"] * 1e-3) / 1e12
        return {"kernel": "numeric Cholesky (extend-add/potrf/trsm/syrk)", "bound": "tensor", "achieved": round(ach, 3),
                "peak": round(dmma, 2), "unit": "TFLOP/s", "frac": round(ach / dmma, 4), "traffic": None,
                "peak_source": "fp64 DMMA microbenchmark measured in this run (not in MEASURED_PEAKS.json)",
                "algorithmic_gflop": round(flops / 1e9, 4), "ms": round(med["factor"], 4)}
    if dom == "newton_iters":
        # per iteration: rebuild W (16 m^2 B) + single-RHS solve (24 nnz(L) B)
        m = 3 * N_CONTACTS
        bytes_it = 16.0 * m * m + 24.0 * wl.F.nnz_L + 8.0 * 4 * wl.body.n_dofs
        ms_it = med["newton_iters"] / N_REDRAW
        ach = bytes_it / (ms_it * 1e-3) / 1e9
        return {"kernel": "Newton iteration (rebuild W + S^T t + solve)", "bound": "hbm", "achieved": round(ach, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None,
                "peak_source": src, "algorithmic_bytes": bytes_it, "ms": round(ms_it, 5)}
    # assemble
    ne = wl.body.mesh.n_tets
    bytes_as = 1440.0 * ne
    ach = bytes_as / (med["assemble"] * 1e-3) / 1e9
    return {"kernel": "corotational assembly", "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None, "peak_source": src,
            "ms": round(med["assemble"], 4)}


# ----------------------------------------------------------------------------
# CPU arms (oracle port of the reference; test infrastructure)
# ----------------------------------------------------------------------------

def cpu_reference_sample(inp, gemm_fraction=0.02):
    """Time the reference algorithm (oracle port) on a bounded sample of one step:
    assembly + SuperLU factorisation + W_g (full), one re-draw's naive-gemm
    rebuild on a fraction of its inner (rank-1) loop, scaled, and one dx.
    Returns the extrapolated ms per step and per Newton iteration."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cn_oracle as orc

    mesh = inp["mesh"]
    t0 = time.perf_counter()
    body = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, density=1000.0, alpha=0.0, beta=0.0)
    A, _ = body.system(mesh.nodes.ravel(), np.zeros(body.n), H, (0.0, -9.81, 0.0))
    F = orc.Factor(A)
    t1 = time.perf_counter()
    tris = inp["tris"]
    pairs = dict(obj_a=np.zeros(N_CONTACTS, int), obj_b=np.ones(N_CONTACTS, int),
                 kind_a=np.full(N_CONTACTS, orc.BARYCENTRIC), kind_b=np.full(N_CONTACTS, orc.WORLD),
                 vert_a=np.full(N_CONTACTS, -1))
    # side A barycentric: build S directly (constraints.py:101-120 semantics)
    rows, cols, vals = [], [], []
    for i in range(N_CONTACTS):
        tri = tris[inp["tri_idx"][i]]
        for nd, w in zip(tri, inp["weights"][i]):
            for k in range(3):
                rows.append(3 * i + k)
                cols.append(3 * nd + k)
                vals.append(w)
    import scipy.sparse as sp

    S = sp.coo_matrix((vals, (rows, cols)), shape=(3 * N_CONTACTS, body.n)).tocsr()
    wg, per = orc.mapping_compliance({0: S}, {0: F})
    t2 = time.perf_counter()
    # rebuild W: two naive gemms of m^3; time a fraction of the rank-1 loop
    D = inp["Ds"][0]
    Dd = orc.block_dense(D)
    m = Dd.shape[0]
    kk = max(1, int(gemm_fraction * m))
    out = np.zeros((m, m))
    t3 = time.perf_counter()
    for p in range(kk):
        out += Dd[:, p, None] * wg[None, p, :]
    t4 = time.perf_counter()
    rebuild_s = 2.0 * (t4 - t3) * (m / kk)
    t = orc.apply_dt(D, inp["lams"][0])
    t5 = time.perf_counter()
    H * F.solve(S.T @ t)
    t6 = time.perf_counter()
    it_s = rebuild_s + (t6 - t5)
    step_s = (t2 - t0) + N_REDRAW * it_s
    return step_s * 1e3, it_s * 1e3, (t1 - t0) * 1e3, (t2 - t1) * 1e3


def cpu_reference_sample_cfg3(budget_scale=1.0):
    """The reference algorithm (oracle port, linear material: the reference has no
    corotational model and factors once per simulation) on a bounded
    sample of one cfg3 step, extrapolated (SURVEY §8d "cfg3: infeasible ... time
    sampled RHS chunks and fitted complexity, labelled extrapolated"):

      detect   : the reference's per-vertex numpy scan, timed on 16 query vertices
                 against the full opposite surface, x (number of surface-vertex queries)
      W_g      : SuperLU single-column solves measured on a 16x10x16-node block of
                 the same family (the fastest SuperLU path; the reference's one-block
                 solve_multi costs more per column), scaled by nnz(L) (this library's
                 nested-dissection analysis of both sizes; SuperLU's MMD fill grows
                 faster, so this favours the CPU) x the number of RHS columns (3 p_o
                 per object); the dense S^T / X of solve_multi (~40 GB) cannot be
                 formed at full size.  The factorisation itself is once per
                 simulation in the reference (linear material) and is reported, not
                 counted
      rebuild  : the naive-order gemm is m rank-1 updates of an m x m array; timed on
                 m' = 3000 for 8 updates, scaled by (m / m')^3 x 2 gemms
      PGS      : the reference's per-group update (local solve + rank-3 column update
                 of length c) timed on 24 groups of a full-length W, x G x 30 sweeps
    Returns (ms per step, ms per Newton iteration, detail dict)."""
    import ctypes

    import scipy.sparse as sp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cn_oracle as orc

    from paper_2306_06946_b200 import _lib
    from paper_2306_06946_b200.mesh import five_tet_grid, surface_triangles

    det = {}
    nxz, ny = CFG3_NXZ, CFG3_NZ
    groups = 7500  # measured contact groups of the GPU arm at the initial state
    m = 3 * groups
    m_obj = [3 * 7500, 3 * 5000]  # lower: all pairs; upper: the two block-block sources
    # --- detection
    lower = five_tet_grid((nxz, ny, nxz), 0.01)
    tris = surface_triangles(lower.tets)
    vids = np.unique(tris)
    T = lower.nodes[tris]
    N = orc.unit_normals(T)
    t0 = time.perf_counter()
    for vid in vids[:16]:
        p = lower.nodes[vid] + np.array([0.0, 0.3, 0.0])
        cp, bary = orc.closest_on_triangles(T, p)
        diff = p - cp
        dist = np.linalg.norm(diff, axis=1)
        np.where(np.einsum("ij,ij->i", diff, N) >= 0, dist, -dist)
        int(np.flatnonzero(dist <= dist.min() + 1e-9).min())
    det_s = (time.perf_counter() - t0) / 16 * (2 * len(vids))
    det["detect_s"] = det_s
    # --- W_g: small-block SuperLU, extrapolated by nnz(L)
    small = five_tet_grid((16, 10, 16), 0.01)
    body = orc.Body(small.nodes, small.tets, young=1e4, poisson=0.4, density=1000.0)
    A, _ = body.system(small.nodes.ravel(), np.zeros(body.n), H, (0.0, -9.81, 0.0))
    t0 = time.perf_counter()
    F = orc.Factor(A)
    fac_small = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    bvec = rng.standard_normal(body.n)
    t0 = time.perf_counter()
    for _ in range(16):
        F.solve(bvec)
    rhs_small = (time.perf_counter() - t0) / 16

    def nnz_l(mesh):
        nn = len(mesh.nodes)
        r = np.repeat(mesh.tets, 4, axis=1).ravel()
        cc = np.tile(mesh.tets, (1, 4)).ravel()
        G = sp.csr_matrix((np.ones(len(r)), (r, cc)), shape=(nn, nn))
        Ap = sp.kron(G, np.ones((3, 3))).tocsr()
        Ap.sort_indices()
        ip = np.ascontiguousarray(Ap.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(Ap.indices, dtype=np.int64)
        xyz = np.ascontiguousarray(mesh.nodes, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().cnb_chol_analyze(Ap.shape[0], ip.ctypes.data, ix.ctypes.data, 3, xyz.ctypes.data, 32,
                                               ctypes.byref(h)))
        info = (ctypes.c_int64 * 9)()
        fl = (ctypes.c_double * 2)()
        _lib.call("cnb_chol_info", h, info, fl)
        _lib.lib().cnb_chol_destroy(h)
        return float(info[2]), float(fl[0])

    nl_small, fl_small = nnz_l(small)
    nl_full, fl_full = nnz_l(lower)
    rhs_full = rhs_small * nl_full / nl_small
    wg_s = rhs_full * sum(m_obj) + 2 * m * m * 8 / 10e9  # + the S X products (bandwidth)
    det.update(wg_s=wg_s, superlu_small_factor_s=fac_small, superlu_small_rhs_ms=rhs_small * 1e3,
               rhs_full_ms=rhs_full * 1e3, nnzL_ratio=nl_full / nl_small,
               factor_once_per_simulation_s=2 * fac_small * fl_full / fl_small)
    # --- rebuild: naive gemm, m rank-1 updates of m x m
    mp = 3000
    a = rng.standard_normal((mp, 8))
    b = rng.standard_normal((8, mp))
    out = np.zeros((mp, mp))
    t0 = time.perf_counter()
    for k in range(8):
        out += a[:, k, None] * b[None, k, :]
    r1 = (time.perf_counter() - t0) / 8
    rebuild_s = 2.0 * m * r1 * (m / mp) ** 2
    det["rebuild_s"] = rebuild_s
    # --- PGS: per-group update on a full-length W (column slices of a row-major c x c)
    c = m
    Wbig = np.empty((c, c))  # row-major c x c (virtual); only the sampled columns are touched
    Wbig[:, :72] = 1e-3
    dc = np.zeros(c)
    lam = np.zeros(c)
    Wd = np.eye(3)
    t0 = time.perf_counter()
    for g in range(24):
        new = orc.local_solve(0, Wd, np.array([-1e-3, 0.0, 0.0]), np.zeros(3), 0.4, H * H)
        dl = new - lam[0:3]
        if dl.any():
            dc += H * H * (Wbig[:, 3 * g:3 * g + 3] @ dl)
    per_group = (time.perf_counter() - t0) / 24
    pgs_s = per_group * groups * 30
    det["pgs_s"] = pgs_s
    it_s = rebuild_s + pgs_s
    step_s = det_s + wg_s + 10 * it_s
    return step_s * 1e3, it_s * 1e3, {k: round(v, 4) for k, v in det.items()}


def cpu_threads():
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    inp = make_inputs()
    vals, its = [], []
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_reference_sample(inp)
    for _ in range(args.steps):
        s, it, _, _ = cpu_reference_sample(inp)
        vals.append(s)
        its.append(it)
    v = statistics.median(vals)
    cores = cpu_threads()
    sample = ("per step: full assembly + SuperLU factorisation + W_g (solve_multi 1500 RHS + S X); one re-draw "
              "with the naive-order gemm timed on 2% of its rank-1 loop and scaled to m, x10 re-draws")
    return {"metric": "ms per full step (cfg1 compliance-update pipeline); also ms per Newton constraint-update "
                      "iteration", "value": round(v, 2), "unit": "ms/step", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v, 2), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1])",
            "config": {"workload": "cfg1: 40x10x10-node 5-tet grid (12000 DoF), 500 barycentric contacts, "
                                   "10 frame re-draws"},
            "impl": "reference", "ms_per_newton_iter": round(statistics.median(its), 2),
            "cpu_baseline": {"value": round(v, 2), "unit": "ms/step", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(v, 2), "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference_cfg3(args):
    vals, its, dets = [], [], None
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_reference_sample_cfg3()
    for _ in range(args.steps):
        v, it, dets = cpu_reference_sample_cfg3()
        vals.append(v)
        its.append(it)
    v = statistics.median(vals)
    sample = ("oracle port of the reference (linear material, factor once per simulation) on a bounded sample of one "
              "cfg3 step, extrapolated: detection on 16 query vertices, W_g from SuperLU single-column solves on a "
              "16x10x16 block scaled by nnz(L), naive-gemm rebuild timed at m'=3000 scaled by m^3, PGS per-group "
              "update timed on 24 groups x G x 30 sweeps; 10 iterations")
    return {"metric": "ms per full time step (cfg3 450k-DoF two-body scene); also ms per Newton constraint-update "
                      "iteration", "value": round(v, 1), "unit": "ms/step", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v, 1), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded meshes of BASELINE configs[3])",
            "config": {"workload": "cfg3: two 5-tet blocks 50x50x30 nodes (450000 DoF), ground plane, 10 fast-scheme "
                                   "iterations, PGS 30 sweeps tol 1e-6"},
            "impl": "reference", "ms_per_newton_iter": round(statistics.median(its), 1),
            "cpu_baseline": {"value": round(v, 1), "unit": "ms/step", "cores": cpu_threads(), "kind": "port",
                             "sample": sample, "extrapolated": True, "detail_s": dets},
            "e2e": {"value": round(v, 1), "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg1", "cfg4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            line = {"cfg3": run_reference_cfg3, "cfg4": run_reference_cfg4}.get(args.workload, run_reference)(args)
            print(json.dumps(line), flush=True)
        return
    import torch

    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    line = {"cfg3": run_gpu_cfg3, "cfg4": run_gpu_cfg4}.get(args.workload, run_gpu_cfg1)(args, rank, world)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            if args.workload == "cfg4":
                v_, procs, secs = cpu_reference_cfg4(steps=1)
                line["cpu_baseline"] = {"value": round(v_, 3), "unit": "scene-steps/s", "cores": procs,
                                        "kind": "port",
                                        "sample": f"oracle port, {procs} processes x 1 thread, one copy each, "
                                                  f"pre-rolled {CFG4_PREROLL} steps then 1 timed step",
                                        "s_per_step_median": round(statistics.median(secs), 3)}
            elif args.workload == "cfg3":
                s_, it, det = cpu_reference_sample_cfg3()
                line["cpu_baseline"] = {"value": round(s_, 1), "unit": "ms/step", "cores": cpu_threads(),
                                        "kind": "port", "extrapolated": True,
                                        "sample": "oracle port of the reference on a bounded, extrapolated sample of "
                                                  "one cfg3 step (see bench.cpu_reference_sample_cfg3)",
                                        "ms_per_newton_iter": round(it, 1), "detail_s": det}
            else:
                inp = make_inputs()
                s_, it, tf, tw = cpu_reference_sample(inp)
                line["cpu_baseline"] = {"value": round(s_, 2), "unit": "ms/step", "cores": cpu_threads(),
                                        "kind": "port",
                                        "sample": "oracle port of the reference on one cfg1 step: full factorisation "
                                                  "+ W_g, naive-gemm rebuild sampled on 2% of its loop and scaled",
                                        "ms_per_newton_iter": round(it, 2)}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
