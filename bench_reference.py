"""Reference arm of bench.py: the UNMODIFIED reference package on the host cores.

This module imports ``contactnewton`` (the reference, pure Python/numpy/scipy)
from ``baseline/_ref`` (``pip install --target`` of /root/reference/pkg) or,
failing that, ``/root/reference/pkg/src``; it never imports the B200 package,
torch, the oracle or the repo's shared library, so the process it runs in
measures the reference and nothing else.  Inputs come from workloads.py
(numpy only), the same seeded arrays the GPU arm uses.

Two measurements:

* ``cfg1_full_step`` — BASELINE configs[1] exactly as the reference runs it,
  timed end to end and NOT extrapolated: assembly + SuperLU factorisation,
  S, W_g = S A^-1 S^T (assemble_Wg constraints.py:155-179), then 10 re-draws
  of W_k = D_k W_g D_k^T (rebuild_W_fast 182-191 through the naive gemm
  linalg.py:121-147) and dx_k = h A^-1 S^T D_k^T lam_k (_mechanical_correction
  solver.py:250-257).  The same step with the rebuild done as numpy BLAS
  ``D @ W_g @ D.T`` is reported beside it as "reference + BLAS gemm" (not the
  reference).
* ``Cfg3Sampler`` — one cfg3 step (450 000 DoF, ~7 500 contact groups, 10
  Newton iterations), infeasible as-is (dense S^T and X alone need ~2 x 40 GB,
  one naive-gemm rebuild takes hours).  Each phase is timed on a
  bounded sample with the reference's own functions and scaled by the
  phase's work count; every figure is labelled extrapolated:
    detect     collision.detect on a subset of surface vertices x (all / subset)
    assemble   SoftBody.assemble of both full bodies (measured, not scaled)
    solves     Factorization.solve_multi on two reduced blocks of the same shape
               family (20x12x20 and 30x18x30 nodes vs 50x30x50), power-law fit in
               n, x (RHS columns of W_g + the free-motion and correction solves)
    rebuild    linalg.gemm at m' x (m / m')^3, two gemms per rebuild
    pgs        solver.pgs on two reduced dense W, per-group cost fit a + b m,
               x groups x sweeps
    prox       fast_update_proximity at two sizes, fit a m + b m^2
    relin      collision.relinearize on a pair subset x (pairs / subset)
  The reference factorises once per simulation (linear material, scene.py:
  411-415), so the factorisation is reported but not added to the step.
"""

from __future__ import annotations

import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads  # noqa: E402

H = workloads.H


def import_reference():
    """The reference package, from baseline/_ref or the reference tree."""
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "contactnewton")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import contactnewton

            return contactnewton, path
    raise ImportError("reference package contactnewton not found (baseline/_ref or /root/reference/pkg/src)")


def host_info():
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        threads = max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        threads = int(threads or os.cpu_count() or 1)
    return {"nproc": os.cpu_count(), "cpu_model": model, "blas_threads": int(threads)}


# ----------------------------------------------------------------------------
# cfg1: the whole step, measured
# ----------------------------------------------------------------------------

def _cfg1_problem(cn, inp):
    from contactnewton import collision as rcol
    from contactnewton import constraints as rcon

    body = cn.SoftBody(cn.TetMesh(inp["nodes"], inp["tets"]), young=5e3, poisson=0.45, density=1000.0,
                       rayleigh_mass=0.0, rayleigh_stiffness=0.0)
    pairs = []
    for i in range(workloads.CFG1_CONTACTS):
        tri = inp["tris"][inp["tri_idx"][i]]
        w = inp["weights"][i]
        p = w @ inp["nodes"][tri]
        pairs.append(rcol.ProximityPair(
            0, 1, rcol.Attachment(rcol.AttachKind.BARYCENTRIC, 0, triangle=tri.copy(), weights=w.copy()),
            rcol.Attachment(rcol.AttachKind.WORLD, 1, world_point=p.copy()), p.copy(), p.copy(),
            np.array([0.0, 1.0, 0.0]), 0.0, i, int(inp["tri_idx"][i])))
    frames = [[rcol.ContactFrame(n=f[0], t1=f[1], t2=f[2]) for f in D] for D in inp["Ds"]]
    return body, pairs, frames, rcon


def cfg1_full_step(blas_rebuild: bool = False):
    """One whole cfg1 step through the reference; returns (seconds, phase seconds)."""
    cn, _ = import_reference()
    inp = workloads.cfg1_inputs()
    body, pairs, frames, rcon = _cfg1_problem(cn, inp)
    ph = {}
    t0 = time.perf_counter()
    st = body.initial_state()
    A, _ = body.assemble(st, H, (0.0, -9.81, 0.0))
    F = cn.factorize(A)
    t1 = time.perf_counter()
    S = rcon.build_signed_mapping(pairs, 0, body.n_dofs, body.fixed_mask)
    wg = rcon.assemble_Wg({0: S}, {0: F})
    t2 = time.perf_counter()
    rebuild = dx_t = 0.0
    for k in range(workloads.CFG1_REDRAWS):
        ta = time.perf_counter()
        D = rcon.assemble_direction(frames[k])
        if blas_rebuild:
            Dd = D.as_dense()
            W = Dd @ wg.wg @ Dd.T
        else:
            W = rcon.rebuild_W_fast(D, wg).W
        tb = time.perf_counter()
        t = D.apply_transposed(inp["lams"][k])
        H * F.solve(S.T @ t)
        tc = time.perf_counter()
        rebuild += tb - ta
        dx_t += tc - tb
        del W
    t3 = time.perf_counter()
    ph.update(assemble_factor_s=t1 - t0, build_wg_s=t2 - t1, rebuild_s=rebuild, dx_s=dx_t,
              newton_iter_s=(rebuild + dx_t) / workloads.CFG1_REDRAWS)
    return t3 - t0, ph


# ----------------------------------------------------------------------------
# cfg3: bounded samples, extrapolated
# ----------------------------------------------------------------------------

class Cfg3Sampler:
    SMALL = ((20, 12, 20), (30, 18, 30))  # reduced blocks of the cfg3 shape family for the solve fit
    GEMM_M = 600             # naive gemm sample size
    PGS_M = (600, 1500)      # reduced W sizes for the per-group fit
    PROX_M = (1500, 3000)
    DETECT_SAMPLE = 24       # surface vertices per body
    RELIN_SAMPLE = 400       # pairs

    def __init__(self, groups: int, sweeps_per_iter: float, newton_iters: int = 10, m_obj=None):
        self.cn, self.ref_path = import_reference()
        cn = self.cn
        from contactnewton import mesh as rmesh

        self.groups = groups
        self.m = 3 * groups
        self.m_obj = m_obj or [3 * groups, 3 * groups]  # the reference stores every U_o at m x m
        self.sweeps = sweeps_per_iter
        self.iters = newton_iters
        (ln, lt), (un, ut) = workloads.cfg3_meshes()
        t0 = time.perf_counter()
        self.bodies = [cn.SoftBody(cn.TetMesh(ln, lt), young=1e4, poisson=0.4, density=1000.0),
                       cn.SoftBody(cn.TetMesh(un, ut), young=2e3, poisson=0.4, density=1000.0)]
        self.states = [self.bodies[0].initial_state(), self.bodies[1].initial_state((0.5, 0.0, 0.0))]
        self.tris = [rmesh.surface_triangles(b.mesh) for b in self.bodies]
        self.vids = [rmesh.surface_vertices(t) for t in self.tris]
        self.n_full = self.bodies[0].n_dofs
        # reduced blocks for the per-RHS solve cost, factorised once (like the reference: once per simulation)
        self.small = []
        for shape in self.SMALL:
            nodes, tets = workloads.five_tet_grid(shape, 0.01)
            b = cn.SoftBody(cn.TetMesh(nodes, tets), young=1e4, poisson=0.4, density=1000.0)
            A, _ = b.assemble(b.initial_state(), H, (0.0, -9.81, 0.0))
            ta = time.perf_counter()
            F = cn.factorize(A)
            self.small.append((b.n_dofs, F, time.perf_counter() - ta))
        rng = np.random.default_rng(0)
        self._rhs = [rng.standard_normal((n, 16)) for n, _, _ in self.small]
        self.setup_s = time.perf_counter() - t0
        self._pgs_inputs = []
        for mm in self.PGS_M:
            B = rng.standard_normal((mm, mm + 4)) / np.sqrt(mm)
            W = B @ B.T + 0.05 * np.eye(mm)
            self._pgs_inputs.append((W, rng.uniform(-0.02, 0.01, mm)))

    def _fit_power(self, xs, ts):
        a = np.log(ts[1] / ts[0]) / np.log(xs[1] / xs[0])
        return a, ts[1] * (self.n_full / xs[1]) ** a

    def step(self):
        """Seconds of one extrapolated cfg3 reference step, with the phase detail."""
        cn = self.cn
        from contactnewton import collision as rcol
        from contactnewton import constraints as rcon
        from contactnewton import linalg as rlin
        from contactnewton import solver as rsol

        det = {}
        # detection: vertex subsets of both bodies against the full opposite surfaces + the ground
        geoms = []
        for k, b in enumerate(self.bodies):
            sel = self.vids[k][np.linspace(0, len(self.vids[k]) - 1, self.DETECT_SAMPLE).astype(int)]
            geoms.append(rcol.MeshGeometry(k, self.states[k].q.reshape(-1, 3), self.tris[k], sel, True, True))
        geoms.append(rcol.PlaneGeometry(2, (0.0, 1.0, 0.0), 0.0))
        t0 = time.perf_counter()
        cn.detect(geoms, 0.005)
        det["detect_s"] = (time.perf_counter() - t0) * (len(self.vids[0]) + len(self.vids[1])) / (
            2 * self.DETECT_SAMPLE)
        # assembly of both full bodies (measured)
        t0 = time.perf_counter()
        for b, s in zip(self.bodies, self.states):
            b.assemble(s, H, (0.0, -9.81, 0.0))
        det["assemble_s"] = time.perf_counter() - t0
        # per-RHS solve cost at full size from the two reduced factors
        per = []
        for (n, F, _), B in zip(self.small, self._rhs):
            best = np.inf
            for _ in range(3):  # best of 3: the fit amplifies timing noise
                t0 = time.perf_counter()
                F.solve_multi(B)
                best = min(best, time.perf_counter() - t0)
            per.append(best / B.shape[1])
        alpha, rhs_full = self._fit_power([self.small[0][0], self.small[1][0]], per)
        det["solve_exponent"] = alpha
        det["solve_per_rhs_full_s"] = rhs_full
        det["build_wg_s"] = rhs_full * sum(self.m_obj)
        det["free_and_correction_s"] = 4 * rhs_full
        # rebuild: two naive gemms of m^3
        mg = self.GEMM_M
        rng = np.random.default_rng(1)
        a, bm = rng.standard_normal((mg, mg)), rng.standard_normal((mg, mg))
        best = np.inf
        for _ in range(2):
            t0 = time.perf_counter()
            rlin.gemm(a, bm)
            best = min(best, time.perf_counter() - t0)
        det["rebuild_s"] = 2 * best * (self.m / mg) ** 3
        # PGS: per-group cost a + b m
        pg = []
        for W, d in self._pgs_inputs:
            t0 = time.perf_counter()
            rsol.pgs(W, d, H, rsol.PgsConfig(max_iterations=2, tolerance=1e-300, friction=0.4))
            pg.append((time.perf_counter() - t0) / (2 * (W.shape[0] // 3)))
        (m1, m2) = self.PGS_M
        b_ = max((pg[1] - pg[0]) / (m2 - m1), 0.0)
        a_ = max(pg[0] - b_ * m1, 0.0)
        det["pgs_per_group_s"] = a_ + b_ * self.m
        det["pgs_s"] = det["pgs_per_group_s"] * self.groups * self.sweeps
        # proximity update: a m + b m^2
        pr = []
        for mm in self.PROX_M:
            g = mm // 3
            frames = [rcol.ContactFrame(np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 0.0]),
                                        np.array([0.0, 0.0, 1.0]))] * g
            D = rcon.assemble_direction(frames)
            U = np.ones((mm, mm))
            wg = rcon.MappingDelassus(U, {0: U, 1: U})
            pairs = [rcol.ProximityPair(0, 1, rcol.Attachment(rcol.AttachKind.VERTEX, 0, vertex=0),
                                        rcol.Attachment(rcol.AttachKind.VERTEX, 1, vertex=0), None, None,
                                        np.zeros(3), 0.0, i, 0) for i in range(g)]
            pa = np.zeros((g, 3))
            t0 = time.perf_counter()
            rcon.fast_update_proximity(pa, pa, wg, D, np.ones(mm), H, pairs)
            pr.append(time.perf_counter() - t0)
        (p1, p2) = self.PROX_M
        bq = max((pr[1] / p2 - pr[0] / p1) / (p2 - p1), 0.0)
        aq = max(pr[0] / p1 - bq * p1, 0.0)
        det["prox_s"] = aq * self.m + bq * self.m ** 2
        # relinearise: per-pair Python loop
        g = self.RELIN_SAMPLE
        rng = np.random.default_rng(2)
        pa, pb = rng.standard_normal((g, 3)), rng.standard_normal((g, 3))
        prev = [rcol.ContactFrame(np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 0.0]),
                                  np.array([0.0, 0.0, 1.0]))] * g
        t0 = time.perf_counter()
        cn.relinearize([None] * g, pa, pb, prev)
        det["relinearize_s"] = (time.perf_counter() - t0) * self.groups / g
        it = det["rebuild_s"] + det["pgs_s"] + det["prox_s"]
        det["newton_iter_s"] = it
        step = (det["detect_s"] + det["assemble_s"] + det["build_wg_s"] + det["free_and_correction_s"]
                + self.iters * (it + det["relinearize_s"]))
        det["factor_small_s"] = [round(f[2], 3) for f in self.small]
        return step, det


def sample_description(s: Cfg3Sampler) -> str:
    return (f"reference package ({s.ref_path}) on bounded samples of one cfg3 step, extrapolated: detect on "
            f"{s.DETECT_SAMPLE} surface vertices per body x (all / sample); SoftBody.assemble of both bodies measured; "
            f"solve_multi per RHS on {s.SMALL[0]} and {s.SMALL[1]}-node blocks fitted as n^a to "
            f"{s.n_full} DoF x (W_g RHS columns + 4 solves); naive gemm at m'={s.GEMM_M} x (m/m')^3 x 2; solver.pgs "
            f"per-group cost fitted a + b m at m'={s.PGS_M} x {s.groups} groups x {s.sweeps} sweeps; "
            f"fast_update_proximity fitted a m + b m^2; relinearize on {s.RELIN_SAMPLE} pairs x scale; "
            f"{s.iters} Newton iterations; factorisation once per simulation (not counted)")


# ----------------------------------------------------------------------------
# cfg4: independent copies of the cfg0 beam, one reference Simulation per process
# ----------------------------------------------------------------------------

CFG4_PREROLL = 12  # the copies start 2 cm above their planes; contact from step ~7


def cfg4_worker(arg):
    """One process, one thread: copy i as a reference Simulation (cfg0 beam over
    its own tilted plane, its own mu and jitter), pre-rolled to the timed region,
    then ``steps`` timed Simulation.step calls.  Returns seconds per step."""
    i, steps, preroll = arg
    cn, _ = import_reference()
    from contactnewton import scene as rsc
    from contactnewton import solver as rsol

    nodes, tets = workloads.five_tet_grid(workloads.CFG0_SHAPE, 0.01)
    tilts, mus, jit = workloads.cfg4_draws(i, 1, nodes.size)
    nrm = workloads.plane_normals(tilts)[0]
    rest = workloads.placement(nodes, workloads.plane_normals(tilts), 0.02)[0]
    soft = rsc.SoftSpec(name="beam", mesh=cn.TetMesh(rest, tets), young=5e3, poisson=0.45, density=1000.0)
    plane = rsc.PlaneSpec(name="ground", normal=tuple(nrm), offset=0.0)
    cfg = rsc.SceneConfig(objects=[soft, plane], h=H, threshold=0.005,
                          pgs=rsol.PgsConfig(max_iterations=1000, tolerance=1e-10, friction=float(mus[0])),
                          newton=rsol.NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0,
                                                   rotation_tol=-1.0),
                          output=rsc.OutputConfig(snapshots=False, metrics=False))
    sim = rsc.Simulation(cfg)
    obj = sim.dynamic_objects[0]
    obj.state.q = obj.state.q + jit[0]
    for _ in range(preroll):
        sim.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step()
    return (time.perf_counter() - t0) / steps


def cfg4_throughput(steps=1, procs=None, preroll=CFG4_PREROLL):
    """scene-steps/s on all host cores: one reference process per core, copy i in
    process i; throughput = sum over processes of 1 / (seconds per step)."""
    import multiprocessing as mp

    procs = procs or (os.cpu_count() or 1)
    keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys:
        os.environ[k] = "1"
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            secs = pool.map(cfg4_worker, [(i, steps, preroll) for i in range(procs)])
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return sum(1.0 / s for s in secs), procs, secs


def cfg1_quick_step():
    """cpu_baseline sample of cfg1 (about 30 s): the whole step except that one of
    the 10 identical re-draws is timed and counted 10 times."""
    cn, _ = import_reference()
    inp = workloads.cfg1_inputs()
    body, pairs, frames, rcon = _cfg1_problem(cn, inp)
    t0 = time.perf_counter()
    A, _ = body.assemble(body.initial_state(), H, (0.0, -9.81, 0.0))
    F = cn.factorize(A)
    S = rcon.build_signed_mapping(pairs, 0, body.n_dofs, body.fixed_mask)
    wg = rcon.assemble_Wg({0: S}, {0: F})
    t1 = time.perf_counter()
    D = rcon.assemble_direction(frames[0])
    rcon.rebuild_W_fast(D, wg)
    H * F.solve(S.T @ D.apply_transposed(inp["lams"][0]))
    t2 = time.perf_counter()
    return (t1 - t0) + workloads.CFG1_REDRAWS * (t2 - t1), t2 - t1
