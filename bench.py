#!/usr/bin/env python
"""Benchmark: particle-updates/s of the Nauticle hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 0-4] [--impl ours|reference]
                  [--mode fast|exact] [--slab] [--comm torch|native]

Workloads (scenes.py; synthetic, seeded — no dataset exists for this path):
  --config 2  (default) BASELINE cfg2: 3D WCSPH dam break, 4.0 M fluid + 1.92 M wall
              particles, dx = 0.005, Wendland C2. One step = cell build + density/EOS
              pass + momentum (G11 + artificial viscosity) pass + symplectic update.
  --config 1  BASELINE cfg1: 1,048,576 random particles in a periodic unit cube, cubic
              spline. One step = cell build + sph_S density + sph_G11 + sph_L0.
  --config 0  BASELINE cfg0: 2D dam break, 23,018 particles (the CPU-runnable case).

value = particle-updates/s = N_active x K / (max over ranks of the device time of K
steps), CUDA events on the context's stream, L2 flushed (256 MiB memset) between
timed steps outside the timed intervals. `e2e` times the same step through the
C-ABI with host buffers: the step's inputs copied from pinned host memory and its
results copied back inside the timed region.

--impl reference times the reference's own CPU implementation (oracle/_ref: the
unmodified reference sources built on the shims) through its public API with
all host threads, on a bounded sample of the same workload; rank 0 only.
Multi-GPU (torchrun): cfg0/2/3 are slab-decomposed along x (whole cell planes per
rank, two ghost planes per face, migration + ghost refresh over NCCL every step;
--comm torch: slab.py over torch.distributed, --comm native: the library's own
nau_migrate / nau_halo_exchange), cfg4 shards the bodies with an all-gather of the
sources every step; `scaling` is "strong" (the workload is fixed as N grows).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-updates/s"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the bounded reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true",
                    help="cfg0/cfg2: run the slab-decomposed path even on one GPU")
    ap.add_argument("--comm", default="torch", choices=["torch", "native"],
                    help="slab exchange driver: torch.distributed (slab.py) or the "
                         "library's own NCCL layer (nau_migrate / nau_halo_exchange)")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"],
                    help="fast: warp-per-particle sums (1e-10 tolerance); exact: reference order, bitwise")
    return ap.parse_args()


# ------------------------------------------------------------------ dist ----
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # plumbing checks on a single-GPU box: every rank on one device over gloo
        # (NAU_BENCH_DEVICE=0 NAU_DIST_BACKEND=gloo); never a measurement
        if "NAU_BENCH_DEVICE" in os.environ:
            self.local = int(os.environ["NAU_BENCH_DEVICE"])
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            backend = os.environ.get("NAU_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if not self.pg:
            return x
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------- clocks ----
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if s[2 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(config):
    """Per-launch DRAM bytes of each hot kernel of BASELINE config `config` from the
    committed ncu capture (profiles/traffic.json, keyed "cfg<k>"; {} if not captured)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(f"cfg{config}", {})
    except OSError:
        return {}


# ------------------------------------------------------------- workloads ----
def stencil_candidates(ctx, dim):
    """C_total = sum_c count_c * sum_{c' in 3^d stencil of c} count_c' (interior cells;
    the cut-off/periodic edges as the domain says). Algorithmic candidate count."""
    _, _, count, _ = ctx.cell_tables()
    cells = [int(x) for x in ctx._dom[1][:dim] - ctx._dom[0][:dim]]
    g = count.reshape(cells[::-1]).astype(np.float64)
    kinds = list(ctx._dom[3][:dim])[::-1]
    acc = np.zeros_like(g)
    import itertools
    for off in itertools.product((-1, 0, 1), repeat=dim):
        sh = g
        for ax, o in enumerate(off):
            if o == 0:
                continue
            if kinds[ax] == 0:
                sh = np.roll(sh, -o, axis=ax)
            else:
                sh = np.roll(sh, -o, axis=ax)
                idx = [slice(None)] * dim
                idx[ax] = -1 if o > 0 else 0
                sh = sh.copy()
                sh[tuple(idx)] = 0
        acc += sh
    return float((g * acc).sum())


WORKLOAD_NAMES = {
    0: "cfg0: 2D WCSPH dam break, 20,000 fluid + 3-layer walls, dx=0.01",
    1: "cfg1: 3D SPH operator microbench, N=1,048,576 periodic, cubic spline",
    2: "cfg2: 3D WCSPH dam break, 4.0M fluid + 3-layer walls, dx=0.005, Wendland C2",
    3: ("cfg3: 3D DEM granular settling, 2,000,000 spheres, untruncated log-normal radii at "
        "seeded random-sequential-addition positions, linear spring-dashpot + Coulomb, dt=1e-6"),
    4: "cfg4: 3D n-body Plummer sphere, N=262,144, eps=0.01, leapfrog dt=1e-3",
}


class Workload:
    name = ""
    dtype = "f64"
    survey = None  # (bytes, fp64 flops) per step by SURVEY.md §8(d)'s convention, basis

    def setup(self, ctx):
        raise NotImplementedError

    def step(self, ctx):
        raise NotImplementedError

    def e2e_step(self, ctx):
        raise NotImplementedError


class Microbench(Workload):
    """BASELINE cfg1."""

    def __init__(self):
        from paper_1710_08259_b200 import scenes
        self.sc = scenes.sph_microbench()
        self.name = WORKLOAD_NAMES[1]
        self.kw = "Wc33220"

    def setup(self, ctx):
        sc, prm = self.sc, self.sc.params
        ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(sc.pos)
        ctx.add_field("A", 1, 1, sc.fields["A"])
        for f, r in (("rho", 1), ("G", 3), ("L", 1)):
            ctx.add_field(f, r, 1, 0.0)
        ctx.boundary_shift()
        ctx.build_cells()
        self.n_active = sc.n
        C = stencil_candidates(ctx, 3)
        nn = float(ctx.neighbor_counts(prm["radius"]).sum())
        N = float(sc.n)
        nc = float(np.prod([b - a for a, b in zip(sc.min_cells, sc.max_cells)]))
        # SURVEY.md §8(d) algorithmic bytes B and flops F per launch (per-particle figure x
        # N): every operator pass is charged 8 flops per stencil candidate (C) plus its
        # per-neighbour flops (n), whether or not the implementation skips candidates.
        # The neighbour-list build is an implementation kernel: its positions read is
        # counted, its candidate tests are already charged to the passes.
        self.kernels = {
            100: ("sph_S density", 32.0 * N, 8.0 * C + 14 * nn),
            102: ("sph_G11 gradient", 64.0 * N, 8.0 * C + 24 * nn),
            103: ("sph_L0 Laplacian", 48.0 * N, 8.0 * C + 27 * nn),
            # fused G11 + L0 (one list walk): x, A, rho in; G, L out; both passes' flops
            110: ("sph_G11+L0 fused", 80.0 * N, 2 * 8.0 * C + (24 + 27) * nn),
            302: ("neighbour-list build", 24.0 * N, 0.0),
            # hash 32 + sort 60 + range 4 + 8 N_c/N + reorder of r, A (16 B per component)
            300: ("cell build", (32.0 + 60.0 + 4.0 + 16.0 * 4) * N + 8.0 * nc, 0.0),
        }
        self.cand_per_particle = C / N
        self.nbr_per_particle = nn / N
        # SURVEY.md §8(d) step roofline: 8 flops per stencil candidate per operator pass
        self.survey = (sum(b for k, (_, b, _) in self.kernels.items() if k not in (110,)),
                       3 * 8.0 * C + (14 + 24 + 27) * nn,
                       "3 passes x 8C + (14 + 24 + 27) n")
        import torch
        self.h_pos = torch.from_numpy(np.ascontiguousarray(sc.pos)).pin_memory()
        self.h_A = torch.from_numpy(np.ascontiguousarray(sc.fields["A"])).pin_memory()
        self.h_out = [torch.empty((r, sc.n), dtype=torch.float64).pin_memory() for r in (1, 3, 1)]
        self.h2d = (self.h_pos.numel() + self.h_A.numel()) * 8
        self.d2h = sum(t.numel() for t in self.h_out) * 8

    def step(self, ctx):
        prm = self.sc.params
        ctx.build_cells()
        ctx.interact("sph_S", [1.0, prm["mass"], 1.0, prm["radius"]], "rho", kernel=self.kw)
        # G = sph_G11(A, m, rho), L = sph_L0(A, m, rho): one fused list walk (FAST mode;
        # the two interact() calls otherwise), bitwise equal to the two calls
        ctx.interact_g11_l0(["A", prm["mass"], "rho", prm["radius"]], "G", "L", kernel=self.kw)

    def e2e_step(self, ctx):
        ctx.upload_async("r", self.h_pos.data_ptr())
        ctx.upload_async("A", self.h_A.data_ptr())
        self.step(ctx)
        for f, t in zip(("rho", "G", "L"), self.h_out):
            ctx.download_async(f, t.data_ptr())

    def config(self):
        return {"workload": self.name, "particles": self.sc.n, "cells": "44^3 periodic",
                "kernel": "cubic spline (Wc33220)",
                "candidates_per_particle": round(self.cand_per_particle, 2),
                "neighbours_per_particle": round(self.nbr_per_particle, 2)}


class DamBreak(Workload):
    """BASELINE cfg2 (dim 3) / cfg0 (dim 2)."""

    def __init__(self, dim):
        from paper_1710_08259_b200 import scenes
        self.dim = dim
        if dim == 3:
            self.sc = scenes.dam_break(3, dx=0.005)
            self.name = WORKLOAD_NAMES[2]
        else:
            self.sc = scenes.dam_break(2, dx=0.01)
            self.name = WORKLOAD_NAMES[0]

    def setup(self, ctx):
        from paper_1710_08259_b200 import nau
        sc, prm = self.sc, self.sc.params
        ctx.set_domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(sc.pos)
        for k in ("rho", "p", "v", "vdot", "mask"):
            v = np.asarray(sc.fields[k]).reshape(-1, sc.n)
            ctx.add_field(k, v.shape[0], 1, v)
        ctx.boundary_shift()
        ctx.build_cells()
        p = nau.WcsphParams()
        p.kernel_family, p.kernel_dim = nau.K_WENDLAND, sc.dim
        p.mass, p.radius, p.rho0, p.B = prm["mass"], prm["radius"], prm["rho0"], prm["B"]
        p.gamma, p.visc, p.dt = prm["gamma"], prm["visc"], prm["dt"]
        for a in range(sc.dim):
            p.g[a] = prm["g"][a]
        f = ctx.fields
        p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = (f["rho"].id, f["p"].id, f["v"].id,
                                                     f["vdot"].id, f["mask"].id)
        self.p = p
        C = stencil_candidates(ctx, sc.dim)
        nn = float(ctx.neighbor_counts(prm["radius"]).sum())
        N = float(sc.n)
        d = sc.dim
        self.n_active = sc.n
        nc = float(np.prod([b - a for a, b in zip(sc.min_cells, sc.max_cells)]))
        # SURVEY.md §8(d) algorithmic bytes B and flops F per launch (per-particle figure x
        # N; 3D figures, scaled by dim): density 40 B, 8C + 14n + 10; G11 + A 88 B,
        # 8C + 42n; integrator 128 B, 20; cell build = hash 32 + sort 60 + range 4 +
        # 8 N_c/N + reorder 16 B per moved component (r, v, rho, mask). The neighbour-
        # list build is an implementation kernel (positions read; its candidate tests are
        # already charged to the two passes).
        self.kernels = {
            200: ("density+EOS", (8.0 * d + 8 + 8) * N, 8.0 * C + 14 * nn + 10 * N),
            201: ("momentum G11+A", (8.0 * d * 3 + 16) * N, 8.0 * C + 42 * nn),
            302: ("neighbour-list build", 8.0 * d * N, 0.0),
            301: ("symplectic integrator", (8.0 * (4 * d + 1) + 8 * 2 * d) * N, 20.0 * N),
            300: ("cell build", (8.0 * d + 8 + 60 + 4 + 16 * (2 * d + 2)) * N + 8.0 * nc, 0.0),
        }
        self.cand_per_particle = C / N
        self.nbr_per_particle = nn / N
        # SURVEY.md §8(d) step roofline: density 8C + 14n + 10, momentum 8C + 42n, integrator 20
        self.survey = (sum(b for _, b, _ in self.kernels.values()),
                       2 * 8.0 * C + (14 + 42) * nn + 30.0 * N,
                       "2 passes x 8C + 56 n + 30 per particle")
        import torch
        self.h_r = torch.from_numpy(np.ascontiguousarray(sc.pos)).pin_memory()
        self.h_v = torch.zeros((d, sc.n), dtype=torch.float64).pin_memory()
        self.h_out = {k: torch.empty((r, sc.n), dtype=torch.float64).pin_memory()
                      for k, r in (("r", d), ("v", d), ("rho", 1), ("p", 1))}
        self.h2d = (self.h_r.numel() + self.h_v.numel()) * 8
        self.d2h = sum(t.numel() for t in self.h_out.values()) * 8

    def step(self, ctx):
        ctx.wcsph_step(self.p)

    def e2e_step(self, ctx):
        ctx.upload_async("r", self.h_r.data_ptr())
        ctx.upload_async("v", self.h_v.data_ptr())
        self.step(ctx)
        for k, t in self.h_out.items():
            ctx.download_async(k, t.data_ptr())

    def config(self):
        sc = self.sc
        return {"workload": self.name, "particles": sc.n, "fluid": sc.params["n_fluid"],
                "dx": sc.params["dx"], "dt": sc.params["dt"], "kernel": f"Wendland C2 (Wp5{sc.dim}220)",
                "candidates_per_particle": round(self.cand_per_particle, 2),
                "neighbours_per_particle": round(self.nbr_per_particle, 2)}


class DemColumn(Workload):
    """BASELINE cfg3: 2 M spheres settling (linear spring-dashpot + Coulomb, mirror walls)."""

    def __init__(self):
        from paper_1710_08259_b200 import scenes
        self.sc = scenes.dem_column()
        self.name = WORKLOAD_NAMES[3]

    def setup(self, ctx):
        from paper_1710_08259_b200 import nau
        sc, prm = self.sc, self.sc.params
        ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(sc.pos)
        for k in ("v", "vdot", "R", "m"):
            v = np.asarray(sc.fields[k]).reshape(-1, sc.n)
            ctx.add_field(k, v.shape[0], 1, v)
        ctx.boundary_shift()
        ctx.build_cells()
        p = nau.DemParams()
        f = ctx.fields
        p.law, p.f_v, p.f_vdot, p.f_R, p.f_m = 8, f["v"].id, f["vdot"].id, f["R"].id, f["m"].id
        p.P, p.Q, p.cf, p.search_radius, p.dt = prm["kn"], prm["en"], prm["cf"], \
            prm["search_radius"], prm["dt"]
        for a in range(3):
            p.g[a] = prm["g"][a]
        self.p = p
        C = stencil_candidates(ctx, 3)
        N = float(sc.n)
        self.n_active = sc.n
        nc = float(np.prod(sc.max_cells))
        self._C = C
        # DEM 88 B, 8C + 40 per contact (contacts counted below);
        # integrator (no mask) 120 B, 20; cell build hash + sort + range + reorder of
        # r, v, R, m (8 components)
        self.kernels = {
            108: ("dem_lsd contact sum", 88.0 * N, 8.0 * C),
            301: ("symplectic integrator", (8.0 * 9 + 8 * 6) * N, 20.0 * N),
            300: ("cell build", (24.0 + 8 + 60 + 4 + 16 * 8) * N + 8.0 * nc, 0.0),
        }
        self.cand_per_particle = C / N
        self.survey = (sum(b for _, b, _ in self.kernels.values()), 8.0 * C + 20.0 * N,
                       "8C + 20 per particle (contact flops not counted)")
        import torch
        self.h_r = torch.from_numpy(np.ascontiguousarray(sc.pos)).pin_memory()
        self.h_v = torch.zeros((3, sc.n), dtype=torch.float64).pin_memory()
        self.h_out = {k: torch.empty((3, sc.n), dtype=torch.float64).pin_memory() for k in ("r", "v")}
        self.h2d = (self.h_r.numel() + self.h_v.numel()) * 8
        self.d2h = sum(t.numel() for t in self.h_out.values()) * 8

    def step(self, ctx):
        ctx.dem_step(self.p)

    def e2e_step(self, ctx):
        ctx.upload_async("r", self.h_r.data_ptr())
        ctx.upload_async("v", self.h_v.data_ptr())
        self.step(ctx)
        for k, t in self.h_out.items():
            ctx.download_async(k, t.data_ptr())

    def config(self):
        sc = self.sc
        return {"workload": self.name, "particles": sc.n, "cells": "x".join(map(str, sc.max_cells)),
                "dt": sc.params["dt"], "candidates_per_particle": round(self.cand_per_particle, 2)}


class Gravity(Workload):
    """BASELINE cfg4: Plummer sphere, direct all-pairs softened gravity, leapfrog."""

    def __init__(self):
        from paper_1710_08259_b200 import scenes
        self.sc = scenes.plummer()
        self.name = WORKLOAD_NAMES[4]

    def setup(self, ctx):
        from paper_1710_08259_b200 import nau
        sc, prm = self.sc, self.sc.params
        ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(sc.pos)
        ctx.add_field("v", 3, 1, sc.fields["v"])
        ctx.add_field("a", 3, 1, 0.0)
        ctx.boundary_shift()
        p = nau.GravityParams()
        p.f_v, p.f_a, p.f_m = ctx.fields["v"].id, ctx.fields["a"].id, -1
        p.m, p.G, p.eps, p.dt = prm["m"], prm["G"], prm["eps"], prm["dt"]
        self.p = p
        ctx.interact("nbody_gravity", [prm["m"], prm["G"], prm["eps"]], "a")  # a(t=0)
        N = float(sc.n)
        self.n_active = sc.n
        self.kernels = {107: ("all-pairs gravity", 56.0 * N, 20.0 * N * N)}
        self.survey = (56.0 * N, 20.0 * N * N, "20 flops per pair")
        import torch
        self.h_r = torch.from_numpy(np.ascontiguousarray(sc.pos)).pin_memory()
        self.h_v = torch.from_numpy(np.ascontiguousarray(sc.fields["v"])).pin_memory()
        self.h_out = {k: torch.empty((3, sc.n), dtype=torch.float64).pin_memory() for k in ("r", "v")}
        self.h2d = (self.h_r.numel() + self.h_v.numel()) * 8
        self.d2h = sum(t.numel() for t in self.h_out.values()) * 8

    def step(self, ctx):
        ctx.leapfrog_step(self.p)

    def e2e_step(self, ctx):
        ctx.upload_async("r", self.h_r.data_ptr())
        ctx.upload_async("v", self.h_v.data_ptr())
        self.step(ctx)
        for k, t in self.h_out.items():
            ctx.download_async(k, t.data_ptr())

    def config(self):
        return {"workload": self.name, "particles": self.sc.n, "pairs_per_step": self.sc.n ** 2}


class GravityShard(Gravity):
    """cfg4 sharded over the ranks: each rank owns N/W bodies (a
    contiguous block of the global order); every step each rank's positions + masses
    reach all ranks as chunk `rank` of a broadcast pipeline (NCCL; slab.pipelined_sources:
    chunk c + 1 in flight while chunk c is evaluated) and every rank sums its bodies
    against the chunks in global order — identical sums to the single-GPU run."""

    def __init__(self, dist):
        super().__init__()
        self.dist = dist

    def setup(self, ctx):
        import torch
        from paper_1710_08259_b200 import nau
        sc, prm = self.sc, self.sc.params
        W, r = self.dist.world, self.dist.rank
        N = sc.n
        assert N % W == 0, "bodies must split evenly for the all-gather"
        nl = N // W
        self.g0 = r * nl
        sl = slice(self.g0, self.g0 + nl)
        ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(np.ascontiguousarray(sc.pos[:, sl]))
        ctx.add_field("v", 3, 1, np.ascontiguousarray(sc.fields["v"][:, sl]))
        ctx.add_field("a", 3, 1, 0.0)
        ctx.boundary_shift()
        self.ctx = ctx
        self.dev = f"cuda:{torch.cuda.current_device()}"
        self.local_rows = torch.empty((nl, 4), dtype=torch.float64, device=self.dev)
        self.src_bufs = [torch.empty((nl, 4), dtype=torch.float64, device=self.dev) for _ in range(2)]
        self.N, self.nl = N, nl
        self.fv, self.fa = ctx.fields["v"].id, ctx.fields["a"].id
        self._forces()  # a(t = 0)
        self.n_active = nl
        self.kernels = {107: ("all-pairs gravity", 56.0 * nl, 20.0 * nl * N)}
        self.survey = (56.0 * nl, 20.0 * nl * N, "20 flops per pair (this rank's bodies)")
        self.h_r = torch.from_numpy(np.ascontiguousarray(sc.pos[:, sl])).pin_memory()
        self.h_v = torch.from_numpy(np.ascontiguousarray(sc.fields["v"][:, sl])).pin_memory()
        self.h_out = {k: torch.empty((3, nl), dtype=torch.float64).pin_memory() for k in ("r", "v")}
        self.h2d = (self.h_r.numel() + self.h_v.numel()) * 8
        self.d2h = sum(t.numel() for t in self.h_out.values()) * 8

    def _forces(self):
        import torch
        ctx, prm = self.ctx, self.sc.params
        ctx._check(ctx.L.nau_pack_sources(ctx.h, -1, prm["m"], self.local_rows.data_ptr()))
        if self.dist.world == 1:
            ctx._check(ctx.L.nau_gravity_sources(ctx.h, self.local_rows.data_ptr(), self.N, self.g0,
                                                 prm["G"], prm["eps"], self.fa))
            return
        # broadcast-pipelined sources: chunk c + 1 is in flight while chunk c is evaluated,
        # chunks consumed in global order (= the single-GPU sums), no host synchronisation
        from paper_1710_08259_b200 import slab
        stream = torch.cuda.ExternalStream(ctx.L.nau_get_stream(ctx.h))
        nl = self.nl

        def consume(c, rows):
            ctx._check(ctx.L.nau_gravity_sources_part(ctx.h, rows.data_ptr(), nl, self.g0 - c * nl,
                                                      prm["G"], prm["eps"], self.fa, int(c > 0)))

        with torch.cuda.stream(stream):  # transfers are ordered after the pack, kernels after them
            slab.pipelined_sources(self.dist.pg, self.local_rows, self.src_bufs, self.dist.world,
                                   self.dist.rank, consume)

    def step(self, ctx):
        dt = self.sc.params["dt"]
        ctx.euler(self.fv, self.fa, 0.5 * dt, self.fv)  # v = euler(v, a, dt/2)
        ctx.euler(0, self.fv, dt, 0)                     # r = euler(r, v, dt) + shift
        self._forces()                                   # a = nbody_gravity(m, G, eps)
        ctx.euler(self.fv, self.fa, 0.5 * dt, self.fv)  # v = euler(v, a, dt/2)

    def config(self):
        c = super().config()
        c["shards"] = self.dist.world
        return c


class _SlabMixin:
    """Common setup of the slab-decomposed decks (paper_1710_08259_b200/slab.py, SURVEY.md
    §8(e)): x-threshold slabs balanced on a fine x-histogram, owned particles + the
    ghosts within one interaction radius of each face; the local set is rebuilt in place
    each step (no full reload); the torch driver re-balances every 100 steps."""

    REBALANCE_EVERY = 100

    def _slab_setup(self, ctx, radius, field_widths):
        import torch
        from paper_1710_08259_b200 import nau, slab
        sc = self.sc
        self.periodic = sc.kinds[0] == 0
        lo = sc.min_cells[0] * sc.cell_size[0]
        hi = sc.max_cells[0] * sc.cell_size[0]
        world, rank = self.dist.world, self.dist.rank
        self.R = radius
        self.bounds = slab.balanced_x_bounds(sc.pos[0], lo, hi, world, 2.0 * radius)
        names = [k for k, _ in field_widths]
        rows = slab.initial_rows(sc, names, self.bounds, rank, radius, self.periodic)
        d = sc.dim
        ctx.set_domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ctx.set_particles(np.ascontiguousarray(rows[:, :d].T))
        for k, w in field_widths + [("gid", 1), ("ghost", 1)]:
            ctx.add_field(k, w, 1, 0.0)
        # room for arrivals: ghosts and immigrants of later steps (rebuilt in place)
        ctx._check(ctx.L.nau_reserve(ctx.h, int(1.25 * len(rows)) + 65536))
        self.rows0 = rows
        return rows

    def _slab_driver(self, ctx, backend):
        import torch
        from paper_1710_08259_b200 import nau, slab
        world, rank = self.dist.world, self.dist.rank
        self.backend = backend
        backend.load(torch.from_numpy(self.rows0).to(backend.device))
        if self.native:
            uid = [nau.Context.comm_unique_id() if rank == 0 else None]
            if world > 1:
                self.dist.pg.broadcast_object_list(uid, src=0)
            ctx.comm_init(uid[0], world, rank)
            ctx.slab_config(0, self.bounds, self.periodic, self.R)
            self.rank_drv = None
        else:
            ex = slab.Exchanger(self.dist.pg, rank, world, self.periodic, backend.device)
            self.rank_drv = slab.SlabRank(backend, ex, self.bounds, self.R, self.periodic,
                                          rebalance_every=self.REBALANCE_EVERY)
        self.steps_done = 0
        self.n_active = int((self.rows0[:, -1] == 0).sum())
        self.h_rows = torch.from_numpy(self.rows0).pin_memory()
        self.h_out = torch.empty_like(self.h_rows).pin_memory()
        self.h2d = self.d2h = self.h_rows.numel() * 8

    def _native_exchange(self, ctx):
        """Migration + halo after the integrator; re-balancing every 100 steps (comm.cu)."""
        if self.dist.world == 1:
            return
        self.steps_done += 1
        if self.steps_done % self.REBALANCE_EVERY == 0:
            ctx.slab_rebalance()
        else:
            ctx.migrate()

    def e2e_step(self, ctx):
        import torch
        from paper_1710_08259_b200 import slab
        dev_rows = self.h_rows.to(self.backend.device, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.backend.load(dev_rows)
        self.step(ctx)
        local = self.backend.pack(self.backend.select_x(-math.inf, math.inf, slab.FLAG_OWNED,
                                                        slab.FLAG_OWNED))
        m = min(local.shape[0], self.h_out.shape[0])
        self.h_out[:m].copy_(local[:m], non_blocking=False)

    def slab_config(self):
        drv = self.rank_drv
        return {"slabs_x": [round(b, 6) for b in (drv.bounds if drv else self.bounds)],
                "halo": f"ghosts within R = {self.R:.6g} of each face (not evaluated)",
                "rebalance_every": self.REBALANCE_EVERY,
                "exchange": ("native NCCL (comm.cu)" if self.native
                             else "torch.distributed (slab.py)")}


class DamBreakSlab(_SlabMixin, DamBreak):
    """cfg2/cfg0 slab-decomposed along x: per step density pass, halo values (rho, p) to
    the ghosts, momentum pass, integrator, then migration + halo in one exchange."""

    FIELDS = ["rho", "p", "v", "vdot", "mask"]

    def __init__(self, dim, dist, native=False):
        super().__init__(dim)
        self.dist = dist
        self.native = native

    def setup(self, ctx):
        from paper_1710_08259_b200 import nau, slab
        sc, prm = self.sc, self.sc.params
        d = sc.dim
        self._slab_setup(ctx, prm["radius"], [("rho", 1), ("p", 1), ("v", d), ("vdot", d),
                                              ("mask", 1)])
        p = nau.WcsphParams()
        p.kernel_family, p.kernel_dim = nau.K_WENDLAND, sc.dim
        p.mass, p.radius, p.rho0, p.B = prm["mass"], prm["radius"], prm["rho0"], prm["B"]
        p.gamma, p.visc, p.dt = prm["gamma"], prm["visc"], prm["dt"]
        for a in range(sc.dim):
            p.g[a] = prm["g"][a]
        f = ctx.fields
        p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = (f["rho"].id, f["p"].id, f["v"].id,
                                                     f["vdot"].id, f["mask"].id)
        self.p = p
        self._slab_driver(ctx, slab.GpuBackend(ctx, p))
        N = float(len(self.rows0))
        self.kernels = {
            200: ("density+EOS", (8.0 * d + 8 + 8) * N, 0.0),
            201: ("momentum G11+A", (8.0 * d * 3 + 16) * N, 0.0),
            302: ("neighbour-list build", 8.0 * d * N, 0.0),
            301: ("symplectic integrator", (8.0 * (4 * d + 1) + 8 * 2 * d) * N, 20.0 * N),
            300: ("cell build", (8.0 * d + 8 + 60 + 4 + 16 * (2 * d + 4)) * N, 0.0),
        }
        self.survey = None  # per-rank slabs: C and n are not counted
        self.cand_per_particle = float("nan")
        self.nbr_per_particle = float("nan")

    def step(self, ctx):
        if not self.native:
            self.rank_drv.step()
            return
        if self.dist.world == 1:
            ctx.wcsph_step(self.p)
            return
        import ctypes as C
        ctx.wcsph_pass(self.p, 0)
        ctx.halo_exchange(["rho", "p"])
        ctx._check(ctx.L.nau_wcsph_ghost_payload(ctx.h, C.byref(self.p)))
        ctx.wcsph_pass(self.p, 1)
        ctx.wcsph_pass(self.p, 2)
        self._native_exchange(ctx)

    def config(self):
        c = super().config()
        c.pop("candidates_per_particle", None)
        c.pop("neighbours_per_particle", None)
        c.update(self.slab_config())
        return c


class DemSlab(_SlabMixin, DemColumn):
    """cfg3 slab-decomposed along x (balanced while the column settles
    in z); the DEM deck is one neighbour pass, so only migration + halo per step."""

    FIELDS = ["v", "vdot", "R", "m"]

    def __init__(self, dist, native=False):
        super().__init__()
        self.dist = dist
        self.native = native

    def setup(self, ctx):
        from paper_1710_08259_b200 import nau, slab
        sc, prm = self.sc, self.sc.params
        self._slab_setup(ctx, prm["search_radius"], [("v", 3), ("vdot", 3), ("R", 1), ("m", 1)])
        p = nau.DemParams()
        f = ctx.fields
        p.law, p.f_v, p.f_vdot, p.f_R, p.f_m = 8, f["v"].id, f["vdot"].id, f["R"].id, f["m"].id
        p.P, p.Q, p.cf, p.search_radius, p.dt = prm["kn"], prm["en"], prm["cf"], \
            prm["search_radius"], prm["dt"]
        for a in range(3):
            p.g[a] = prm["g"][a]
        self.p = p
        self._slab_driver(ctx, slab.GpuBackend(ctx, None, step_fn=lambda: ctx.dem_step(p)))
        N = float(len(self.rows0))
        self.kernels = {108: ("dem_lsd contact sum", 88.0 * N, 0.0),
                        301: ("symplectic integrator", 8.0 * 15 * N, 20.0 * N),
                        300: ("cell build", (24.0 + 8 + 60 + 4 + 16 * 10) * N, 0.0)}
        self.cand_per_particle = float("nan")

    def step(self, ctx):
        if self.native:
            ctx.dem_step(self.p)
            self._native_exchange(ctx)
        else:
            self.rank_drv.step()

    def config(self):
        sc = self.sc
        c = {"workload": self.name, "particles": sc.n, "dt": sc.params["dt"]}
        c.update(self.slab_config())
        return c


def make_workload(cfg, dist=None, slab=False, native=False):
    if slab and cfg in (0, 2):
        return DamBreakSlab(3 if cfg == 2 else 2, dist, native)
    if slab and cfg == 4:
        return GravityShard(dist)
    if slab and cfg == 3:
        return DemSlab(dist, native)
    return {1: Microbench, 2: lambda: DamBreak(3), 0: lambda: DamBreak(2), 3: DemColumn,
            4: Gravity}[cfg]()


# ------------------------------------------------------------ timing ----
def timed_steps(ctx, fn, steps, flush):
    """Per-step CUDA events on the context stream; L2 flush between steps, untimed."""
    import torch
    stream = torch.cuda.ExternalStream(ctx.L.nau_get_stream(ctx.h))
    evs = []
    with torch.cuda.stream(stream):
        for _ in range(steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(ctx)
            e1.record(stream)
            evs.append((e0, e1))
    stream.synchronize()
    ctx.sync()
    return sum(a.elapsed_time(b) for a, b in evs)


def timed_pipelined(ctx, fn, steps):
    """K end-to-end steps as ONE device-timed interval: the context's copy streams are
    fenced after the start event and joined before the stop event, so every step's
    H2D and D2H copy lies inside it while copies overlap neighbouring steps' passes.
    No L2 flush: each step streams > 126 MB (L2) of host data in and out."""
    import torch
    stream = torch.cuda.ExternalStream(ctx.L.nau_get_stream(ctx.h))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        ctx.io_fence()
        for _ in range(steps):
            fn(ctx)
        ctx.io_join()
        e1.record(stream)
    stream.synchronize()
    ctx.sync()
    return e0.elapsed_time(e1)


def run_ours(args, dist):
    import torch
    from paper_1710_08259_b200 import nau

    use_slab = args.config in (0, 2, 3, 4) and (args.slab or dist.world > 1)
    wl = make_workload(args.config, dist, use_slab, args.comm == "native")
    ctx = nau.Context(dist.local)
    ctx.set_mode(args.mode == "fast")
    # one stream for everything: torch's row tensors, copies and collectives run in the
    # context's stream order (warm-up steps included), never beside the library's kernels
    torch.cuda.set_stream(torch.cuda.ExternalStream(ctx.L.nau_get_stream(ctx.h)))
    wl.setup(ctx)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{dist.local}")
    for _ in range(args.warmup):
        wl.step(ctx)
    ctx.sync()
    # ---- device-resident timed region (no per-kernel events: the step may replay as a
    # CUDA graph, nau_wcsph_step) ----
    clocks = Clocks(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.launches
    ms = timed_steps(ctx, wl.step, args.steps, flush)
    launches = ctx.launches - l0
    clk = clocks.stop()
    torch.cuda.synchronize()
    dist.barrier()
    # ---- per-kernel times: a second pass of the same steps with launch events ----
    ctx.profile(True)
    ms_prof = timed_steps(ctx, wl.step, args.steps, flush)
    prof = {cls: ctx.profile_ms(cls) for cls in wl.kernels}
    if not any(c for _, c in prof.values()):
        print("profile empty:", prof, ctx.L.nau_last_error(ctx.h, None), file=sys.stderr)
    ctx.profile(False)
    ms_max = dist.max(ms)
    n_total = dist.sum(float(wl.n_active))
    value = n_total * args.steps / (ms_max * 1e-3)
    # ---- end-to-end through the C-ABI with host buffers ----
    for _ in range(2):
        wl.e2e_step(ctx)
    dist.barrier()
    ms_e2e = dist.max(timed_pipelined(ctx, wl.e2e_step, args.steps))
    e2e = n_total * args.steps / (ms_e2e * 1e-3)
    # ---- roofline of the dominant kernel ----
    # T* = max(B / BW_HBM, F / P_FP64) with B, F the algorithmic bytes and flops of one
    # launch; frac = T* / T (T = mean CUDA-event launch time on the context stream).
    peaks, peak_kind = measured_peaks()
    hbm_peak = peaks["hbm_gbs"]
    fp64_peak = nau.fp64_peak_tflops(dist.local)
    fp64_src = ("builder-measured: nau_fp64_peak_tflops (csrc/fp64peak.cu, independent DFMA "
                "chains on every SM) in this run; MEASURED_PEAKS.json has no FP64 figure")
    traffic = ncu_traffic(args.config if args.mode == "fast" else f"{args.config}_exact")

    def tstar(B, F):
        t_hbm = B / (hbm_peak * 1e9)
        t_fp = F / (fp64_peak * 1e12)
        return max(t_hbm, t_fp), ("hbm" if t_hbm >= t_fp else "fp64")

    per_kernel = {}
    for cls, (label, B, F) in wl.kernels.items():
        tot, cnt = prof[cls]
        if cnt == 0:
            continue
        t = tot / cnt * 1e-3
        ts, bnd = tstar(B, F)
        tr = traffic.get(label)
        per_kernel[label] = {"ms_per_launch": round(tot / cnt, 4), "launches": cnt,
                             "share_of_step": round(tot / ms_prof, 4), "bound": bnd,
                             "t_star_ms": round(ts * 1e3, 4), "frac": round(ts / t, 4),
                             "algorithmic_GB_s": round(B / t / 1e9, 1),
                             "fp64_TFLOP_s": round(F / t / 1e12, 3) if F else 0.0,
                             "dram_bytes_ncu": tr.get("dram_bytes") if isinstance(tr, dict) else tr}
    dom_cls = max((c for c in wl.kernels if prof[c][1]), key=lambda c: prof[c][0])
    label, B, F = wl.kernels[dom_cls]
    tot, cnt = prof[dom_cls]
    t = tot / cnt * 1e-3
    ts, bnd = tstar(B, F)
    tr = traffic.get(label)
    dram = tr.get("dram_bytes") if isinstance(tr, dict) else tr
    roofline = {
        "kernel": label, "bound": bnd,
        "achieved": round(F / t / 1e12, 3) if bnd == "fp64" else round(B / t / 1e9, 1),
        "peak": round(fp64_peak, 2) if bnd == "fp64" else hbm_peak,
        "unit": "TFLOP/s" if bnd == "fp64" else "GB/s",
        "frac": round(ts / t, 4),
        "traffic": dram,
        "algorithmic_bytes": B, "algorithmic_flops": F,
        "traffic_overhead": (round(dram / B, 2) if dram else None),
        "hbm": {"achieved_GB_s": round(B / t / 1e9, 1), "peak": hbm_peak,
                "frac": round(B / t / 1e9 / hbm_peak, 4), "peak_source": peak_kind},
        "fp64": {"achieved_tflops": round(F / t / 1e12, 3), "peak_tflops": round(fp64_peak, 2),
                 "frac": round(F / t / 1e12 / fp64_peak, 4), "peak_source": fp64_src,
                 "issued_flops_ncu": tr.get("fp64_flops") if isinstance(tr, dict) else None},
        "note": ("B and F are SURVEY.md §8(d)'s per-particle figures x N (F charges 8 flops per "
                 "stencil candidate plus the per-neighbour flops); achieved = F / mean "
                 "CUDA-event launch time; frac = T*/T with T* = max(B/BW_HBM, F/P_FP64); "
                 "traffic = ncu DRAM bytes per launch (profiles/traffic.json), "
                 "traffic_overhead = traffic / B (neighbour-list and stencil re-reads)"),
    }
    if wl.survey:  # the whole step against T* = max(B / BW_HBM, F / P_FP64), SURVEY.md §8(d)
        Bs, Fs, basis = wl.survey
        t_hbm = Bs / (hbm_peak * 1e9) * 1e3
        t_fp = Fs / (fp64_peak * 1e12) * 1e3
        roofline["step"] = {"t_star_ms": round(max(t_hbm, t_fp), 4), "hbm_ms": round(t_hbm, 4),
                            "fp64_ms": round(t_fp, 4),
                            "frac": round(max(t_hbm, t_fp) / (ms_max / args.steps), 4),
                            "flops": basis}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "particle-updates/s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if use_slab else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(wl.config(), mode=args.mode,
                       parallelism=((f"bodies sharded over {dist.world} GPU(s), NCCL all-gather"
                                     if args.config == 4 else
                                     f"x-slabs over {dist.world} GPU(s), NCCL halo+migration")
                                    if use_slab else
                                    ("replicas" if dist.world > 1 else "single GPU")),
                       l2="flushed between timed steps (256 MiB memset, untimed)"),
        "e2e": {"value": round(e2e, 1), "unit": "particle-updates/s",
                "h2d_bytes_per_step": int(wl.h2d), "d2h_bytes_per_step": int(wl.d2h),
                "ms_per_step": round(ms_e2e / args.steps, 4),
                "timing": ("K steps as one device interval; per step r, v (A) uploaded from "
                           "and results downloaded to pinned host memory via "
                           "nau_upload_async / nau_download_async (copy streams overlap "
                           "neighbouring steps' passes); no L2 flush: each step streams "
                           "more than L2 through host copies")},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "kernels": per_kernel,
        "clocks": clk,
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, wl, full_steps=REF_FULL_STEPS[args.config]
                                            if args.config in (0, 2) else None)
    # torch tensors allocated inside the ExternalStream(ctx stream) regions must be
    # released before the context destroys that stream
    import gc
    torch.cuda.synchronize()
    wl = None
    gc.collect()
    torch.cuda.synchronize()
    ctx.close()
    return line


# ----------------------------------------------------- CPU reference ----
def _ref_deck(config, sc):
    """The workload as a reference Case (oracle/_ref: the unmodified reference sources),
    assembled the way tests/helpers.hpp:26-80 does, with its equations in deck order.
    Returns (case, equations as (name, text), components per RHS, note)."""
    from oracle import ref
    prm = sc.params
    rc = ref.RefCase(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds, sc.pos)
    if config == 1:
        rc.field("A", sc.fields["A"]).field("rho", np.full(sc.n, prm["rho0"]))
        rc.field("G", np.zeros((3, sc.n))).field("L", np.zeros(sc.n))
        rc.constant("one", 1.0).constant("m", prm["mass"]).constant("R", prm["radius"])
        eqs = [("density", "rho=sph_S(one,m,one,Wp53220,R)"),
               ("gradient", "G=sph_G11(A,m,rho,Wp53220,R)"),
               ("laplacian", "L=sph_L0(A,m,rho,Wp53220,R)")]
        comps = [1, 3, 1]
        note = "Wendland Wp53220 (the reference has no cubic spline; same candidate loop)"
    elif config == 3:
        rng = np.random.default_rng(0)
        rc.field("v", rng.uniform(-0.01, 0.01, (3, sc.n))).field("vdot", sc.fields["vdot"])
        rc.field("R", sc.fields["R"]).field("m", sc.fields["m"])
        rc.constant("E", 2.06e6).constant("nu", 0.33).constant("cf", prm["cf"])
        rc.constant("Rs", prm["search_radius"]).constant("g", prm["g"]).variable("dt", prm["dt"])
        eqs = [("accel", "vdot=dem_l(v,R,E,nu,m,cf,Rs)+g"), ("velocity", "v=euler(v,vdot,dt)"),
               ("position", "r=euler(r,v,dt)")]
        comps = [3, 3, 3]
        note = ("the reference's stock Hertz dem_l through the same contact loop "
                "(it has no linear spring-dashpot law)")
    elif config == 4:
        rc.field("v", sc.fields["v"]).field("a", sc.fields["a"])
        rc.constant("m", prm["m"]).constant("G", prm["G"]).constant("eps", prm["eps"])
        rc.variable("dth", 0.5 * prm["dt"]).variable("dt", prm["dt"])
        eqs = [("kick1", "v=euler(v,a,dth)"), ("drift", "r=euler(r,v,dt)"),
               ("force", "a=nbody_gravity(m,G,eps)"), ("kick2", "v=euler(v,a,dth)")]
        comps = [3, 3, 3, 3]
        note = "nbody_gravity all pairs (interactions.cpp:195-214), leapfrog as equation order"
    else:
        rng = np.random.default_rng(0)
        vel = rng.uniform(-0.1, 0.1, (sc.dim, sc.n))  # non-zero so sph_A does its full work
        for k in ("rho", "p", "vdot", "mask"):
            rc.field(k, sc.fields[k])
        rc.field("v", vel)
        rc.constant("one", 1.0).constant("mass", prm["mass"]).constant("R", prm["radius"])
        rc.constant("B", prm["B"]).constant("rho0", prm["rho0"]).constant("gam", prm["gamma"])
        rc.constant("visc", prm["visc"]).constant("g", prm["g"]).variable("dt", prm["dt"])
        eqs = scenes_wcsph(sc)
        comps = [1, 1, sc.dim, sc.dim, sc.dim]
        note = f"Wendland Wp5{sc.dim}220"
    for name, text in eqs:
        rc.equation(name, text)
    return rc, eqs, comps, note


def scenes_wcsph(sc):
    from paper_1710_08259_b200 import scenes
    return scenes.wcsph_equations(sc)


def _scene(config):
    from paper_1710_08259_b200 import scenes
    return {1: scenes.sph_microbench, 2: lambda: scenes.dam_break(3, dx=0.005),
            0: lambda: scenes.dam_break(2), 3: scenes.dem_column, 4: scenes.plummer}[config]()


def cpu_baseline(args, wl=None, full_steps=None, sample_steps=None):
    """Time the reference's own CPU path (oracle/_ref) on the box's host cores:
    (1) `full_steps` full-N Case::solve_step(ThreadPool(P)) calls (SURVEY.md §8(d)'s
    anchor; skipped when None), and (2) the bounded sample estimate: build_cells over
    all particles + every equation's RHS over a spread sample of particles."""
    from oracle import ref
    threads = os.cpu_count() or 1
    if not ref.available():
        return cpu_baseline_port(args)
    sc = wl.sc if wl else _scene(args.config)
    rc, eqs, comps, kernel_note = _ref_deck(args.config, sc)
    exprs = [t.split("=", 1)[1] for _, t in eqs]
    n = sc.n
    t0 = time.perf_counter()
    rc.build_cells()
    t_build = time.perf_counter() - t0

    def sample_cost(count):
        chunks = 8
        per = max(1, count // chunks)
        t = 0.0
        for e, c in zip(exprs, comps):
            for k in range(chunks):
                i0 = min(n - per, int((k + 0.5) * n / chunks))
                s = time.perf_counter()
                rc.eval(e, c, i0=i0, count=per, threads=threads)
                t += time.perf_counter() - s
        return t, per * chunks

    t, cnt = sample_cost(64 * threads)
    target = max(1.0, args.cpu_seconds - t_build)
    scale = target / max(t, 1e-6)
    cnt2 = int(min(n, max(cnt, cnt * scale)))
    t, cnt = sample_cost(cnt2)
    per_particle = t_build / n + t / cnt
    est = 1.0 / per_particle
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                 if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = "unknown"
    sample = (f"sample estimate: build_cells over all {n} particles ({t_build:.2f} s, "
              f"single-threaded as in the reference) + every equation's RHS over {cnt} particles "
              f"in 8 spread chunks on ThreadPool({threads}) ({t:.2f} s)")
    out = {"unit": "particle-updates/s", "cores": threads, "kind": "reference",
           "sample_estimate": round(est, 1)}
    if full_steps:
        # the full deck: lazy build_cells, every equation over all N, staging, NaN audit,
        # swap, boundary shift (Case::solve_step, case.cpp:9-67) on ThreadPool(P)
        rc.boundary_shift()
        ts = []
        for _ in range(full_steps):
            s0 = time.perf_counter()
            rc.solve_step(threads)
            ts.append(time.perf_counter() - s0)
        t_full = sum(ts)
        out["value"] = round(n * full_steps / t_full, 1)
        out["full_steps"] = {"steps": full_steps, "seconds": round(t_full, 2),
                             "per_step_s": [round(x, 3) for x in ts]}
        out["sample"] = (f"reference Case path (oracle/_ref, unmodified sources): {full_steps} "
                         f"full-N Case::solve_step(ThreadPool({threads})) over all {n} particles "
                         f"({t_full:.2f} s; value = N x steps / that time); {sample} gives "
                         f"{est:.4g}; {kernel_note}; host CPU: {model}")
    else:
        out["value"] = round(est, 1)
        out["sample"] = (f"reference Case path (oracle/_ref, unmodified sources): {sample}; "
                         f"{kernel_note}; host CPU: {model}")
    if sample_steps:
        # the reference arm's K timed steps: each a bounded sample of the step (a full
        # build_cells + every equation's RHS over the same spread particles), sized so that
        # warm-up + K steps take ~2 minutes; the full-N anchor above stays the value
        k_steps, w_steps = sample_steps
        budget = 120.0 / max(1, k_steps + w_steps)
        per_rhs = t / cnt
        ns = int(min(n, max(64 * threads, (budget - t_build) / max(per_rhs, 1e-12))))

        def one():
            s0 = time.perf_counter()
            rc.build_cells()
            _, m = sample_cost(ns)
            return time.perf_counter() - s0, m

        for _ in range(w_steps):
            one()
        ts, m = [], ns
        for _ in range(k_steps):
            dt_s, m = one()
            ts.append(dt_s)
        mean = sum(ts) / max(len(ts), 1)
        out["sample_steps"] = {"steps": k_steps, "warmup": w_steps, "particles_per_step": m,
                               "mean_s": round(mean, 4), "min_s": round(min(ts), 4),
                               "max_s": round(max(ts), 4),
                               "full_step_estimate": round(1.0 / (t_build / n + (mean - t_build) / m), 1)}
    del rc
    return out


def cpu_baseline_port(args):
    return {"value": None, "unit": "particle-updates/s", "cores": 0, "kind": "port",
            "sample": "oracle/_ref not present on this machine"}


REF_FULL_STEPS = {0: 20, 1: 1, 2: 1, 3: 2, 4: 1}


def run_reference(args, dist):
    """The reference arm: the unmodified reference (oracle/_ref) on the box's host threads.
    `value` = N x steps / time of full-N Case::solve_step calls (the anchor SURVEY.md §8(d)
    asks for); the --steps K / --warmup W steps the contract counts are bounded SAMPLES of
    that step (a full build_cells + every equation's RHS over a fixed spread of particles),
    so ms_per_step x K is the wall time actually spent in them."""
    if dist.rank != 0:
        return None
    cb = cpu_baseline(args, full_steps=REF_FULL_STEPS[args.config],
                      sample_steps=(args.steps, args.warmup))
    n = _scene(args.config).n if cb["value"] else None
    ss = cb.get("sample_steps")
    per_step_ms = ss["mean_s"] * 1e3 if ss else (n / cb["value"] * 1e3 if cb["value"] else None)
    return {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "particle-updates/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms,
            "ms_per_full_step": (n / cb["value"] * 1e3) if cb["value"] else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES[args.config], "threads": cb["cores"],
                       "timed": (f"value: {cb.get('full_steps', {}).get('steps')} full-N "
                                 "Case::solve_step call(s) on all host threads (the reference's "
                                 "whole step); steps/warmup/ms_per_step: bounded sample steps ("
                                 f"{ss['particles_per_step'] if ss else 0} particles' RHS + a full "
                                 "build_cells each), whose full-step estimate is "
                                 f"{ss['full_step_estimate'] if ss else None} particle-updates/s")},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "particle-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        line = run_reference(args, dist)
    else:
        line = run_ours(args, dist)
    if dist.rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
