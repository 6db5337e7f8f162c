"""Seeded synthetic inputs for the BASELINE.json configurations.

No dataset is involved: every input is generated here. Random draws use the
reference's counter RNG (RandomState, /root/reference/proj/include/nauticle/
sfl/random_state.hpp:22-41), restated vectorised so that draw k of particle i
equals the reference's k-th ``rand`` call at particle i (pinned in
tests/test_oracle.py against oracle/_ref).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(x):
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def uniform_draws(seed: int, n: int, ndraws: int, a=0.0, b=1.0) -> np.ndarray:
    """out[k, i] = RandomState(seed).uniform(i, a, b) at its k-th call for particle i."""
    with np.errstate(over="ignore"):
        s = _mix(np.uint64(seed) ^ np.uint64(0x6E61757469636C65))
        pi = _mix(np.arange(n, dtype=np.uint64) + np.uint64(0x9E3779B9))
        out = np.empty((ndraws, n), np.float64)
        for k in range(ndraws):
            x = _mix(s ^ pi ^ np.uint64(k))
            u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            out[k] = a + u * (b - a)
    return out


@dataclass
class Scene:
    name: str
    dim: int
    min_cells: list
    max_cells: list
    cell_size: list
    kinds: list
    pos: np.ndarray                      # (dim, n)
    fields: dict = field(default_factory=dict)   # name -> (comps, n) or (n,)
    params: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.pos.shape[1]


# ---------------------------------------------------------------- cfg1 ----
def sph_microbench(n=1_048_576, seed=1, neighbours=50.0, rho0=1000.0) -> Scene:
    """BASELINE cfg1: N uniform-random particles in the periodic unit cube.

    2h is chosen so the expected neighbour count within 2h is `neighbours`
    (excluding self): (4/3) pi (2h)^3 N = neighbours. The domain needs an
    integer number of cells (domain.hpp:26-30): floor(1/2h) cells of 1/that.
    Draws 0,1,2 of particle i are x,y,z; draw 3 is the scalar field A.
    """
    two_h = (3.0 * neighbours / (4.0 * math.pi * n)) ** (1.0 / 3.0)
    cells = int(math.floor(1.0 / two_h))
    cs = 1.0 / cells
    d = uniform_draws(seed, n, 4)
    # draws are in [0,1); the computed domain is [0, cells*cs) (== 1.0 for 44 cells)
    hi = cells * cs
    pos = np.ascontiguousarray(d[:3] * hi if hi != 1.0 else d[:3])
    return Scene("sph_microbench", 3, [0, 0, 0], [cells] * 3, [cs] * 3, [0, 0, 0], pos,
                 fields={"A": d[3].copy()},
                 params={"radius": two_h, "h": 0.5 * two_h, "mass": rho0 / n, "rho0": rho0})


# ------------------------------------------------------------ cfg0 / cfg2 ----
def _lattice(box_lo, box_hi, dx):
    """Cell-centred lattice points ((i+1/2) dx per axis) of an index box [lo, hi)."""
    axes = [(np.arange(l, h, dtype=np.float64) + 0.5) * dx for l, h in zip(box_lo, box_hi)]
    if any(len(a) == 0 for a in axes):
        return np.zeros((len(axes), 0))
    mesh = np.meshgrid(*axes, indexing="ij")
    # axis 0 fastest in the flattened order
    return np.stack([m.transpose(tuple(range(len(axes)))[::-1]).ravel() for m in mesh])


def dam_break(dim=2, dx=0.01, fluid=None, tank=None, layers=3, rho0=1000.0, gravity=9.81,
              alpha=0.02, cfl=0.2, gamma=7.0, kernel_family=0) -> Scene:
    """BASELINE cfg0 (2D, defaults) / cfg2 (dim=3, dx=0.005): WCSPH dam break.

    Fluid block at ((i+1/2)dx, ...) from the origin; `layers` of fixed wall
    particles on the floor and the side walls of the tank (open top). Wendland
    C2 with h = 2 dx, cell size 2h, Tait EOS with c0 = 10 sqrt(2 g H), gamma = 7,
    artificial viscosity alpha, dt = cfl h / c0. Walls carry mask 0.
    """
    if fluid is None:
        fluid = (1.0, 2.0) if dim == 2 else (1.0, 0.5, 1.0)
    if tank is None:
        tank = (4.0, 3.0) if dim == 2 else (3.2, 1.0, 1.5)
    nf = [int(round(f / dx)) for f in fluid]
    nt = [int(round(t / dx)) for t in tank]
    fpos = _lattice([0] * dim, nf, dx)
    L = layers
    boxes = []
    if dim == 2:
        boxes.append(([-L, -L], [nt[0] + L, 0]))          # floor incl. corners
        boxes.append(([-L, 0], [0, nt[1]]))               # left wall
        boxes.append(([nt[0], 0], [nt[0] + L, nt[1]]))    # right wall
    else:
        boxes.append(([-L, -L, -L], [nt[0] + L, nt[1] + L, 0]))
        boxes.append(([-L, -L, 0], [0, nt[1] + L, nt[2]]))
        boxes.append(([nt[0], -L, 0], [nt[0] + L, nt[1] + L, nt[2]]))
        boxes.append(([0, -L, 0], [nt[0], 0, nt[2]]))
        boxes.append(([0, nt[1], 0], [nt[0], nt[1] + L, nt[2]]))
    wpos = np.concatenate([_lattice(lo, hi, dx) for lo, hi in boxes], axis=1)
    pos = np.ascontiguousarray(np.concatenate([fpos, wpos], axis=1))
    n_f, n = fpos.shape[1], pos.shape[1]
    h = 2.0 * dx
    radius = 2.0 * h
    cell = radius
    H = fluid[-1]
    c0 = 10.0 * math.sqrt(2.0 * gravity * H)
    B = c0 * c0 * rho0 / gamma
    mass = rho0 * dx ** dim
    dt = cfl * h / c0
    g = [0.0] * dim
    g[-1] = -gravity
    max_cells = [int(math.ceil(t / cell - 1e-9)) + 1 for t in tank]
    min_cells = [-1] * dim
    mask = np.zeros(n)
    mask[:n_f] = 1.0
    # initial hydrostatic density via the inverse Tait EOS (walls at rho0)
    rho = np.full(n, rho0)
    depth = H - fpos[-1]
    rho[:n_f] = rho0 * (1.0 + rho0 * gravity * depth / B) ** (1.0 / gamma)
    return Scene(
        f"dam_break_{dim}d", dim, min_cells, max_cells, [cell] * dim, [2] * dim, pos,
        fields={"rho": rho, "p": np.zeros(n), "v": np.zeros((dim, n)), "vdot": np.zeros((dim, n)),
                "mask": mask},
        params={"dx": dx, "h": h, "radius": radius, "mass": mass, "rho0": rho0, "c0": c0, "B": B,
                "gamma": gamma, "alpha": alpha, "visc": alpha * c0 * h, "dt": dt, "g": g,
                "n_fluid": n_f, "kernel_family": kernel_family})


# ---------------------------------------------------------------- cfg3 ----
def _rsa_place(R, box, seed, max_tries=100000):
    """Seeded random sequential addition (csrc/scenes_rsa.c, libnau_scenes.so): sphere s
    in index order, attempt t at a uniform centre in [R_s, box - R_s] drawn with the
    reference's counter RNG (seed + 1 + t, particle s, draws 0-2), accepted when it
    overlaps no earlier sphere (hash grid of cell 2 max R)."""
    import ctypes as C
    import os
    lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnau_scenes.so"))
    lib.nau_rsa_place.restype = C.c_long
    lib.nau_rsa_place.argtypes = [C.c_long, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
    R = np.ascontiguousarray(R, np.float64)
    b = np.ascontiguousarray(box, np.float64)
    pos = np.zeros((3, len(R)))
    rc = lib.nau_rsa_place(len(R), R.ctypes.data, b.ctypes.data, seed, max_tries, pos.ctypes.data)
    if rc:
        raise RuntimeError(f"random sequential addition: sphere {rc - 1} unplaced")
    return pos


def dem_column(n=2_000_000, seed=3, box=(0.3, 0.3, 1.2), median=1e-3, sigma=0.2,
               rho_s=2500.0, kn=1e5, en=0.5, mu=0.5, dt=1e-6, gravity=9.81,
               placement="rsa") -> Scene:
    """BASELINE cfg3: n spheres, log-normal radii (median, sigma_log; untruncated) from
    Box-Muller on draws 0,1 of the reference RNG, at seeded random-sequential-addition
    positions (non-overlapping, _rsa_place) in the column, settling under gravity with
    symmetric (mirror-image) walls — the floor is the z-low wall (interactions.cpp:168-170
    mirror mechanism). Linear spring-dashpot normal force k_n, restitution e_n, Coulomb
    friction mu; cell = search radius = 2 r_max (the largest realised radius).
    placement="lattice": the round-1 jittered cubic lattice (radii clamped at 0.95 s/2)."""
    d = uniform_draws(seed, n, 5)
    u1 = np.maximum(d[0], 2.0 ** -53)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * d[1])
    R = median * np.exp(sigma * z)
    if placement == "rsa":
        pos = np.ascontiguousarray(_rsa_place(R, box, seed))
        s = None
    else:
        s = (box[0] * box[1] * box[2] / n) ** (1.0 / 3.0)
        nx, ny = int(box[0] / s), int(box[1] / s)
        nz = int(math.ceil(n / (nx * ny)))
        s = min(box[0] / nx, box[1] / ny, box[2] / nz)
        R = np.minimum(R, 0.95 * 0.5 * s)
        k = np.arange(n)
        site = np.stack([(k % nx + 0.5) * s, ((k // nx) % ny + 0.5) * s, (k // (nx * ny) + 0.5) * s])
        room = 0.5 * s - R  # jitter keeps every sphere inside its lattice cube
        pos = np.ascontiguousarray(site + (2.0 * d[2:5] - 1.0) * room * 0.999)
    rmax = float(R.max())
    cs = 2.0 * rmax
    cells = [int(math.ceil(b / cs)) for b in box]
    m = rho_s * 4.0 / 3.0 * math.pi * R ** 3
    return Scene("dem_column", 3, [0, 0, 0], cells, [cs] * 3, [1, 1, 1], pos,
                 fields={"v": np.zeros((3, n)), "vdot": np.zeros((3, n)), "R": R, "m": m},
                 params={"kn": kn, "en": en, "cf": mu, "dt": dt, "g": [0.0, 0.0, -gravity],
                         "search_radius": cs, "rho_s": rho_s, "lattice": s,
                         "placement": placement})


def dem_equations():
    """The DEM deck as SFL equation text (dem_lsd is registered beside dem_l)."""
    return [("accel", "vdot=dem_lsd(v,R,kn,en,m,cf,Rs)+g"), ("velocity", "v=euler(v,vdot,dt)"),
            ("position", "r=euler(r,v,dt)")]


# ---------------------------------------------------------------- cfg4 ----
def plummer(n=262_144, seed=4, eps=0.01, dt=1e-3, rmax=10.0) -> Scene:
    """BASELINE cfg4: Plummer sphere, G = M = a = 1, m = 1/n, seeded draws of the
    reference RNG: inverse-CDF radius (truncated at rmax), isotropic directions,
    speed q v_esc with q rejection-sampled from q^2 (1 - q^2)^(7/2); centre of mass
    and momentum removed. A cut-off box far outside rmax (escapers deactivate,
    particle_system.cpp:77-84)."""
    tries = 64
    d = uniform_draws(seed, n, 5 + 2 * tries)
    xmax = (rmax * rmax / (1.0 + rmax * rmax)) ** 1.5
    X = np.maximum(d[0] * xmax, 1e-300)
    r = 1.0 / np.sqrt(X ** (-2.0 / 3.0) - 1.0)
    ct = 2.0 * d[1] - 1.0
    st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
    ph = 2.0 * math.pi * d[2]
    pos = np.stack([r * st * np.cos(ph), r * st * np.sin(ph), r * ct])
    q = np.full(n, 0.5)
    done = np.zeros(n, bool)
    for t in range(tries):
        qt, yt = d[5 + 2 * t], 0.1 * d[6 + 2 * t]
        acc = ~done & (yt < qt * qt * (1.0 - qt * qt) ** 3.5)
        q[acc] = qt[acc]
        done |= acc
    vesc = math.sqrt(2.0) * (1.0 + r * r) ** -0.25
    ct2 = 2.0 * d[3] - 1.0
    st2 = np.sqrt(np.maximum(0.0, 1.0 - ct2 * ct2))
    ph2 = 2.0 * math.pi * d[4]
    v = np.stack([st2 * np.cos(ph2), st2 * np.sin(ph2), ct2]) * (q * vesc)
    pos -= pos.mean(axis=1, keepdims=True)
    v -= v.mean(axis=1, keepdims=True)
    box = rmax + 5.0
    return Scene("plummer", 3, [-1, -1, -1], [1, 1, 1], [box] * 3, [2, 2, 2],
                 np.ascontiguousarray(pos),
                 fields={"v": np.ascontiguousarray(v), "a": np.zeros((3, n))},
                 params={"m": 1.0 / n, "G": 1.0, "eps": eps, "dt": dt})


def wcsph_equations(scene: Scene, kernel_keyword=None):
    """The dam-break deck as SFL equation text (for the reference oracle)."""
    kw = kernel_keyword or f"Wp5{scene.dim}220"
    return [
        ("density", f"rho=sph_S(one,mass,one,{kw},R)"),
        ("eos", "p=B*((rho/rho0)^gam-1)"),
        ("momentum", f"vdot=-1/rho*sph_G11(p,mass,rho,{kw},R)+visc*sph_A(v,mass,rho,{kw},R)+g"),
        ("velocity", "v=euler(v,vdot*mask,dt)"),
        ("position", "r=euler(r,v,dt)"),
    ]
