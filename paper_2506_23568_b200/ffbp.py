"""HHFFBPA on the GPU: the drop-in for hhsar.ffbp.

Reference: /root/reference/pkg/src/hhsar/ffbp.py.  ``hhffbpa_reconstruct``
keeps its signature, provenance keys and exceptions.  The reference's Python
loops over subarrays (ffbp.py:470-492) become a fixed sequence of batched
launches on one stream:

  1. hhsar_leaf_boxes + hhsar_grid_plan -- lattice metadata of EVERY grid of
     EVERY level at once (bit-exact float64), then one device->host copy of
     the small descriptors to size the lattice pools (the only mid-pipeline
     synchronisation);
  2. hhsar_grid_newton -- every (u, v) column of every grid, warm-started
     along n, pruned to the near band, with containment / near / leaf delay
     masks and per-grid counters;
  3. hhsar_leaf_bp -- all leaves, downconverted on store;
  4. hhsar_merge_level per merge stage -- all parents of a level at once;
  5. hhsar_merge_cartesian -- the final landing on the region grid;
then one device->host copy of the volume and counters, after which the
reference's error checks run in the reference's order.

``merge_factor`` (keyword, default 2 = the reference's binary tree) selects
the N-ary schedule BASELINE configs 0/2/4 ask for: grids only at tree levels
1, 1+s, 1+2s, ... (merge factor 2^s) and every merge sums 2^s children with
the reference's N-ary _merge_onto_points (ffbp.py:351-374).
"""

from __future__ import annotations

from dataclasses import dataclass

import functools

import numpy as np

from . import _native
from .bpa import (ImageVolume, _finish, bpa_volume_device, check_delay_window,
                  default_grid_dims, el_f32x4, region_grid)
from .errors import ConfigError, NumericDomainError
from .model import (C_LIGHT, Subarray, boundary_lattice, leaf_bounds,
                    partition_subarrays, validate_geometry)
from .rangecomp import CubeUpload, RangeProfileSet, profile_axis, range_compress, to_device_cube
from .spectrum import TWO_PI, SubarrayExtents

GRID_PAD = 2  # ffbp.py:32
MAX_NEWTON_ITER = 126  # HHSAR_MAX_NEWTON_ITER (include/hhsar_b200.h)
BOUNDARY_PER_AXIS = 5  # ffbp.py:237


def default_levels(aperture) -> int:
    """ffbp.py:35-39: max(1, floor(log2(min(nx, ny))) - 2)."""
    side = min(aperture.nx, aperture.ny)
    return max(1, int(np.floor(np.log2(side))) - 2)


@dataclass(frozen=True)
class FfbpParams:
    """Tuning knobs (ffbp.py:42-71), same validation."""

    levels: int | None = None
    gamma: float = 1.4
    kernel: str = "linear"
    margin: float = 0.25

    def __post_init__(self):
        if self.levels is not None and self.levels < 1:
            raise ConfigError("levels must be at least 1")
        if not self.gamma >= 1.0:
            raise ConfigError("oversampling factor must be at least 1")
        if self.kernel not in ("linear", "cubic"):
            raise ConfigError(f"unknown interpolation kernel '{self.kernel}'")
        if not 0.0 <= self.margin <= 1.0:
            raise ConfigError("margin must lie in [0, 1]")


def _kernel_id(kernel: str) -> int:
    if kernel == "linear":
        return 0
    if kernel == "cubic":
        return 1
    raise ConfigError(f"unknown interpolation kernel '{kernel}'")


# ---------------------------------------------------------------------------
# schedule (host, O(#subarrays))
# ---------------------------------------------------------------------------

class Schedule:
    """Which subarrays carry grids, in launch order, and the merge fan-outs.

    Subarray j of 1-based tree level L covers leaves [j 2^(L-1), (j+1) 2^(L-1))
    (model.py:383-386 pairs consecutive children).
    """

    @staticmethod
    @functools.lru_cache(maxsize=16)
    def shared(n_elements: int, levels: int, merge_factor: int = 2) -> "Schedule":
        """Memoised, read-only schedule (a pure function of three integers)."""
        sc = Schedule(n_elements, levels, merge_factor)
        for a in (sc.grids, sc.bounds):
            a.setflags(write=False)
        return sc

    def __init__(self, n_elements: int, levels: int, merge_factor: int = 2):
        s = int(round(np.log2(merge_factor)))
        if merge_factor < 2 or 2 ** s != merge_factor:
            raise ConfigError("merge factor must be a power of two >= 2")
        self.levels = levels
        self.merge_factor = merge_factor
        self.bounds = leaf_bounds(n_elements, levels)
        self.n_leaves = len(self.bounds) - 1
        self.grid_levels = list(range(1, levels, s)) or [1]
        rows, self.level_slices = [], []
        for lev in self.grid_levels:
            span = 1 << (lev - 1)
            lf0 = np.arange(0, self.n_leaves, span)
            g0 = sum(len(r) for r in rows)
            rows.append(lf0)
            self.level_slices.append((g0, g0 + lf0.size))
        lf0 = np.concatenate(rows)
        span = np.concatenate([np.full(r.size, 1 << (lev - 1)) for r, lev in
                               zip(rows, self.grid_levels)])
        g = np.zeros(lf0.size, dtype=_native.GRID_DTYPE)
        g["leaf_lo"] = lf0
        g["leaf_hi"] = lf0 + span
        g["start"] = self.bounds[lf0]
        g["stop"] = self.bounds[lf0 + span]
        g["is_leaf"] = span == 1
        self.grids = g
        # children per parent for each merge stage, and for the final landing
        self.fanouts = [1 << (b - a) for a, b in zip(self.grid_levels[:-1], self.grid_levels[1:])]
        last = self.level_slices[-1]
        self.final_children = last[1] - last[0]

    @property
    def n_grids(self) -> int:
        return self.grids.size


def make_geom(region, kgrid, gamma: float, margin: float, pad: int, window_hi: float,
              tol: float = 1e-9, max_iter: int = 50, z_floor: float = 1e-4) -> np.ndarray:
    """hhsar_geom with every constant computed in float64 exactly as the
    reference computes it (spectrum.py:256-272, ffbp.py:241-269).  Cached
    per argument set (read-only: native calls only read it)."""
    k_min, k_max = kgrid.k_min, kgrid.k_max
    key = (_region_tuple(region), float(k_min), float(k_max), float(gamma), float(margin),
           int(pad), float(window_hi), float(tol), int(max_iter), float(z_floor))
    hit = _GEOMS.get(key)
    if hit is not None:
        return hit
    extents = (region.x_max - region.x_min, region.y_max - region.y_min,
               region.z_max - region.z_min)
    diag = float(getattr(region, "diagonal", np.linalg.norm(extents)))
    center = [(region.x_min + region.x_max) / 2, (region.y_min + region.y_max) / 2,
              (region.z_min + region.z_max) / 2]
    geom = _native.host_struct(_native.GEOM_DTYPE, dict(
        region=[region.x_min, region.x_max, region.y_min, region.y_max, region.z_min,
                region.z_max],
        center=center, k_min=k_min, k_max=k_max, c_uv=k_max / np.pi,
        c_nhi=k_max / (2.0 * TWO_PI), c_nlo=k_min / (2.0 * TWO_PI),
        step=np.full(3, 1.0 / gamma)[0], margin=margin, max_step=0.5 * diag, tol=tol,
        z_floor=z_floor, window_hi=window_hi, pad=pad, max_iter=max_iter))
    geom.setflags(write=False)
    if len(_GEOMS) > 64:
        _GEOMS.clear()
    _GEOMS[key] = geom
    return geom


_GEOMS = {}


# ---------------------------------------------------------------------------
# device lattices
# ---------------------------------------------------------------------------

# the landing gathers from a (v[i], v[i+1]) pair-staged copy of the top
# lattices (hhsar_merge_cartesian span arguments); False gathers directly
LANDING_PAIRS = True
# the landing evaluates z runs by series where accurate (hhsar_merge_cartesian
# picks); False forces the per-voxel float64 form (HHSAR_LANDING_PER_VOXEL)
LANDING_SERIES = True
LANDING_PER_VOXEL = 16


class Lattices:
    """All grids of a schedule on the device: descriptors + global pools.

    Pools are indexed by desc.offset: positions float64 [P,3] (valid points
    only are meaningful), valid uint8 [P], values complex64 [P] stored
    downconverted, stats int64 [G,6].
    """

    def __init__(self, descs, descs_dev, positions, valid, stats, geom):
        self.descs = descs
        self.descs_dev = descs_dev
        self.positions = positions
        self.valid = valid
        self.stats = stats
        self.geom = geom
        self.npts = np.prod(descs["dims"].astype(np.int64), axis=1)
        self.values = None
        self.gate = None

    def desc_ptr(self, g: int):
        import ctypes
        return ctypes.c_void_p(self.descs_dev.data_ptr() + int(g) * _native.GRID_DTYPE.itemsize)

    def points_in(self, g0: int, g1: int) -> int:
        return int(self.npts[g0:g1].sum())


def build_lattices(el_dev, sched: Schedule, region, kgrid, gamma: float, margin: float,
                   pad: int, window_hi: float, tol: float = 1e-9, max_iter: int = 50,
                   newton_grids=None, gate_dt=None, gate_bins: int = 0) -> Lattices:
    """Plan + Newton for every grid of the schedule (ffbp.py:179-307).

    Every grid is planned (metadata is cheap and needed by any rank that
    merges it); ``newton_grids`` (bool per grid) restricts the Newton
    inversion to the grids this process will actually evaluate points of
    (multi-GPU subtree ownership).  Unselected grids keep valid = 0 and zero
    counters.
    """
    pending = plan_lattices(el_dev, sched, region, kgrid, gamma, margin, pad, window_hi, tol,
                            max_iter, gate_dt, gate_bins)
    return finish_lattices(pending, newton_grids)


_PLAN_UPLOADS = {}


def _plan_upload(sched: Schedule, region):
    """Pinned host image of the plan's inputs -- grid descriptors | leaf
    bounds | boundary lattice | status word (8-byte aligned pieces) -- built
    once per (schedule, region) and reused: its content never changes and
    the device copy is taken asynchronously from it."""
    import torch
    key = (id(sched), sched.n_grids, tuple(float(v) for v in _region_tuple(region)))
    hit = _PLAN_UPLOADS.get(key)
    if hit is not None and hit[3] is sched:
        return hit[:3]
    bl = np.ascontiguousarray(boundary_lattice(region, BOUNDARY_PER_AXIS))
    parts = [sched.grids.view(np.uint8).reshape(-1), sched.bounds.astype(np.int64).view(np.uint8),
             bl.view(np.uint8).reshape(-1), np.zeros(40, dtype=np.uint8)]
    cuts = np.cumsum([0] + [p.size for p in parts])
    staged = torch.empty(int(cuts[-1]), dtype=torch.uint8, pin_memory=True)
    sn = staged.numpy()
    for p, a in zip(parts, cuts[:-1]):
        sn[a:a + p.size] = p
    if len(_PLAN_UPLOADS) > 8:
        _PLAN_UPLOADS.clear()
    _PLAN_UPLOADS[key] = (staged, cuts, bl.shape[0], sched)
    return staged, cuts, bl.shape[0]


_PLAN_DEVICE = {}


def _plan_device_inputs(staged, dev):
    import torch
    key = (staged.data_ptr(), staged.numel(), torch.device(dev).index)
    hit = _PLAN_DEVICE.get(key)
    if hit is None or hit[1] is not staged:
        if len(_PLAN_DEVICE) > 8:
            _PLAN_DEVICE.clear()
        hit = (staged.to(dev), staged)  # once, synchronous
        _PLAN_DEVICE[key] = hit
    return hit[0]


def _region_tuple(region):
    return (region.x_min, region.x_max, region.y_min, region.y_max, region.z_min, region.z_max)


def plan_lattices(el_dev, sched: Schedule, region, kgrid, gamma: float, margin: float, pad: int,
                  window_hi: float, tol: float = 1e-9, max_iter: int = 50, gate_dt=None,
                  gate_bins: int = 0, cached=None):
    """Launch the leaf boxes + plan kernels and the asynchronous readback of
    the descriptors (pinned) on the current stream; returns a pending plan
    for finish_lattices (which is the only host wait).  With ``gate_dt``
    (profile bin width) and ``gate_bins`` (profile length) the leaf range
    gate (hhsar_leaf_range_gate) comes back with the plan as lat.gate.

    ``cached`` (a PlanCache of an earlier plan of the SAME geometry): the
    plan kernels still run, but nothing is read back -- the host takes the
    descriptors and sizes from the cache, so no host wait remains and the
    step can be captured in a CUDA graph (StepGraph)."""
    import ctypes
    import torch
    dev = el_dev.device
    stream = _native.stream_handle()
    staged, cuts, n_b = _plan_upload(sched, region)
    up = torch.empty(staged.shape, dtype=torch.uint8, device=dev)
    if cached is not None:
        # a device-resident copy of the (constant) plan inputs: a D2D copy,
        # so the plan never queues behind cube uploads in the H2D engine
        up.copy_(_plan_device_inputs(staged, dev), non_blocking=True)
    else:
        up.copy_(staged, non_blocking=True)
    if _trace:
        _trace("plan inputs up")
    descs_dev = up[cuts[0]:cuts[1]]
    bounds = up[cuts[1]:cuts[2]]
    boundary = up[cuts[2]:cuts[3]]
    status = up[cuts[3]:cuts[4]]  # int32 status, pad, int64 totals[2], int64 gate[2]
    leaf_box = torch.empty((sched.n_leaves, 6), dtype=torch.float64, device=dev)
    _native.call("hhsar_leaf_boxes", _native.ptr(el_dev), _native.ptr(bounds), sched.n_leaves,
                 _native.ptr(leaf_box), stream)
    geom = make_geom(region, kgrid, gamma, margin, pad, window_hi, tol, max_iter)
    # the plan also writes every grid's pool offset / work-list offset and
    # the two totals, so the host only reads them back
    _native.call("hhsar_grid_plan", _native.ptr(descs_dev), sched.n_grids, _native.ptr(leaf_box),
                 _native.ptr(boundary), n_b, _native.ptr(geom), _native.ptr(status),
                 _native.c_void_p_offset(status, 8), stream)
    if gate_dt is not None:
        a, b = sched.level_slices[0]
        _native.call("hhsar_leaf_range_gate",
                     ctypes.c_void_p(descs_dev.data_ptr() + a * _native.GRID_DTYPE.itemsize),
                     b - a, _native.ptr(geom), float(gate_dt), int(gate_bins),
                     _native.c_void_p_offset(status, 24),
                     stream)
    if cached is not None:
        return dict(el_dev=el_dev, sched=sched, descs_dev=descs_dev, geom=geom,
                    host_d=None, host_s=cached.status, done=None, back=None,
                    keep=(staged, up, leaf_box), cached=cached)
    back = torch.empty(int(cuts[1]) + 40, dtype=torch.uint8, pin_memory=True)
    back[:cuts[1]].copy_(descs_dev, non_blocking=True)
    back[cuts[1]:].copy_(status, non_blocking=True)
    done = torch.cuda.Event()
    done.record()
    return dict(el_dev=el_dev, sched=sched, descs_dev=descs_dev, geom=geom,
                host_d=back[:cuts[1]], host_s=back[cuts[1]:].numpy(),
                done=done, back=back, keep=(staged, up, leaf_box), cached=None)


_trace = None  # optional host-timeline hook (tools/host_overhead.py)


def finish_lattices(p, newton_grids=None, row_split=None) -> Lattices:
    """Wait for the plan, size the pools, launch Newton (current stream).

    ``row_split`` = (rank, world, grids) with ``newton_grids``: of each listed
    grid this process inverts only its share of the active rectangle's
    u-rows (rows [lo + n r / W, lo + n (r + 1) / W)); a column's planes are
    solved in order within the column only, so the union over ranks is the
    full inversion (dist.hhffbpa_sharded_device sums the shares)."""
    import torch
    cached = p.get("cached")
    if cached is None:
        p["done"].synchronize()
    if _trace:
        _trace("plan synced")
    sched, descs_dev, geom = p["sched"], p["descs_dev"], p["geom"]
    dev = descs_dev.device
    stream = _native.stream_handle()
    # the plan's pinned read-back IS the host descriptor table from here on
    # (edited in place, uploaded from, kept alive with the lattices); a
    # cached plan brings its own copy
    if cached is not None:
        if (newton_grids is not None) != (cached.masked_dev is not None):
            raise ValueError("a cached plan and newton_grids must come together")
        host = cached.descs
    else:
        host = p["host_d"].numpy().view(_native.GRID_DTYPE)
    status = p["host_s"]
    if int(status[:4].view(np.int32)[0]):
        raise NumericDomainError("compressed coordinates undefined this close to the array plane")
    # offsets, column offsets and both totals came from the plan (device scan)
    total, n_cols, g_b0, g_w = (int(v) for v in status[8:40].view(np.int64))
    n_cols_masked = None
    if newton_grids is not None and cached is not None:
        # the cached restricted work list over the recomputed plan (D2D)
        descs_dev.copy_(cached.masked_dev, non_blocking=True)
        n_cols = n_cols_masked = cached.n_cols
    elif newton_grids is not None:
        # Newton work list restricted to the selected grids: re-derive the
        # column offsets and send the descriptors back up
        if row_split is not None:
            r, world, gl = row_split
            for g in gl:
                lo, hi = int(host["act_lo"][g, 0]), int(host["act_hi"][g, 0])
                n = hi - lo + 1
                if n > 0:
                    host["act_lo"][g, 0] = lo + n * r // world
                    host["act_hi"][g, 0] = lo + n * (r + 1) // world - 1
        span = np.maximum(host["act_hi"].astype(np.int64) - host["act_lo"] + 1, 0)
        cols = np.where(np.asarray(newton_grids, dtype=bool), span[:, 0] * span[:, 1], 0)
        starts = np.cumsum(cols)
        n_cols = int(starts[-1])
        host["col_offset"][0] = 0
        host["col_offset"][1:] = starts[:-1]
        n_cols_masked = n_cols
        back, up = p["back"], p["keep"][1]
        nb = host.nbytes
        up[:nb].copy_(back[:nb], non_blocking=True)
    if _trace:
        _trace("worklist built")
    positions = torch.empty((total, 3), dtype=torch.float64, device=dev)
    # valid flags and per-grid counters zeroed by one fill
    vb = -(-total // 8) * 8
    zero = torch.zeros(vb + sched.n_grids * _native.GRID_STATS * 8, dtype=torch.uint8, device=dev)
    valid = zero[:total]
    stats = zero[vb:].view(torch.int64).view(sched.n_grids, _native.GRID_STATS)
    if _trace:
        _trace("pools allocated")
    _native.call("hhsar_grid_newton", _native.ptr(descs_dev), sched.n_grids, n_cols,
                 None, _native.ptr(geom), _native.ptr(positions), _native.ptr(valid),
                 _native.ptr(stats), stream)
    lat = Lattices(host, descs_dev, positions, valid, stats, geom)
    lat.keep = (p["back"], p["keep"][1])  # pinned staging must outlive the async copy
    lat.gate = (g_b0, g_w) if g_w > 0 else None
    lat.status = status
    lat.n_cols_masked = n_cols_masked
    return lat


@dataclass
class DeviceRun:
    """Device-side result of one HHFFBPA pass (everything still in HBM)."""
    volume: object            # complex64 [vox_end - vox_begin]
    lattices: Lattices
    sched: Schedule
    flags: object             # int64 [n_merge_stages + 1]
    oow: object               # int64 [1]


class Pipeline:
    """The fused HHFFBPA stages on device-resident envelopes, callable on
    grid subsets (the multi-GPU driver in dist.py runs each rank's subtrees).

    ``env`` holds envelope rows [env_row0, env_row0 + env.shape[0]) of the
    aperture; kernels index rows by global element number, so the pointer
    handed to them is shifted back by env_row0 rows (only owned rows are
    ever dereferenced).
    """

    def __init__(self, env, el_dev, el4, t0: float, dt: float, k_ref: float, kgrid, region,
                 final_dims, params: FfbpParams, levels: int, merge_factor: int = 2,
                 window_hi=None, newton_grids=None, env_row0: int = 0, sched=None, lat=None):
        import ctypes
        import torch
        self.dev = env.device
        self.env, self.el4 = env, el4
        self.t0, self.dt, self.k_ref = float(t0), float(dt), float(k_ref)
        self.region, self.final_dims, self.params = region, tuple(final_dims), params
        self.kid = _kernel_id(params.kernel)
        if window_hi is None:
            window_hi = t0 + (env.shape[1] - 1) * dt
        self.sched = sched or Schedule.shared(int(el_dev.shape[0]), levels, merge_factor)
        self.lat = lat or build_lattices(el_dev, self.sched, region, kgrid, params.gamma,
                                         params.margin, src_pad_of(params), window_hi,
                                         newton_grids=newton_grids)
        self.values = torch.empty(int(self.lat.npts.sum()), dtype=torch.complex64,
                                  device=self.dev)
        self.lat.values = self.values
        self.n_stages = len(self.sched.fanouts)
        counters = torch.zeros(self.n_stages + 2, dtype=torch.int64, device=self.dev)
        self.flags, self.oow = counters[:self.n_stages + 1], counters[self.n_stages + 1:]
        self.env_ptr = ctypes.c_void_p(env.data_ptr() - int(env_row0) * env.shape[1] * 8)

    def leaves(self, g0=None, g1=None):
        """Level-1 subimages of leaf grids [g0, g1) (default: all)."""
        a, b = self.sched.level_slices[0]
        g0 = a if g0 is None else g0
        g1 = b if g1 is None else g1
        if g1 <= g0:
            return
        lat = self.lat
        p_begin = int(lat.descs["offset"][g0])
        p_end = int(lat.descs["offset"][g1 - 1] + lat.npts[g1 - 1])
        _native.call("hhsar_leaf_bp", lat.desc_ptr(g0), g1 - g0, p_begin, p_end,
                     int(lat.npts[g0:g1].max()), _native.ptr(lat.positions),
                     _native.ptr(lat.valid), _native.ptr(self.el4), self.env_ptr,
                     self.env.shape[1], self.t0, self.dt, self.k_ref, _native.ptr(lat.geom), 1,
                     _native.ptr(self.values), _native.ptr(self.oow), _native.stream_handle())

    def merge(self, k: int, p0=None, p1=None):
        """Merge stage k: parents [p0, p1) of grid level k+1 (default: all)
        from their children at grid level k."""
        fan = self.sched.fanouts[k]
        c0, _ = self.sched.level_slices[k]
        a, b = self.sched.level_slices[k + 1]
        p0 = a if p0 is None else p0
        p1 = b if p1 is None else p1
        if p1 <= p0:
            return
        lat = self.lat
        ch0 = c0 + (p0 - a) * fan
        _native.call("hhsar_merge_level", lat.desc_ptr(p0), p1 - p0, lat.points_in(p0, p1),
                     _native.ptr(lat.positions), _native.ptr(lat.valid), lat.desc_ptr(ch0),
                     (p1 - p0) * fan, fan, _native.ptr(self.values), _native.ptr(lat.geom),
                     self.kid, 1, _native.ptr(self.values),
                     _native.c_void_p_offset(self.flags, k), _native.stream_handle())

    def land(self, vox_range=None):
        """Final Cartesian landing of voxels [vb, ve) (default: all)."""
        import torch
        origin, step = region_grid(self.region, self.final_dims)
        n_vox = int(np.prod(self.final_dims))
        vb, ve = vox_range if vox_range is not None else (0, n_vox)
        vol = torch.empty(ve - vb, dtype=torch.complex64, device=self.dev)
        c0, c1 = self.sched.level_slices[-1]
        d = np.asarray(self.final_dims, dtype=np.int64)
        span0 = int(self.lat.descs["offset"][c0])  # the children's pool span (pair staging)
        span = int(self.lat.descs["offset"][c1 - 1]) + int(self.lat.npts[c1 - 1]) - span0
        if not LANDING_PAIRS:
            span = 0
        _native.call("hhsar_merge_cartesian", _native.ptr(np.ascontiguousarray(origin)),
                     _native.ptr(np.ascontiguousarray(step)), _native.ptr(d), vb, ve,
                     self.lat.desc_ptr(c0), c1 - c0, _native.ptr(self.values), span0, span,
                     _native.ptr(self.lat.geom),
                     self.kid | (0 if LANDING_SERIES else LANDING_PER_VOXEL), _native.ptr(vol),
                     _native.c_void_p_offset(self.flags, self.n_stages), _native.stream_handle())
        return vol

    def run(self, vox_range=None) -> DeviceRun:
        self.leaves()
        for k in range(self.n_stages):
            self.merge(k)
        vol = self.land(vox_range)
        return DeviceRun(volume=vol, lattices=self.lat, sched=self.sched, flags=self.flags,
                         oow=self.oow)


def hhffbpa_device(env, el_dev, el4, t0: float, dt: float, k_ref: float, kgrid, region,
                   final_dims, params: FfbpParams, levels: int, merge_factor: int = 2,
                   vox_range=None, window_hi=None) -> DeviceRun:
    """The fused HHFFBPA pipeline on device-resident envelopes (levels >= 2)."""
    return Pipeline(env, el_dev, el4, t0, dt, k_ref, kgrid, region, final_dims, params, levels,
                    merge_factor, window_hi).run(vox_range)


def src_pad_of(params) -> int:
    return GRID_PAD + (3 if params.kernel == "cubic" else 2)  # ffbp.py:468


_GEO_STREAMS = {}


def geometry_stream(device):
    """High-priority side stream for the data-independent grid construction
    (its small plan kernels must not queue behind the range-compression
    CTAs: the host waits on them)."""
    import torch
    key = torch.device(device).index
    if key not in _GEO_STREAMS:
        _GEO_STREAMS[key] = torch.cuda.Stream(device=device, priority=-1)
    return _GEO_STREAMS[key]




def leaf_range_gate(lat, sched, dt: float, n_t: int) -> tuple[int, int]:
    """Delay-bin window [b0, b0 + w) that holds every delay the leaf stage can
    read.  A valid leaf point lies on a near-band plane w in [near_lo,
    near_hi] of its lattice (ffbp.py:294-301: only the two rings nearest the
    region's image carry values) where Newton converged to n = origin_n +
    step w within tol (ffbp.py:271-282).  n = c_nhi sqrt(r^2 - gap) - c_nlo r
    (spectrum.py:255-257) increases with the vertex distance sum r, so r lies
    in [r(n_lo), r(n_hi)] with r(n) = (c_nlo n + c_nhi sqrt(n^2 + A gap)) / A,
    A = c_nhi^2 - c_nlo^2; the four vertices lie within Dc of the element-box
    centre c, so |p - c| lies within r/4 -+ Dc and the leaf kernel's staging
    windows |p - c| -+ |e - c| within r/4 -+ (Dc + hd) (hd: half the element
    box's 3-D diagonal), plus 4 bins of pad each side.  Only the leaf stage
    reads envelopes (merges read lattices), so profiles outside the gate are
    never needed: config 4 keeps 128 of 4,096 bins (the containment boxes
    would keep 288).  Host restatement of hhsar_leaf_range_gate (the step
    uses the device one, which comes back with the plan; tests check the
    two agree: same float64 operations in the same order)."""
    d = lat.descs
    g = lat.geom
    a, b = sched.level_slices[0]
    ext = np.asarray(d["ext"][a:b], dtype=np.float64)
    box = np.asarray(d["box"][a:b], dtype=np.float64)
    origin_n = np.asarray(d["origin"][a:b, 2], dtype=np.float64)
    near_lo = np.asarray(d["near_lo"][a:b, 2], dtype=np.float64)
    near_hi = np.asarray(d["near_hi"][a:b, 2], dtype=np.float64)
    c_nhi, c_nlo, step, tol = (float(g[k][0]) for k in ("c_nhi", "c_nlo", "step", "tol"))
    A = c_nhi * c_nhi - c_nlo * c_nlo
    gap = 4.0 * (ext[:, 1] - ext[:, 0]) ** 2 + 4.0 * (ext[:, 3] - ext[:, 2]) ** 2
    Ag = A * gap
    n_lo = (origin_n + step * near_lo) - tol
    n_hi = (origin_n + step * near_hi) + tol
    r_lo = (c_nlo * n_lo + c_nhi * np.sqrt(n_lo * n_lo + Ag)) / A
    r_hi = (c_nlo * n_hi + c_nhi * np.sqrt(n_hi * n_hi + Ag)) / A
    c = 0.5 * (box[:, :3] + box[:, 3:])
    z2 = c[:, 2] * c[:, 2]
    dc = np.zeros(b - a)
    for q in range(4):
        vx, vy = ext[:, q >> 1], ext[:, 2 + (q & 1)]
        dc = np.maximum(dc, np.sqrt(((c[:, 0] - vx) ** 2 + (c[:, 1] - vy) ** 2) + z2))
    e = box[:, 3:] - box[:, :3]
    hd = 0.5 * np.sqrt((e[:, 0] ** 2 + e[:, 1] ** 2) + e[:, 2] ** 2)
    pad = dc + hd
    d_min = max(float((0.25 * r_lo - pad).min()), 0.0)
    d_max = float((0.25 * r_hi + pad).max())
    inv_bin = 2.0 / (C_LIGHT * dt)
    b0 = max(0, int(np.floor(d_min * inv_bin)) - 4)
    b1 = min(n_t, int(np.ceil(d_max * inv_bin)) + 5)
    w = min(n_t - b0, -(-(b1 - b0) // 32) * 32)
    return b0, w


def hhffbpa_from_cube(cube_dev, el_dev, el4, kgrid, region, final_dims, params: FfbpParams,
                      levels: int, merge_factor: int = 2, upsample: int = 8,
                      vox_range=None, gate: bool = True, upload=None, marks=None,
                      plan_cache=None) -> DeviceRun:
    """Whole HHFFBPA step from a device cube.  Plan + Newton run on a
    high-priority side stream; once the plan's descriptors are on the host
    the range compression is launched on the caller's stream for the delay
    bins the leaf stage can read only (hhsar_leaf_range_gate, computed with
    the plan; ``gate=False`` computes full profiles); the leaf stage waits
    for both.  The gate puts the plan's host round trip ahead of the
    compression but shrinks the profiles to the leaf stage's reach (config
    2/3/4: 256/352/288 of 1,024/2,048/4,096 bins; config 4 68.7 GB of
    profiles -> 4.8 GB).

    ``upload`` (a rangecomp.CubeUpload whose tensor is ``cube_dev``, or a
    zero-argument factory of one, then ``cube_dev`` may be None): the cube is
    still crossing PCIe; the compression runs chunk by chunk as rows land.
    A factory is called right after the plan's small host->device copy is
    queued, so that copy does not wait behind gigabytes of cube chunks in
    the copy engine (the plan's round trip gates the compression).
    ``marks`` (a dict) receives CUDA events recorded on the caller's stream
    around the range compression ("rc0", "rc1").  ``plan_cache`` (PlanCache
    of an earlier step of the same geometry): no host wait at all (see
    plan_lattices) -- the form StepGraph captures.
    """
    import torch
    from .rangecomp import profile_axis, range_compress_device, range_compress_window
    if _trace:
        _trace("enter")
    n_t, dt, k_ref, _ = profile_axis(kgrid, upsample)
    window_hi = 0.0 + (n_t - 1) * dt
    main = torch.cuda.current_stream()
    geo = geometry_stream(el_dev.device)
    geo.wait_stream(main)
    sched = Schedule.shared(int(el_dev.shape[0]), levels, merge_factor)
    if _trace:
        _trace("schedule")
    with torch.cuda.stream(geo):
        pending = plan_lattices(el_dev, sched, region, kgrid, params.gamma, params.margin,
                                src_pad_of(params), window_hi,
                                gate_dt=dt if gate else None, gate_bins=n_t, cached=plan_cache)
    if callable(upload):
        upload = upload()
        cube_dev = upload.tensor
    newton_first = False
    chunks = upload.chunks if upload is not None else None
    if marks is not None:
        marks["rc0"] = torch.cuda.Event(enable_timing=True)
        marks["rc1"] = torch.cuda.Event(enable_timing=True)
    if not gate:
        if upload is not None:
            upload.wait(main)
        if marks is not None:
            marks["rc0"].record(main)
        env, dt, k_ref = range_compress_device(cube_dev, kgrid, upsample)
        t0 = 0.0
    else:
        # after the plan's round trip Newton is queued first (high-priority
        # geometry stream), then the gated compression: on small problems
        # Newton's latency-bound fix-up is the critical path; at config 4
        # this order measured 15.94 vs 16.01 ms per graph step (compression
        # first), config 3 equal within 0.005 ms
        if plan_cache is None:
            pending["done"].synchronize()
        n_cols, b0, w = (int(v) for v in pending["host_s"][16:40].view(np.int64))
        newton_first = True
        with torch.cuda.stream(geo):
            lat = finish_lattices(pending)
        if _trace:
            _trace("gate")
        if marks is not None and not chunks:
            marks["rc0"].record(main)
        env, t0, dt, k_ref = range_compress_window(cube_dev, kgrid, upsample, b0, w,
                                                   chunks=chunks,
                                                   row0=upload.row0 if upload else 0)
    if marks is not None:
        if chunks and gate:
            marks["rc0"] = None  # compression interleaved with the upload
        marks["rc1"].record(main)
    if not newton_first:
        with torch.cuda.stream(geo):
            lat = finish_lattices(pending)
    main.wait_stream(geo)
    # blocks allocated on the side stream are used on the main one from here
    for t in (lat.positions, lat.valid, lat.stats, lat.keep[1]):
        t.record_stream(main)
    pipe = Pipeline(env, el_dev, el4, t0, dt, k_ref, kgrid, region, final_dims, params, levels,
                    merge_factor, window_hi, sched=sched, lat=lat)
    if _trace:
        _trace("pipeline ready")
    return pipe.run(vox_range)


@dataclass
class PlanCache:
    """Host copy of a plan (descriptor table + status words) for one
    geometry: the plan is a pure function of the element positions, the
    region, the band and the parameters, so a later step of the same
    geometry can size its pools and launches from it without waiting for
    its own (recomputed) plan."""
    descs: np.ndarray   # GRID_DTYPE [G] (pool / work-list offsets filled in)
    status: np.ndarray  # uint8 [40]: status word, totals, gate
    # a plan whose Newton work list was restricted to some grids
    # (newton_grids, the multi-GPU ranks): the restricted descriptor table on
    # the device (copied over each recomputed plan) and its column count
    masked_dev: object = None
    n_cols: int = -1

    @staticmethod
    def of(run: DeviceRun) -> "PlanCache":
        return PlanCache.of_lattices(run.lattices)

    @staticmethod
    def of_lattices(lat) -> "PlanCache":
        import torch
        descs = lat.descs.copy()
        masked = None
        if getattr(lat, "n_cols_masked", None) is not None:
            masked = torch.as_tensor(descs.view(np.uint8)).to(lat.descs_dev.device)
        return PlanCache(descs=descs, status=np.asarray(lat.status).copy(), masked_dev=masked,
                         n_cols=-1 if masked is None else int(lat.n_cols_masked))


class StepGraph:
    """One HHFFBPA step (hhffbpa_from_cube) captured in a CUDA graph.

    Small configs are launch- and latency-bound: config 2's step is ~60
    launches and one plan round trip.  An eager step first records the plan
    (PlanCache); a second eager step with the cached plan checks the result
    is bit-identical to the first; then the same host sequence -- plan,
    Newton (with its side-stream fix-up), gated compression, leaves, merges,
    landing, every kernel recomputed -- is captured once and replayed.
    Fixed per graph: the geometry (element positions, region, band,
    parameters) and the cube buffer's address; the cube's contents may
    change between replays.  ``replay()`` returns the DeviceRun whose
    tensors the graph rewrites each time."""

    def __init__(self, cube_dev, el_dev, el4, kgrid, region, final_dims, params, levels,
                 merge_factor=2, upsample=8, vox_range=None):
        import torch
        args = (cube_dev, el_dev, el4, kgrid, region, final_dims, params, levels, merge_factor,
                upsample, vox_range)
        first = hhffbpa_from_cube(*args)
        torch.cuda.synchronize()
        if int(first.oow.cpu()[0]):
            raise NumericDomainError("leaf delays outside the range gate: use "
                                     "hhffbpa_reconstruct, which redoes the step ungated")
        self.cache = PlanCache.of(first)
        check = hhffbpa_from_cube(*args, plan_cache=self.cache)
        torch.cuda.synchronize()
        if not (torch.equal(check.volume, first.volume) and
                torch.equal(check.lattices.stats, first.lattices.stats)):
            raise RuntimeError("cached-plan step differs from the planned step")
        del first, check
        side = torch.cuda.Stream(device=el_dev.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # capture-safe warm-up on a side stream
            hhffbpa_from_cube(*args, plan_cache=self.cache)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run = hhffbpa_from_cube(*args, plan_cache=self.cache)
        self._args = args  # the captured buffers stay alive with the graph

    def replay(self) -> DeviceRun:
        self.graph.replay()
        return self.run


def _core_sizes(descs) -> np.ndarray:
    return np.prod(descs["core_hi"].astype(np.int64) - descs["core_lo"] + 1, axis=1)


def _raise_core(masked: float):
    raise NumericDomainError(
        f"{100 * masked:.0f}% of core lattice points have no valid inverse "
        "position; the region is incompatible with this subarray")


def check_grids(run: DeviceRun, stats: np.ndarray):
    """The reference's SubimageGrid health checks (ffbp.py:127-133) in the
    reference's order: each leaf as built, then after its delay mask
    (ffbp.py:331-335), then every parent level by level (vectorised: the
    first failing grid in that order raises)."""
    sched, descs = run.sched, run.lattices.descs
    size = _core_sizes(descs)
    g0, g1 = sched.level_slices[0]
    # leaves: [built, masked] interleaved per grid, then the parents in order
    leaf = np.stack([1.0 - stats[g0:g1, 1] / size[g0:g1],
                     1.0 - stats[g0:g1, 3] / size[g0:g1]], axis=1).reshape(-1)
    parents = 1.0 - stats[g1:, 1] / size[g1:]
    masked = np.concatenate([leaf, parents])
    bad = np.flatnonzero(masked >= 0.5)
    if bad.size:
        _raise_core(float(masked[bad[0]]))


def provenance_of(run: DeviceRun, stats, flags, final_dims, params, levels, upsample,
                  merge_factor=2) -> dict:
    sched = run.sched
    level_points = []
    for k, (a, b) in enumerate(sched.level_slices):
        col = 2 if k == 0 else 0
        level_points.append([int(v) for v in stats[a:b, col]])
    n_final = int(np.prod(final_dims))
    level_points.append([n_final])
    merge_flags = [int(f) for f in flags[:-1]]
    final_flags = int(flags[-1])
    merged_total = sum(sum(p) for p in level_points[1:])
    flagged_total = sum(merge_flags) + final_flags
    prov = {"algorithm": "hhffbpa", "levels": levels, "gamma": params.gamma,
            "kernel": params.kernel, "margin": params.margin, "upsample": upsample,
            "dims": list(final_dims), "level_points": level_points, "merge_flags": merge_flags,
            "final_flags": final_flags,
            "flagged_fraction": (flagged_total / merged_total) if merged_total else 0.0}
    if merge_factor != 2:
        prov["merge_factor"] = merge_factor
    return prov


def _prepare(cube, region, final_dims, params, upsample):
    """The reference's argument checks and defaults (ffbp.py:445-458)."""
    if params is None:
        params = FfbpParams()
    validate_geometry(cube.aperture, region)
    kgrid = cube.freqs
    if final_dims is None:
        final_dims = default_grid_dims(region, kgrid)
    final_dims = tuple(int(d) for d in final_dims)
    levels = params.levels if params.levels is not None else default_levels(cube.aperture)
    return params, kgrid, final_dims, levels


def _device_elements(cube, region, kgrid, upsample, levels):
    """Element positions on the device + the checks that need them."""
    import torch
    _native.library()
    el_dev = torch.tensor(np.ascontiguousarray(cube.aperture.elements, dtype=np.float64),
                          device="cuda")
    n_t, dt, k_ref, _ = profile_axis(kgrid, upsample)
    check_delay_window(RangeProfileSet(envelopes=torch.empty((0, n_t)), t0=0.0, dt=dt,
                                       upsample=upsample, k_ref=k_ref, aperture=cube.aperture,
                                       freqs=kgrid, elements_dev=el_dev), region)
    if region.z_min <= 0.0:
        raise ConfigError("region must sit strictly in front of the array")
    leaf_bounds(cube.aperture.n_elements, levels)  # ConfigError when too deep (model.py:371-376)
    return el_dev


def _volume_of(run, final_dims, origin, step, params, levels, upsample, merge_factor):
    """Device run -> host ImageVolume with the reference's checks and
    provenance (one device->host round trip)."""
    import torch
    extra = torch.cat([run.flags, run.lattices.stats.reshape(-1)])
    volume, tail = _finish(run.volume, run.oow, final_dims, origin, step, {}, extra)
    n_flags = run.flags.numel()
    flags = tail[:n_flags]
    stats = tail[n_flags:].reshape(-1, _native.GRID_STATS)
    check_grids(run, stats)
    prov = provenance_of(run, stats, flags, final_dims, params, levels, upsample, merge_factor)
    object.__setattr__(volume, "provenance", prov)
    return volume


def hhffbpa_reconstruct(cube, region, final_dims=None, params: FfbpParams | None = None,
                        upsample: int = 8, *, merge_factor: int = 2) -> ImageVolume:
    """Cartesian volume by factorised backprojection (ffbp.py:415-513)."""
    params, kgrid, final_dims, levels = _prepare(cube, region, final_dims, params, upsample)
    origin, step = region_grid(region, final_dims)
    if levels == 1:  # ffbp.py:460-464: plain BPA onto the final grid
        profiles = range_compress(cube, upsample)
        check_delay_window(profiles, region)
        el4 = el_f32x4(profiles.elements_dev)
        vol, oow = bpa_volume_device(profiles.envelopes, el4, region, final_dims, profiles.t0,
                                     profiles.dt, profiles.k_ref)
        n = int(np.prod(final_dims))
        prov = {"algorithm": "hhffbpa", "levels": 1, "gamma": params.gamma,
                "kernel": params.kernel, "margin": params.margin, "upsample": upsample,
                "dims": list(final_dims), "level_points": [[n]], "merge_flags": [],
                "final_flags": 0, "flagged_fraction": 0.0}
        return _finish(vol, oow, final_dims, origin, step, prov)[0]
    el_dev = _device_elements(cube, region, kgrid, upsample, levels)
    # the cube streams in by chunks (pinned input: DMA straight from the
    # caller's buffer) while the plan, Newton and the range compression of
    # the rows already landed run
    uploads = []

    def start_upload():
        uploads.append(CubeUpload(cube.values))
        return uploads[0]

    run = hhffbpa_from_cube(None, el_dev, el_f32x4(el_dev), kgrid, region, final_dims,
                            params, levels, merge_factor, upsample, upload=start_upload)
    cube_dev = uploads[0].tensor
    if int(run.oow.cpu()[0]):
        # a leaf delay outside the range gate (the gate is a geometric bound;
        # this never fired on the BASELINE configs): redo on full profiles so
        # the out-of-window verdict is the reference's
        run = hhffbpa_from_cube(cube_dev, el_dev, el_f32x4(el_dev), kgrid, region, final_dims,
                                params, levels, merge_factor, upsample, gate=False)
    return _volume_of(run, final_dims, origin, step, params, levels, upsample, merge_factor)


_D2H_STREAMS = {}


def _d2h_stream(device):
    import torch
    key = torch.device(device).index
    if key not in _D2H_STREAMS:
        _D2H_STREAMS[key] = torch.cuda.Stream(device=device)
    return _D2H_STREAMS[key]


class _InFlight:
    """One volume of a stream: its upload, device run, and the asynchronous
    copy-back (volume + counters into pinned memory on a D2H stream)."""

    def __init__(self, upload, run, d2h):
        import torch
        self.upload, self.run = upload, run
        d2h.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(d2h):
            finite = torch.isfinite(torch.view_as_real(run.volume)).all().reshape(1)
            self.scalars_dev = torch.cat([run.oow.reshape(-1)[:1], finite.to(torch.int64),
                                          run.flags, run.lattices.stats.reshape(-1)])
            self.volume = torch.empty(run.volume.shape, dtype=run.volume.dtype, pin_memory=True)
            self.scalars = torch.empty(self.scalars_dev.shape, dtype=torch.int64,
                                       pin_memory=True)
            self.volume.copy_(run.volume, non_blocking=True)
            self.scalars.copy_(self.scalars_dev, non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record(d2h)
        run.volume.record_stream(d2h)


def hhffbpa_reconstruct_stream(cubes, region, final_dims=None, params: FfbpParams | None = None,
                               upsample: int = 8, *, merge_factor: int = 2):
    """hhffbpa_reconstruct over a sequence of cubes of ONE geometry (same
    aperture, band and region: e.g. repeated handheld scans), as a
    generator of ImageVolume, one per cube, in order.

    Every volume is computed exactly as hhffbpa_reconstruct computes it
    (plan, Newton, gated compression, leaves, merges, landing, the
    reference's checks and provenance); what changes is the overlap of the
    host transfers: the upload of cube i+1 (H2D, copy engine) runs while
    volume i is finished and copied back (D2H, the other direction of the
    link), and from the second volume on the plan comes from a PlanCache of
    the first (the device still recomputes it), so the host never waits
    inside a volume.  Per volume the link then carries the cube in and the
    volume out concurrently: the period is ~max(upload, compute tail +
    copy-back) instead of their sum."""
    import torch
    it = iter(cubes)
    try:
        first = next(it)
    except StopIteration:
        return
    params, kgrid, final_dims, levels = _prepare(first, region, final_dims, params, upsample)
    if levels == 1:
        yield hhffbpa_reconstruct(first, region, final_dims, params, upsample,
                                  merge_factor=merge_factor)
        for cube in it:
            yield hhffbpa_reconstruct(cube, region, final_dims, params, upsample,
                                      merge_factor=merge_factor)
        return
    origin, step = region_grid(region, final_dims)
    el_dev = _device_elements(first, region, kgrid, upsample, levels)
    el4 = el_f32x4(el_dev)
    elements = np.asarray(first.aperture.elements)
    main = torch.cuda.current_stream()
    d2h = _d2h_stream(el_dev.device)
    cache = None

    def same_geometry(cube):
        el = np.asarray(cube.aperture.elements)
        if el is not elements and not np.array_equal(el, elements):
            raise ConfigError("hhffbpa_reconstruct_stream: every cube must share the "
                              "first cube's aperture")
        if cube.freqs != first.freqs:
            raise ConfigError("hhffbpa_reconstruct_stream: every cube must share the "
                              "first cube's frequency grid")

    def upload(cube):
        from .rangecomp import copy_stream
        with torch.cuda.stream(copy_stream(el_dev.device)):  # allocated on the H2D queue
            up = CubeUpload(cube.values)
        up.tensor.record_stream(main)
        return up

    def launch(cube, up):
        """Queue one volume; the first plans on the host (and starts its upload
        right after the plan's copy), the later ones reuse its PlanCache."""
        nonlocal cache
        if cache is None:
            ups = []
            run = hhffbpa_from_cube(None, el_dev, el4, kgrid, region, final_dims, params,
                                    levels, merge_factor, upsample,
                                    upload=lambda: ups.append(upload(cube)) or ups[0])
            cache = PlanCache.of(run)
            up = ups[0]
        else:
            run = hhffbpa_from_cube(up.tensor, el_dev, el4, kgrid, region, final_dims, params,
                                    levels, merge_factor, upsample, upload=up, plan_cache=cache)
        return _InFlight(up, run, d2h)

    def complete(fl: _InFlight, cube):
        fl.done.synchronize()
        sc = fl.scalars.numpy()
        run = fl.run
        if int(sc[0]):  # out-of-window leaf delay: redo ungated, as hhffbpa_reconstruct
            run = hhffbpa_from_cube(fl.upload.tensor, el_dev, el4, kgrid, region, final_dims,
                                    params, levels, merge_factor, upsample, gate=False)
            return _volume_of(run, final_dims, origin, step, params, levels, upsample,
                              merge_factor)
        if not int(sc[1]):
            raise ConfigError("volume values must be finite")
        n_flags = run.flags.numel()
        flags = sc[2:2 + n_flags]
        stats = sc[2 + n_flags:].reshape(-1, _native.GRID_STATS)
        check_grids(run, stats)
        prov = provenance_of(run, stats, flags, final_dims, params, levels, upsample,
                             merge_factor)
        return ImageVolume._trusted(fl.volume.numpy().reshape(final_dims), origin, step, prov)

    cube, up = first, None
    pending = None
    while cube is not None:
        nxt = next(it, None)
        if nxt is not None:
            same_geometry(nxt)
        flight = launch(cube, up)
        # the next cube's upload is queued right behind this one's
        up_next = upload(nxt) if nxt is not None else None
        if pending is not None:
            yield complete(*pending)
        pending = (flight, cube)
        cube, up = nxt, up_next
    if pending is not None:
        yield complete(*pending)


# ---------------------------------------------------------------------------
# single-subimage API (build_subimage_grid, level1_reconstruct, merge_pair)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SubimageGrid:
    """Lattice of one subarray (ffbp.py:74-158), host arrays.

    Positions of masked points are not computed on the GPU (their values are
    zero and nothing reads them); they hold the region centre.
    """

    subarray: object
    extents: SubarrayExtents
    origin: np.ndarray
    step: np.ndarray
    positions: np.ndarray
    valid: np.ndarray
    core: tuple | None = None

    def __post_init__(self):
        origin = np.asarray(self.origin, dtype=float).reshape(3)
        step = np.asarray(self.step, dtype=float).reshape(3)
        if np.any(step > 1.0 + 1e-12) or np.any(step <= 0.0):
            raise ConfigError("lattice step must lie in (0, 1]")
        pos = np.asarray(self.positions, dtype=float)
        valid = np.asarray(self.valid, dtype=bool)
        if pos.ndim != 4 or pos.shape[-1] != 3 or valid.shape != pos.shape[:3]:
            raise ConfigError("positions must be (nu, nv, nn, 3) with a matching validity mask")
        core = self.core
        if core is None:
            core = tuple((0, n - 1) for n in valid.shape)
        else:
            core = tuple((int(a), int(b)) for a, b in core)
            for (a, b), n in zip(core, valid.shape):
                if not 0 <= a <= b < n:
                    raise ConfigError("core bounds must lie inside the lattice")
        masked = 1.0 - valid[tuple(slice(a, b + 1) for a, b in core)].mean()
        if masked >= 0.5:
            _raise_core(masked)
        for k, v in (("core", core), ("origin", origin), ("step", step), ("positions", pos),
                     ("valid", valid)):
            object.__setattr__(self, k, v)

    @property
    def dims(self):
        return self.positions.shape[:3]

    @property
    def n_points(self) -> int:
        return int(np.prod(self.dims))

    @property
    def n_valid(self) -> int:
        return int(self.valid.sum())

    @property
    def masked_fraction(self) -> float:
        return 1.0 - self.valid.mean()

    def lattice_coords(self, uvn):
        return (np.asarray(uvn, dtype=float) - self.origin) / self.step


@dataclass(frozen=True)
class Subimage:
    """Complex samples of one subarray's partial image (ffbp.py:161-176)."""

    grid: SubimageGrid
    values: np.ndarray
    downconverted: bool = False

    def __post_init__(self):
        v = np.asarray(self.values)
        if not np.iscomplexobj(v):
            v = v.astype(np.complex128)
        if v.shape != self.grid.dims:
            raise ConfigError(f"value shape {v.shape} does not match grid dims {self.grid.dims}")
        if not np.all(v[~self.grid.valid] == 0.0):
            raise ConfigError("masked lattice points must carry zero values")
        object.__setattr__(self, "values", v)


def _one_desc(ext, origin, dims, start, stop, offset=0):
    d = np.zeros(1, dtype=_native.GRID_DTYPE)
    d["ext"] = ext
    d["origin"] = origin
    d["dims"] = dims
    d["start"], d["stop"], d["offset"] = start, stop, offset
    return d


def build_subimage_grid(aperture, subarray, region, kgrid, gamma: float = 1.4,
                        margin: float = 0.25, tol: float = 1e-9, max_iter: int = 50,
                        pad: int = GRID_PAD) -> SubimageGrid:
    """One subarray's lattice (ffbp.py:179-307) through the batched kernels."""
    import torch
    if isinstance(aperture, SubarrayExtents) or (hasattr(aperture, "x_min") and
                                                  not hasattr(aperture, "elements")):
        ext = aperture if isinstance(aperture, SubarrayExtents) else SubarrayExtents(
            aperture.x_min, aperture.x_max, aperture.y_min, aperture.y_max)
        el = np.array([[ext.x_min, ext.y_min, 0.0], [ext.x_max, ext.y_max, 0.0]])
    else:
        el = np.asarray(aperture.elements, dtype=float)
        if subarray is not None:
            el = el[subarray.start:subarray.stop]
        ext = SubarrayExtents(float(el[:, 0].min()), float(el[:, 0].max()),
                              float(el[:, 1].min()), float(el[:, 1].max()))
    if not gamma >= 1.0:
        raise ConfigError("oversampling factor must be at least 1")
    if region.z_min <= 0.0:
        raise ConfigError("region must sit strictly in front of the array")
    if int(pad) != pad or pad < 1:
        raise ConfigError("pad must be an integer >= 1")
    if not 1 <= int(max_iter) <= MAX_NEWTON_ITER:
        # the batched grid build carries iteration counts in 7 bits
        raise ConfigError(f"max_iter must lie in [1, {MAX_NEWTON_ITER}]")
    _native.library()
    el_dev = torch.as_tensor(np.ascontiguousarray(el), device="cuda")
    sched = Schedule(el.shape[0], 1)
    sched.grids["is_leaf"] = 0
    lat = build_lattices(el_dev, sched, region, kgrid, gamma, margin, int(pad), np.inf, tol,
                         max_iter)
    d = lat.descs[0]
    dims = tuple(int(v) for v in d["dims"])
    center = np.array([(region.x_min + region.x_max) / 2, (region.y_min + region.y_max) / 2,
                       (region.z_min + region.z_max) / 2])
    valid = lat.valid.cpu().numpy().astype(bool).reshape(dims)
    pos = lat.positions.cpu().numpy().reshape(dims + (3,))
    pos = np.where(valid[..., None], pos, center)
    core = tuple((int(d["core_lo"][a]), int(d["core_hi"][a])) for a in range(3))
    return SubimageGrid(subarray=subarray, extents=ext, origin=d["origin"].copy(),
                        step=np.full(3, 1.0 / gamma), positions=pos, valid=valid, core=core)


def _geom_for(kgrid, gamma=1.4):
    return _native.host_struct(_native.GEOM_DTYPE, dict(
        k_min=kgrid.k_min, k_max=kgrid.k_max, c_uv=kgrid.k_max / np.pi,
        c_nhi=kgrid.k_max / (2.0 * TWO_PI), c_nlo=kgrid.k_min / (2.0 * TWO_PI),
        step=1.0 / gamma))


def level1_reconstruct(profiles: RangeProfileSet, subarray, grid: SubimageGrid) -> Subimage:
    """Backproject one subarray onto its grid (ffbp.py:310-340); the delay
    mask uses the 8 corners of the subarray's 3-D element bbox."""
    import torch
    flat = grid.positions.reshape(-1, 3)
    mask = grid.valid.ravel().copy()
    if mask.any():
        els = np.asarray(profiles.aperture.elements)[subarray.start:subarray.stop]
        lo, hi = els.min(axis=0), els.max(axis=0)
        corners = np.stack([np.where(np.array(bits), hi, lo) for bits in np.ndindex(2, 2, 2)])
        pts = flat[mask]
        dmax = np.linalg.norm(pts[:, None, :] - corners[None], axis=2).max(axis=1)
        mask[mask] = 2.0 * dmax / C_LIGHT <= profiles.window[1]
    if not np.array_equal(mask, grid.valid.ravel()):
        grid = SubimageGrid(subarray=grid.subarray, extents=grid.extents, origin=grid.origin,
                            step=grid.step, positions=grid.positions,
                            valid=mask.reshape(grid.dims), core=grid.core)
    dev = profiles.envelopes.device
    desc = _one_desc(grid.extents.as_tuple(), grid.origin, grid.dims, subarray.start,
                     subarray.stop)
    desc_dev = _native.device_struct(desc, dev)
    pos = torch.as_tensor(np.ascontiguousarray(flat), device=dev)
    val = torch.as_tensor(mask.astype(np.uint8), device=dev)
    out = torch.empty(flat.shape[0], dtype=torch.complex64, device=dev)
    oow = torch.zeros(1, dtype=torch.int64, device=dev)
    geom = _geom_for(profiles.freqs, 1.0 / float(grid.step[0]))
    _native.call("hhsar_leaf_bp", _native.ptr(desc_dev), 1, 0, flat.shape[0], flat.shape[0],
                 _native.ptr(pos), _native.ptr(val),
                 _native.ptr(el_f32x4(profiles.elements_dev)), _native.ptr(profiles.envelopes),
                 profiles.envelopes.shape[1], float(profiles.t0), float(profiles.dt),
                 float(profiles.k_ref), _native.ptr(geom), 0, _native.ptr(out), _native.ptr(oow),
                 _native.stream_handle())
    bad = int(oow.cpu()[0])
    if bad:
        raise NumericDomainError(
            f"{bad} point-element delays fell outside the profile window; "
            "enlarge the upsampled profile or shrink the geometry")
    return Subimage(grid=grid, values=out.cpu().numpy().reshape(grid.dims), downconverted=False)


def merge_pair(a: Subimage, b: Subimage, parent_grid: SubimageGrid, kgrid,
               kernel: str = "linear"):
    """Merge two sibling subimages onto their parent's grid (ffbp.py:377-412)."""
    import torch
    kid = _kernel_id(kernel)
    parent = parent_grid.subarray
    if parent is not None:
        for child in (a, b):
            csa = child.grid.subarray
            if csa is not None and not (parent.start <= csa.start and csa.stop <= parent.stop):
                raise ConfigError("children must cover element slices inside the parent subarray")
    _native.library()
    grids = (a.grid, b.grid, parent_grid)
    sizes = [g.n_points for g in grids]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    descs = np.concatenate([_one_desc(g.extents.as_tuple(), g.origin, g.dims, 0, 0, o)
                            for g, o in zip(grids, offs[:-1])])
    dev = torch.device("cuda")
    descs_dev = _native.device_struct(descs, dev)
    pos = torch.as_tensor(np.concatenate([g.positions.reshape(-1, 3) for g in grids]), device=dev)
    val = torch.as_tensor(np.concatenate([g.valid.ravel() for g in grids]).astype(np.uint8),
                          device=dev)
    vals = np.zeros(offs[-1], dtype=np.complex64)
    vals[:offs[2]] = np.concatenate([np.asarray(s.values).ravel() for s in (a, b)])
    values = torch.as_tensor(vals, device=dev)
    geom = _geom_for(kgrid, 1.0 / float(parent_grid.step[0]))
    stream = _native.stream_handle()
    base = descs_dev.data_ptr()
    import ctypes
    for k, s in enumerate((a, b)):
        if not s.downconverted:
            _native.call("hhsar_downconvert", ctypes.c_void_p(base + k * descs.itemsize), 1,
                         sizes[k], _native.ptr(pos), _native.ptr(val), _native.ptr(geom),
                         _native.ptr(values), stream)
    flagged = torch.zeros(1, dtype=torch.int64, device=dev)
    _native.call("hhsar_merge_level", ctypes.c_void_p(base + 2 * descs.itemsize), 1, sizes[2],
                 _native.ptr(pos), _native.ptr(val), ctypes.c_void_p(base), 2, 2,
                 _native.ptr(values), _native.ptr(geom), kid, 0, _native.ptr(values),
                 _native.ptr(flagged), stream)
    out = values[offs[2]:].cpu().numpy().reshape(parent_grid.dims)
    return Subimage(grid=parent_grid, values=out, downconverted=False), int(flagged.cpu()[0])
