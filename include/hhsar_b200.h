/*
 * hhsar_b200.h -- C ABI of the B200-native HHFFBPA / BPA hot path.
 *
 * Every entry point takes caller-owned DEVICE buffers (plain pointers and
 * sizes; complex values are interleaved float32 re/im = complex64), a CUDA
 * stream handle (cudaStream_t passed as void*), and returns an int status:
 * 0 = OK, 1 = bad argument, 2 = CUDA error (hhsar_last_error() has text).
 * Calls are asynchronous on the given stream; nothing synchronises except
 * where noted.  No C++ exceptions cross the ABI.  Process-wide state: the
 * last-error string (thread-local) and per-device caches -- SM count,
 * kernel occupancy, one high-priority side stream per device (used by
 * hhsar_grid_newton's fix-up) -- each created once under a mutex and keyed
 * by the caller's current device, so calls are thread-safe per stream and
 * one process may drive several GPUs.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/hhsar):
 *   hhsar_bp_gather        <- _kernels.backproject_gather   (_kernels.py:98-110)
 *   hhsar_lattice_interp   <- _kernels.lattice_interpolate  (_kernels.py:354-378)
 *   hhsar_invert_newton    <- _kernels._invert_newton_jit    (_kernels.py:255-351,
 *                             called via spectrum.invert_lattice, spectrum.py:327-407)
 *   hhsar_bpa_cartesian    <- bpa.bpa_reconstruct's meshgrid + backproject
 *                             (bpa.py:163-176)
 *   hhsar_range_compress   <- rangecomp.range_compress (rangecomp.py:61-101):
 *                             zero pad + IDFT + demodulation in one pass
 *   hhsar_range_pad / hhsar_range_demod
 *                          <- the same around a library IDFT (rangecomp.py:86-96),
 *                             for n_t outside the fused kernel's sizes
 *   hhsar_volume_dot / hhsar_volume_residual <- metrics.psnr (metrics.py:126-150)
 *   hhsar_mip              <- metrics.max_intensity_projection (metrics.py:170-190)
 *   hhsar_leaf_boxes / hhsar_grid_plan / hhsar_grid_newton
 *                          <- ffbp.build_subimage_grid for every subarray of
 *                             every level at once (ffbp.py:179-307) plus the
 *                             leaf delay mask of ffbp.level1_reconstruct
 *                             (ffbp.py:320-335)
 *   hhsar_leaf_bp          <- ffbp.level1_reconstruct's backproject
 *                             (ffbp.py:336-340) fused with _downconvert_samples
 *                             (ffbp.py:343-348)
 *   hhsar_merge_level      <- ffbp.merge_pair / _merge_onto_points for every
 *                             parent of a level (ffbp.py:351-412)
 *   hhsar_merge_cartesian  <- the final Cartesian landing (ffbp.py:493-495)
 *   hhsar_downconvert      <- ffbp._downconvert_samples (ffbp.py:343-348)
 *   hhsar_simulate / hhsar_simulate_uniform
 *                          <- simulator.simulate_measurement (simulator.py:41-69)
 */
#ifndef HHSAR_B200_H
#define HHSAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HHSAR_OK 0
#define HHSAR_EINVAL 1
#define HHSAR_ECUDA 2

/* largest Newton iteration cap the batched grid build accepts (7-bit
 * iteration counts; the reference default is 50, ffbp.py:182) */
#define HHSAR_MAX_NEWTON_ITER 126

/* Geometry constants shared by the grid, leaf and merge kernels.  Host code
 * computes every derived constant in float64 exactly as the reference does
 * (e.g. c_uv = k_max / pi, c_nhi = k_max / (2 * 2pi)) so the lattice bounds
 * built on the device are bit-identical to the reference's. */
typedef struct hhsar_geom {
    double region[6];   /* x_min, x_max, y_min, y_max, z_min, z_max          */
    double center[3];   /* region.center                                       */
    double k_min, k_max;
    double c_uv;        /* k_max / pi                 (spectrum.py:268, 271)   */
    double c_nhi;       /* k_max / (2 * TWO_PI)       (spectrum.py:256)        */
    double c_nlo;       /* k_min / (2 * TWO_PI)                                */
    double step;        /* 1 / gamma                  (ffbp.py:241)            */
    double margin;      /*                            (ffbp.py:269)            */
    double max_step;    /* 0.5 * region.diagonal      (ffbp.py:260)            */
    double tol;         /* Newton max-norm tolerance  (ffbp.py:182)            */
    double z_floor;     /* 1e-4                       (spectrum.py:331)        */
    double window_hi;   /* profile window upper bound [s] (rangecomp.py:56-58) */
    int32_t pad;        /* lattice pad steps (src_pad, ffbp.py:468)            */
    int32_t max_iter;   /* Newton iteration cap (50)                           */
} hhsar_geom;

/* One subimage lattice.  Filled by hhsar_grid_plan (bounds, dims, masks'
 * index ranges, and offset/col_offset when it is given `totals`) except
 * start/stop/leaf range (host). */
typedef struct hhsar_grid_desc {
    double ext[4];       /* lateral element bbox x_min,x_max,y_min,y_max       */
    double box[6];       /* 3-D element bbox: lo xyz, hi xyz                   */
    double lo[3], hi[3]; /* (u,v,n) image of the region's 5^3 boundary lattice */
    double origin[3];    /* (u,v,n) of lattice index 0                         */
    double slack_lo[3];  /* containment bounds region_min - slack              */
    double slack_hi[3];  /*                    region_max + slack              */
    int32_t dims[3];     /* nu, nv, nn                                         */
    int32_t near_lo[3];  /* index range of the two-ring band (ffbp.py:294-301) */
    int32_t near_hi[3];
    int32_t core_lo[3];  /* index range of the region image (ffbp.py:302-304)  */
    int32_t core_hi[3];
    int32_t is_leaf;     /* apply the level-1 delay-window mask                */
    int32_t act_lo[2];   /* (u, v) index rectangle of the columns Newton must  */
    int32_t act_hi[2];   /* run: near band AND reachable |tu|, |tv| (empty if  */
                         /* lo > hi); every other column is masked outright    */
    int64_t start, stop; /* element slice [start, stop)                        */
    int64_t leaf_lo, leaf_hi; /* leaf index range [leaf_lo, leaf_hi)           */
    int64_t offset;      /* first lattice point in the global pools            */
    int64_t col_offset;  /* first active column in the Newton work list        */
} hhsar_grid_desc;

/* Per-grid counters written by hhsar_grid_newton (int64 each):
 * [0] valid points, [1] valid core points   (SubimageGrid built, ffbp.py:305)
 * [2] valid after the leaf delay mask, [3] core valid after it (ffbp.py:331-335)
 * [4] Newton iterations executed, [5] Newton solves executed (points whose
 * inversion had to run; pruned columns run none)                             */
#define HHSAR_GRID_STATS 6

const char *hhsar_last_error(void);
int hhsar_version(void);
int hhsar_device_sm_count(void);
/* Host-only: writes sizeof/offsetof facts of the structs above into out[0..n)
 * (sizeof geom, sizeof grid_desc, offsets of geom.window_hi, geom.pad,
 * desc.dims, desc.is_leaf, desc.start, desc.offset, desc.col_offset) and
 * returns how many facts exist.  Lets a binding verify its struct mirrors. */
int hhsar_abi_layout(int64_t *out, int n);

/* ---- operator level ---------------------------------------------------- */

/* backproject_gather: out[n] (complex64), oow[n] = count of element delays
 * outside [0, n_t-1] samples (skipped). points/el_pos float64 [.,3]. */
int hhsar_bp_gather(const double *points, int64_t n, const double *el_pos, int64_t m,
                    const void *envelopes, int64_t n_t, double t0, double dt,
                    double k_ref, void *out, int64_t *oow, void *stream);

/* lattice_interpolate: values complex64 [nu][nv][nn], coords float64 [n,3]
 * (lattice-index units) -> out complex64 [n], ok uint8 [n]; kernel 0 =
 * linear, 1 = cubic (Keys a = -1/2).  Out-of-hull points give 0, ok = 0. */
int hhsar_lattice_interp(const void *values, int64_t nu, int64_t nv, int64_t nn,
                         const double *coords, int64_t n, int kernel, void *out,
                         uint8_t *ok, void *stream);

/* _invert_newton_jit: float64 targets/guesses [n,3] -> pos [n,3], ok, iters. */
int hhsar_invert_newton(const double *ext4, double k_min, double k_max,
                        const double *targets, const double *guesses, int64_t n,
                        double tol, int max_iter, double max_step, double z_floor,
                        double *pos, uint8_t *ok, int64_t *iters, void *stream);

/* ---- direct BPA --------------------------------------------------------- */

/* Full-aperture BPA on the region_grid voxels (values[nx][ny][nz], z
 * fastest).  Only flattened voxels [vox_begin, vox_end) are computed and
 * written to out[0 .. vox_end - vox_begin) (voxel sharding; vox_end < 0
 * means "to the end").  origin/step/dims are HOST arrays.  el_xyz: float32
 * [m][4] (x, y, z, unused).  oow_total: one int64 accumulated with the
 * number of out-of-window point-element delays. */
int hhsar_bpa_cartesian(const double *origin, const double *step, const int64_t *dims,
                        int64_t vox_begin, int64_t vox_end, const float *el_xyz, int64_t m, const void *envelopes,
                        int64_t n_t, double t0, double dt, double k_ref,
                        void *out, int64_t *oow_total, void *stream);

/* ---- range compression -------------------------------------------------- */

/* Zero-pad cube[n_el][n_f] (complex64) into spec[n_el][n_t]. */
int hhsar_range_pad(const void *cube, int64_t n_el, int64_t n_f, int64_t n_t,
                    void *spec, void *stream);
/* In place: prof[e][i] *= scale * exp(j * a * (dt * i)) with a = (k_min -
 * k_ref) * c (float64 phase per bin, rangecomp.py:94-96); turns the
 * unnormalised IDFT into demodulated envelopes. */
int hhsar_range_demod(void *prof, int64_t n_el, int64_t n_t, double a, double dt,
                      float scale, void *stream);
/* Fused range compression (rangecomp.py:61-101 in one HBM pass): per element
 * row, zero-pad cube[e][0..n_f) to n_t bins, unnormalised inverse DFT,
 * multiply by exp(j a (dt i)); out[n_el][n_t] complex64.  n_t must be a
 * power of two in [16, 8192] (other sizes: cuFFT + hhsar_range_demod). */
int hhsar_range_compress(const void *cube, int64_t n_el, int64_t n_f, int64_t n_t, double a,
                         double dt, void *out, void *stream);

/* The same, keeping only delay bins [b0, b0 + w) of every row (a range
 * gate): out[n_el][w], out[e][i] = envelope[e][b0 + i].  Bins outside the
 * gate are neither stored nor, in the last radix-16 pass, computed; for
 * n_t = 4096 (n_f = 1024 or 512) and n_t = 2048 (n_f = 512 or 256) with
 * w <= 512 a 64-column split with one shared-memory exchange evaluates only
 * the window's bins (a 4- or 2-point DFT per 16-entry column slice, a
 * 16-term Horner chain per bin).  An
 * envelope gated this way is a profile with t0' = t0 + b0 dt and w bins. */
int hhsar_range_compress_window(const void *cube, int64_t n_el, int64_t n_f, int64_t n_t,
                                double a, double dt, int64_t b0, int64_t w, void *out,
                                void *stream);

/* ---- HHFFBPA: grids ------------------------------------------------------ */

/* 3-D bbox of every leaf's elements: el_pos float64 [N][3], bounds int64
 * [n_leaves+1] -> box float64 [n_leaves][6]. */
int hhsar_leaf_boxes(const double *el_pos, const int64_t *bounds, int64_t n_leaves,
                     double *box, void *stream);

/* Lattice metadata of n_grids grids (ffbp.py:226-304 without the Newton
 * part).  boundary: float64 [n_b][3] (region.boundary_lattice(5)).  status
 * (int32, device) receives 1 if any boundary point is outside the
 * compressed-coordinate domain (spectrum.py:253-255).  grids, leaf_box,
 * boundary, status are device pointers; geom is a HOST pointer (as in every
 * call taking an hhsar_geom).  totals (int64 [2], device, optional): when
 * given, every desc.offset / desc.col_offset is set to the exclusive prefix
 * sum of the lattice sizes / active-column counts in grid order and
 * totals = {lattice points, active columns} (the pool and work-list sizes
 * hhsar_grid_newton needs), so the host reads them back with the descs. */
int hhsar_grid_plan(hhsar_grid_desc *grids, int64_t n_grids, const double *leaf_box,
                    const double *boundary, int64_t n_b, const hhsar_geom *geom,
                    int32_t *status, int64_t *totals, void *stream);

/* Range gate of the leaf stage: gate[0] = b0, gate[1] = w (int64, device)
 * such that every delay bin a valid leaf point can read through
 * hhsar_leaf_bp lies in [b0, b0 + w) (w a multiple of 32 unless clipped at
 * n_t), from the plan's descriptors of the n_leaves leaf grids (device
 * descs): the near-band n range of each leaf lattice bounds the vertex
 * distance sum of its valid points, hence their distances to every leaf
 * element.  geom: the plan's (host) geometry.  Feed it to
 * hhsar_range_compress_window.  No reference counterpart: the reference
 * computes every bin (rangecomp.py:61-101). */
int hhsar_leaf_range_gate(const hhsar_grid_desc *leaves, int64_t n_leaves, const hhsar_geom *geom,
                          double dt, int64_t n_t, int64_t *gate, void *stream);

/* Newton inversion of every ACTIVE (u, v) column of every grid (desc.act_*
 * rectangle, at desc.col_offset in a work list of n_cols columns), warm
 * started along n (ffbp.py:271-282), then the containment, near-band and
 * (leaf grids) delay-window masks.  positions float64 [P][3], valid uint8
 * [P] (P = sum of lattice sizes, at desc.offset; the caller zeroes valid,
 * inactive columns are never touched), stats int64
 * [n_grids][HHSAR_GRID_STATS] (zeroed by the caller).  block_grid: optional
 * int32 [ceil(n_cols / 128)], the grid of each 128-column block's first
 * column (device pointer); NULL = the kernel binary-searches col_offset. */
int hhsar_grid_newton(const hhsar_grid_desc *grids, int64_t n_grids, int64_t n_cols,
                      const int32_t *block_grid, const hhsar_geom *geom, double *positions,
                      uint8_t *valid, int64_t *stats, void *stream);

/* ---- HHFFBPA: leaf BPA and merges ----------------------------------------- */

/* Level-1 subimages: for every valid lattice point of every leaf grid,
 * backproject the leaf's elements [desc.start, desc.stop) and store the value
 * at values[desc.offset + i] (complex64; masked points get 0).  With
 * downconvert != 0 the stored value is f * exp(-j Phi_leaf(pos)), ready for
 * the next merge (ffbp.py:343-348).  positions/valid/values are the global
 * lattice pools indexed by desc.offset; the grids' points occupy the pool
 * range [point_begin, point_end) and the largest grid has max_grid_points
 * points (host-known sizes; the kernel compacts the valid points itself).
 * el_xyz float32 [N][4].  oow_total accumulates out-of-window delays. */
int hhsar_leaf_bp(const hhsar_grid_desc *grids, int64_t n_grids, int64_t point_begin,
                  int64_t point_end, int64_t max_grid_points, const double *positions,
                  const uint8_t *valid, const float *el_xyz, const void *envelopes,
                  int64_t n_t, double t0, double dt, double k_ref, const hhsar_geom *geom,
                  int downconvert, void *values, int64_t *oow_total, void *stream);

/* One merge stage over the global lattice pools.  Parents: parent_grids
 * [n_parents] whose points are contiguous from parent_grids[0].offset
 * (n_parent_points in total); parent p merges children [p*fanout,
 * (p+1)*fanout) of child_grids, whose DOWNCONVERTED values are read from
 * values_in.  For each valid parent point: sum over children of
 * interp(f'_c at llt_c(p)) * exp(+j Phi_c(p)); zeroed and counted in
 * *flagged when outside any child's hull (ffbp.py:351-374).  With
 * downconvert != 0 the result is stored times exp(-j Phi_parent(p)).
 * kernel 0 linear, 1 cubic.  geom is a HOST pointer. */
int hhsar_merge_level(const hhsar_grid_desc *parent_grids, int64_t n_parents,
                      int64_t n_parent_points, const double *positions, const uint8_t *valid,
                      const hhsar_grid_desc *child_grids, int64_t n_child_grids, int fanout,
                      const void *values_in, const hhsar_geom *geom, int kernel,
                      int downconvert, void *values_out, int64_t *flagged, void *stream);

/* In place values[i] *= exp(-j Phi_grid(pos_i)) on valid points, 0 on masked
 * ones, for the points of grids[0..n_grids) (contiguous from grids[0].offset);
 * _downconvert_samples (ffbp.py:343-348) for the single-merge API. */
int hhsar_downconvert(const hhsar_grid_desc *grids, int64_t n_grids, int64_t n_points,
                      const double *positions, const uint8_t *valid, const hhsar_geom *geom,
                      void *values, void *stream);

/* Final landing on the Cartesian region_grid voxels [nx][ny][nz] (z
 * fastest), all n_children children, no downconversion (ffbp.py:493-495).
 * Voxels [vox_begin, vox_end) of the flattened volume are written to
 * out[0 .. vox_end - vox_begin) (voxel sharding across GPUs).  The
 * children's lattices occupy pool points [span_begin, span_begin +
 * span_points) of child_values; with span_points > 0 the landing stages a
 * 16-byte (v[i], v[i+1]) pair copy of that span for its gathers
 * (span_points = 0: gathers from child_values directly).  The z-series
 * evaluation is used where its truncation is negligible; kernel |
 * HHSAR_LANDING_PER_VOXEL forces the per-voxel float64 form. */
#define HHSAR_LANDING_PER_VOXEL 16
int hhsar_merge_cartesian(const double *origin, const double *step, const int64_t *dims,
                          int64_t vox_begin, int64_t vox_end,
                          const hhsar_grid_desc *child_grids, int64_t n_children,
                          const void *child_values, int64_t span_begin, int64_t span_points,
                          const hhsar_geom *geom, int kernel, void *out, int64_t *flagged,
                          void *stream);

/* ---- input synthesis ------------------------------------------------------ */

/* Born cube s[e][f] = sum_q refl_q exp(-2j k_f |el_e - pos_q|) (complex64
 * out; float64 phases).  refl complex128 [n_s]. */
int hhsar_simulate(const double *el_pos, int64_t n_el, const double *pos,
                   const double *refl, int64_t n_s, const double *k, int64_t n_f,
                   void *out, void *stream);

/* The same Born cube on a uniform frequency grid k_f = k0 + f dk (every
 * FrequencyGrid, model.py:30-70): float64 distance and phase seed per 8
 * frequencies, fp32 phasor recurrence and accumulation (~1e-5 relative to
 * hhsar_simulate; the input generator for the large configs).  n_f <= 2048. */
int hhsar_simulate_uniform(const double *el_pos, int64_t n_el, const double *pos,
                           const double *refl, int64_t n_s, double k0, double dk, int64_t n_f,
                           void *out, void *stream);

/* ---- image-quality metrics ------------------------------ */

/* psnr (metrics.py:126-150), pass 1: out5 (device, float64) = [sum |t|^2,
 * Re sum conj(t) r, Im sum conj(t) r, sum |r|^2, max |r|] over n complex
 * samples (dtype 0 = complex64, 1 = complex128), float64 accumulation in a
 * fixed reduction order.  np.vdot(tst, ref) = out5[1] + j out5[2]. */
int hhsar_volume_dot(const void *test, const void *ref, int64_t n, int dtype, double *out5,
                     void *stream);

/* psnr pass 2: out1 (device) = sum |s t - r|^2 for the complex scale s. */
int hhsar_volume_residual(const void *test, const void *ref, int64_t n, int dtype,
                          double scale_re, double scale_im, double *out1, void *stream);

/* max_intensity_projection (metrics.py:170-190): out (device, float64) =
 * per-pixel max |v| along `axis` of the [dims[0]][dims[1]][dims[2]] volume
 * (dims host), dB-scaled to its own peak, clipped at floor_db < 0 and mapped
 * onto [0, 1]; an all-zero volume gives zeros. */
int hhsar_mip(const void *volume, const int64_t *dims, int dtype, int axis, double floor_db,
              double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HHSAR_B200_H */
