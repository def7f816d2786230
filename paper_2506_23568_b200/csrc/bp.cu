// Backprojection gather kernels (reference: _kernels.py:44-110, bpa.py:144-176).
//
// One "unit" is one (voxel, element) pair: distance, delay-bin lookup with
// linear interpolation of the complex64 envelope, carrier phase exp(j 2 k_ref
// d) with explicit range reduction, complex accumulate.  FP32 + SFU bound;
// element positions are staged in shared memory per chunk and broadcast.
#include "common.cuh"

namespace hhsar {

constexpr int BP_THREADS = 256;
constexpr int BP_CHUNK = 512;   // elements staged per shared-memory pass

struct BpConst {
    float inv_bin;   // 2 / (c * dt): metres -> delay-bin index
    float x0;        // t0 / dt
    float rev;       // k_ref / pi: metres -> carrier revolutions (2 k_ref d / 2 pi)
    float xmax;      // n_t - 1
    int n_t;
};

// One unit: returns false (and contributes nothing) when the delay is outside
// the profile window, exactly like the reference's skip-and-count.
__device__ __forceinline__ bool bp_unit(float d, const BpConst &k, const float2 *__restrict__ row,
                                        float2 &acc) {
    const float x = fmaf(d, k.inv_bin, -k.x0);
    if (!(x >= 0.f && x <= k.xmax)) return false;
    int i = min((int)x, k.n_t - 2);
    const float f = x - (float)i;
    const float2 v0 = __ldg(row + i), v1 = __ldg(row + i + 1);
    const float er = fmaf(f, v1.x - v0.x, v0.x), ei = fmaf(f, v1.y - v0.y, v0.y);
    // carrier exp(j k_ref c tau) = exp(j 2 pi * d k_ref / pi): reduce the
    // revolution count to [-0.5, 0.5] before the SFU sincos
    const float rv = d * k.rev;
    const float red = __fsub_rn(rv, rintf(rv));
    float s, c;
    __sincosf(6.283185307f * red, &s, &c);
    acc.x = fmaf(er, c, fmaf(-ei, s, acc.x));
    acc.y = fmaf(er, s, fmaf(ei, c, acc.y));
    return true;
}

// ---------------------------------------------------------------------------
// Tiled Cartesian BPA (the config-1 hot kernel).
//
// A CTA owns a VX x TY x TZ voxel tile (each thread VX voxels along x) and
// walks the elements in chunks.  Per chunk and element it derives the delay
// window the whole tile can touch (point-to-box distance .. farthest box
// corner, +-2 bins) and stages just those bins into shared memory as
// (v_i, v_{i+1} - v_i) float4 pairs, so every unit does ONE 16-byte LDS and
// two FMAs for the envelope interpolation.  Elements whose window is wider
// than TW bins or touches the profile edges take a per-unit checked path
// (global loads, exact out-of-window skip-and-count) -- a block-uniform
// branch, so the fast path carries no per-unit bounds checks: the tile-level
// window proves every delay is inside [0, n_t-1].
// Floor/fraction and the carrier revolution count use the 1.5*2^23
// round-to-integer trick on the FMA pipe (no F2I/I2F/FRND), sqrt is the SFU
// approximation, and sin/cos take an explicitly range-reduced argument.
// ---------------------------------------------------------------------------
constexpr int TL_TY = 16, TL_TZ = 16;  // VX x 16 x 16 voxels per tile (VX: template)
constexpr int TL_THREADS = TL_TY * TL_TZ;
constexpr int TL_CHUNK = 64;   // elements per staging pass
constexpr int TL_W = 32;       // staged bins per element (32 x 16 B = 512 B)
constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23
constexpr unsigned MAGIC_BITS = 0x4B400000u;

struct BpFast {
    float inv_bin, x0, rev, xmax;
    float cbin;    // -0.5 - x0
    float kfrac;   // MAGIC - x0
    float alpha;   // k_ref c dt: carrier radians per delay bin
    int n_t;
    double alpha_d;  // the same in float64 (staging)
    double kc_t0;    // k_ref c t0
};

template <int VX, int MINB, bool PAIR>
__global__ void __launch_bounds__(TL_THREADS, MINB)
bpa_tile_kernel(double ox, double oy, double oz, double sx, double sy, double sz, int nx, int ny,
                int nz, int64_t vb, int64_t ve, const float4 *__restrict__ el, int m,
                const float2 *__restrict__ env, BpFast k, float2 *__restrict__ out,
                int64_t *__restrict__ oow_total, int tx_base, int n_tiles, int split,
                float2 *__restrict__ part, int *__restrict__ arrivals,
                const float2 *__restrict__ rot) {
    constexpr int TL_VX = VX;  // voxels per thread along x
    __shared__ float4 s_env[TL_CHUNK * TL_W];  // 32 KB
    __shared__ float4 s_el[TL_CHUNK];          // x, y, z, bits(byte offset | -1 = slow)
    __shared__ int s_lo[TL_CHUNK];
    const int tiles_z = (nz + TL_TZ - 1) / TL_TZ, tiles_y = (ny + TL_TY - 1) / TL_TY;
    // work item = (tile, element split s), tile-major: a tile's split CTAs
    // run at about the same time, so the partial-sum slabs they exchange
    // (below) live only briefly in L2; the envelope rows the resident CTAs
    // read at any moment stay a few MB (every CTA walks its element range
    // in step with the others)
    const int sidx = blockIdx.x % split;
    const int b = blockIdx.x / split;
    const int tz = b % tiles_z, ty = (b / tiles_z) % tiles_y;
    const int tx = tx_base + b / (tiles_z * tiles_y);
    const int per = ((m + split - 1) / split + TL_CHUNK - 1) / TL_CHUNK * TL_CHUNK;
    const int e_begin = min(m, sidx * per), e_end = min(m, e_begin + per);
    const int t = threadIdx.x;
    const int iz = tz * TL_TZ + (t % TL_TZ), iy = ty * TL_TY + (t / TL_TZ), ix0 = tx * TL_VX;
    const int izc = min(iz, nz - 1), iyc = min(iy, ny - 1);
    // voxel coordinates exactly as numpy builds them (origin + step * i), then f32
    const float py = (float)__dadd_rn(oy, __dmul_rn(sy, (double)iyc));
    const float pz = (float)__dadd_rn(oz, __dmul_rn(sz, (double)izc));
    float px[TL_VX];
#pragma unroll
    for (int v = 0; v < TL_VX; ++v)
        px[v] = (float)__dadd_rn(ox, __dmul_rn(sx, (double)min(ix0 + v, nx - 1)));
    // flattened index / ownership of voxel v, recomputed where needed (keeps
    // the inner loop's register budget for the accumulators)
    auto flat_of = [&](int v) { return ((int64_t)(ix0 + v) * ny + iy) * nz + iz; };
    auto live_of = [&](int v) {
        const int64_t f = flat_of(v);
        return ix0 + v < nx && iy < ny && iz < nz && f >= vb && f < ve;
    };
    // tile bounding box (float32, from the clamped corner voxels)
    const float bx0 = (float)__dadd_rn(ox, __dmul_rn(sx, (double)min(ix0, nx - 1)));
    const float bx1 = (float)__dadd_rn(ox, __dmul_rn(sx, (double)min(ix0 + TL_VX - 1, nx - 1)));
    const float by0 = (float)__dadd_rn(oy, __dmul_rn(sy, (double)min(ty * TL_TY, ny - 1)));
    const float by1 = (float)__dadd_rn(oy, __dmul_rn(sy, (double)min(ty * TL_TY + TL_TY - 1, ny - 1)));
    const float bz0 = (float)__dadd_rn(oz, __dmul_rn(sz, (double)min(tz * TL_TZ, nz - 1)));
    const float bz1 = (float)__dadd_rn(oz, __dmul_rn(sz, (double)min(tz * TL_TZ + TL_TZ - 1, nz - 1)));

    static_assert(!PAIR || VX % 2 == 0, "pair path needs an even VX");
    float2 acc[PAIR ? 1 : TL_VX];
    f2x pa[PAIR ? TL_VX : 1], pb[PAIR ? TL_VX : 1];
#pragma unroll
    for (int v = 0; v < (PAIR ? TL_VX : 1); ++v) pa[v] = pb[v] = pk2(0.f, 0.f);
#pragma unroll
    for (int v = 0; v < (PAIR ? 1 : TL_VX); ++v) acc[v] = make_float2(0.f, 0.f);
    unsigned bad = 0;
    const BpConst kc{k.inv_bin, k.x0, k.rev, k.xmax, k.n_t};

    for (int c0 = e_begin; c0 < e_end; c0 += TL_CHUNK) {
        const int cn = min(TL_CHUNK, e_end - c0);
        __syncthreads();
        if (t < cn) {
            const float4 e = el[c0 + t];
            const float qx = fminf(fmaxf(e.x, bx0), bx1) - e.x;
            const float qy = fminf(fmaxf(e.y, by0), by1) - e.y;
            const float qz = fminf(fmaxf(e.z, bz0), bz1) - e.z;
            const float fx = fmaxf(fabsf(e.x - bx0), fabsf(e.x - bx1));
            const float fy = fmaxf(fabsf(e.y - by0), fabsf(e.y - by1));
            const float fz = fmaxf(fabsf(e.z - bz0), fabsf(e.z - bz1));
            const float xlo = sqrtf(qx * qx + qy * qy + qz * qz) * k.inv_bin - k.x0;
            const float xhi = sqrtf(fx * fx + fy * fy + fz * fz) * k.inv_bin - k.x0;
            const int lo = max((int)floorf(xlo) - 2, 0);
            const int hi = min((int)floorf(xhi) + 2, k.n_t - 1);
            const bool fast = xlo >= 1.f && xhi <= k.xmax - 1.f && hi - lo + 1 <= TL_W;
            const unsigned off = (unsigned)(t * TL_W - lo) * 16u - MAGIC_BITS * 16u;
            s_el[t] = make_float4(e.x, e.y, e.z, __int_as_float(fast ? (int)off : -1));
            s_lo[t] = fast ? lo : -1;
        }
        __syncthreads();
        for (int q = t; q < cn * TL_W; q += TL_THREADS) {
            const int j = q / TL_W, lo = s_lo[j];
            if (lo < 0) continue;
            const int bin = lo + (q % TL_W);
            const float2 *row = env + (int64_t)(c0 + j) * k.n_t;
            const float2 v0 = __ldg(row + min(bin, k.n_t - 1));
            const float2 v1 = __ldg(row + min(bin + 1, k.n_t - 1));
            // pre-rotate by the carrier at the bin: exp(j k_ref c (t0 + bin dt)),
            // float64 phase rounded once, from the per-launch table (keeps the
            // staging's sincos and conversions off the SFU the units saturate)
            const float2 r = __ldg(rot + bin);
            const float2 dv = bin < k.n_t - 1 ? make_float2(v1.x - v0.x, v1.y - v0.y)
                                              : make_float2(0.f, 0.f);
            const float2 a = cmul(v0, r), b2 = cmul(dv, r);
            s_env[q] = make_float4(a.x, a.y, b2.x, b2.y);
        }
        __syncthreads();
        for (int j = 0; j < cn; ++j) {
            const float4 e = s_el[j];
            const float dy = py - e.y, dz = pz - e.z;
            const float dyz = fmaf(dy, dy, dz * dz);
            const int offb = __float_as_int(e.w);
            // one fast unit at distance d: window lookup + lerp + carrier + MAC
            auto unit = [&](float d, unsigned base, float2 &a) {
                // i = round(x - 0.5) = floor(x) (x - 1 at exact integers, f = 1):
                // MAGIC + (x - 0.5) rounds at the units place.  (MAGIC - 0.5 is
                // not an fp32 number, so the 0.5 shift cannot ride in one FFMA.)
                const float tb = __fadd_rn(fmaf(d, k.inv_bin, k.cbin), MAGIC);
                // f = x - i = d * inv_bin + (MAGIC - x0 - tb): one rounding
                const float f = fmaf(d, k.inv_bin, __fsub_rn(k.kfrac, tb));
                const unsigned byte = (unsigned)__float_as_int(tb) * 16u + base;
                const float4 w = *reinterpret_cast<const float4 *>(
                    reinterpret_cast<const char *>(s_env) + byte);
                const float er = fmaf(f, w.z, w.x), ei = fmaf(f, w.w, w.y);
                // The carrier k_ref c tau = alpha (x + x0) splits into the
                // staged bin rotation (alpha (i + x0), exact float64) and
                // alpha f with f in [0, 1]: the explicit range reduction is
                // free and the SFU sees |angle| <= alpha (a few revolutions).
                float s, c;
                __sincosf(k.alpha * f, &s, &c);
                a.x = fmaf(er, c, fmaf(-ei, s, a.x));
                a.y = fmaf(er, s, fmaf(ei, c, a.y));
            };
            if (PAIR && offb != -1) {  // compile-time PAIR
                // Voxels in pairs with packed fp32x2 arithmetic (FADD2/FFMA2/
                // FMUL2): same per-lane operations and roundings as `unit`,
                // half the FMA-pipe issue slots.  The complex MAC is kept as two
                // pair accumulators A += (er, ei) c, B += (er, ei) s, combined
                // once at the end: re = A.x - B.y, im = A.y + B.x.
                const unsigned base = (unsigned)offb;
                const f2x nex = bc2(-e.x), vdyz = bc2(dyz);
#pragma unroll
                for (int v = 0; v < TL_VX; v += 2) {
                    const f2x dx = add2(pk2(px[v], px[v + 1]), nex);
                    const f2x a2 = fma2(dx, dx, vdyz);
                    const f2x d = pk2(sqrt_approx(lo2(a2)), sqrt_approx(hi2(a2)));
                    const f2x tb = add2(fma2(d, bc2(k.inv_bin), bc2(k.cbin)), bc2(MAGIC));
                    const f2x f = fma2(d, bc2(k.inv_bin), sub2(bc2(k.kfrac), tb));
                    const unsigned b0 = (unsigned)__float_as_int(lo2(tb)) * 16u + base;
                    const unsigned b1 = (unsigned)__float_as_int(hi2(tb)) * 16u + base;
                    const float4 w0 = *reinterpret_cast<const float4 *>(
                        reinterpret_cast<const char *>(s_env) + b0);
                    const float4 w1 = *reinterpret_cast<const float4 *>(
                        reinterpret_cast<const char *>(s_env) + b1);
                    const f2x e0 = fma2(bc2(lo2(f)), pk2(w0.z, w0.w), pk2(w0.x, w0.y));
                    const f2x e1 = fma2(bc2(hi2(f)), pk2(w1.z, w1.w), pk2(w1.x, w1.y));
                    const f2x ang = mul2(f, bc2(k.alpha));
                    float s0, c0, s1, c1;
                    __sincosf(lo2(ang), &s0, &c0);
                    __sincosf(hi2(ang), &s1, &c1);
                    pa[v] = fma2(e0, bc2(c0), pa[v]);
                    pb[v] = fma2(e0, bc2(s0), pb[v]);
                    pa[v + 1] = fma2(e1, bc2(c1), pa[v + 1]);
                    pb[v + 1] = fma2(e1, bc2(s1), pb[v + 1]);
                }
            } else if (offb != -1) {
                const unsigned base = (unsigned)offb & ~1u;
#pragma unroll
                for (int v = 0; v < TL_VX; ++v) {
                    const float dx = px[v] - e.x;
                    unit(sqrt_approx(fmaf(dx, dx, dyz)), base, acc[v]);
                }
            } else {
                const float2 *row = env + (int64_t)(c0 + j) * k.n_t;
#pragma unroll
                for (int v = 0; v < TL_VX; ++v) {
                    const float dx = px[v] - e.x;
                    const float d = sqrtf(fmaf(dx, dx, dyz));
                    float2 a = make_float2(0.f, 0.f);
                    const bool ok = bp_unit(d, kc, row, a);
                    if (live_of(v)) {
                        if constexpr (PAIR) {
                            pa[v] = add2(pa[v], pk2(a.x, a.y));  // (re, im) of the term
                        } else {
                            acc[v].x += a.x;
                            acc[v].y += a.y;
                        }
                        bad += !ok;
                    }
                }
            }
        }
    }
    if (bad) atomicAdd((unsigned long long *)oow_total, (unsigned long long)bad);
    float2 mine[TL_VX];
#pragma unroll
    for (int v = 0; v < TL_VX; ++v) {
        if constexpr (PAIR)
            mine[v] = make_float2(lo2(pa[v]) - hi2(pb[v]), hi2(pa[v]) + lo2(pb[v]));
        else
            mine[v] = acc[v];
    }
    if (split == 1) {
#pragma unroll
        for (int v = 0; v < TL_VX; ++v)
            if (live_of(v)) out[flat_of(v) - vb] = mine[v];
        return;
    }
    // split > 1: the tile's CTAs each park their partial sums (8 KB) in a
    // per-tile scratch slab; the LAST one to finish (per-tile arrival counter)
    // adds the slabs in split order -- deterministic, no second kernel, and
    // the slabs live only as long as the tile is in flight, so they stay in
    // L2 instead of round-tripping through HBM
    constexpr int SLOTS = TL_THREADS * TL_VX;
    float2 *slab = part + ((int64_t)b * split + sidx) * SLOTS;
#pragma unroll
    for (int v = 0; v < TL_VX; ++v) slab[t * TL_VX + v] = mine[v];
    __threadfence();
    __shared__ int s_last;
    __syncthreads();
    if (t == 0) s_last = atomicAdd(arrivals + b, 1) == split - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();  // every other slab of the tile is visible
    float2 sum[TL_VX];
#pragma unroll
    for (int v = 0; v < TL_VX; ++v) sum[v] = make_float2(0.f, 0.f);
    for (int r = 0; r < split; ++r) {
        const float2 *src = part + ((int64_t)b * split + r) * SLOTS + t * TL_VX;
#pragma unroll
        for (int v = 0; v < TL_VX; ++v) {
            const float2 p = r == sidx ? mine[v] : __ldcg(src + v);
            sum[v].x += p.x;
            sum[v].y += p.y;
        }
    }
#pragma unroll
    for (int v = 0; v < TL_VX; ++v)
        if (live_of(v)) out[flat_of(v) - vb] = sum[v];
    // the slabs are dead: drop their L2 lines without writing them back
    // (discard.global.L2), so the scratch never reaches HBM
    __syncthreads();  // every thread of this CTA has read the slabs
    constexpr int LINES = SLOTS * (int)sizeof(float2) / 128;  // per slab
    const char *tile_slabs = reinterpret_cast<const char *>(part + (int64_t)b * split * SLOTS);
    for (int l = t; l < split * LINES; l += TL_THREADS)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(tile_slabs + (int64_t)l * 128)
                     : "memory");
}

// Generic gather for arbitrary points (operator-level backproject_gather).
__global__ void __launch_bounds__(BP_THREADS)
bp_gather_kernel(const double *__restrict__ pts, int64_t n, const float4 *__restrict__ el, int m,
                 const float2 *__restrict__ env, BpConst k, float2 *__restrict__ out,
                 int64_t *__restrict__ oow) {
    __shared__ float4 s_el[BP_CHUNK];
    const int64_t p = (int64_t)blockIdx.x * BP_THREADS + threadIdx.x;
    const bool live = p < n;
    float px = 0.f, py = 0.f, pz = 0.f;
    if (live) {
        px = (float)pts[3 * p];
        py = (float)pts[3 * p + 1];
        pz = (float)pts[3 * p + 2];
    }
    float2 acc = make_float2(0.f, 0.f);
    int64_t bad = 0;
    for (int c0 = 0; c0 < m; c0 += BP_CHUNK) {
        const int cn = min(BP_CHUNK, m - c0);
        __syncthreads();
        for (int j = threadIdx.x; j < cn; j += BP_THREADS) s_el[j] = el[c0 + j];
        __syncthreads();
        if (live)
            for (int j = 0; j < cn; ++j) {
                const float4 e = s_el[j];
                const float dx = px - e.x, dy = py - e.y, dz = pz - e.z;
                const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                bad += !bp_unit(d, k, env + (int64_t)(c0 + j) * k.n_t, acc);
            }
    }
    if (live) {
        out[p] = acc;
        oow[p] = bad;
    }
}

__global__ void el_to_f32x4(const double *__restrict__ el, int64_t m, float4 *__restrict__ o) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) o[i] = make_float4((float)el[3 * i], (float)el[3 * i + 1], (float)el[3 * i + 2], 0.f);
}

// Element-split factor that best fills the last wave: work items = tiles x
// split, resident slots = SMs x CTAs/SM; pick split in [1, 8] maximising
// items / (slots * ceil(items / slots)) (ties -> smaller split).
int tile_split(int64_t tiles, int64_t m, int per_sm) {
    const double slots = (double)sm_count() * (per_sm > 0 ? per_sm : 1);
    int best = 1;
    double best_eff = 0.0;
    for (int sp = 1; sp <= 8 && (int64_t)sp * TL_CHUNK <= m; ++sp) {
        const double waves = tiles * (double)sp / slots;
        const double eff = waves / ceil(waves);
        if (eff > best_eff + 0.01) {
            best_eff = eff;
            best = sp;
        }
    }
    return best;
}

// exp(j k_ref c (t0 + dt bin)) per delay bin (float64 phase, reduced, then
// the fp32 sincos), shared by every element's window staging
__global__ void bp_rot_kernel(float2 *__restrict__ rot, int n_t, double kc_t0, double alpha_d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_t) rot[i] = cis_reduced(kc_t0 + alpha_d * (double)i);
}

struct TileArgs {
    const double *origin, *step;
    int nx, ny, nz;
    int64_t vb, ve;
    const float4 *el;
    int m;
    const float2 *env;
    BpFast k;
    float2 *out;
    int64_t *oow;
    const float2 *rot;
    cudaStream_t s;
};

template <int VX, int MINB, bool PAIR>
int launch_tile(const TileArgs &a) {
    const int per_sm = occupancy((const void *)bpa_tile_kernel<VX, MINB, PAIR>, TL_THREADS);
    // only tiles intersecting [vb, ve) matter; x-slab sharding keeps that a
    // contiguous run of tile columns
    const int64_t plane = (int64_t)a.ny * a.nz;
    const int tx0 = (int)((a.vb / plane) / VX);
    const int tx1 = (int)(((a.ve - 1) / plane) / VX);
    const int64_t per_x = (int64_t)((a.ny + TL_TY - 1) / TL_TY) * ((a.nz + TL_TZ - 1) / TL_TZ);
    const int64_t tiles = (int64_t)(tx1 - tx0 + 1) * per_x;
    const int split = tile_split(tiles, a.m, per_sm);
    float2 *part = nullptr;
    int *arrivals = nullptr;
    if (split > 1) {
        const size_t slab = (size_t)TL_THREADS * VX * sizeof(float2);
        if (cudaMallocAsync(&part, (size_t)tiles * split * slab + tiles * sizeof(int), a.s) !=
            cudaSuccess)
            return set_error(HHSAR_ECUDA, "bpa_cartesian: scratch allocation failed");
        arrivals = reinterpret_cast<int *>(reinterpret_cast<char *>(part) + tiles * split * slab);
        cudaMemsetAsync(arrivals, 0, tiles * sizeof(int), a.s);
    }
    bpa_tile_kernel<VX, MINB, PAIR><<<(unsigned)(tiles * split), TL_THREADS, 0, a.s>>>(
        a.origin[0], a.origin[1], a.origin[2], a.step[0], a.step[1], a.step[2], a.nx, a.ny, a.nz,
        a.vb, a.ve, a.el, a.m, a.env, a.k, a.out, a.oow, tx0, (int)tiles, split, part, arrivals,
        a.rot);
    if (part) cudaFreeAsync(part, a.s);
    return check_launch("bpa_tile_kernel");
}

BpConst make_bp_const(int64_t n_t, double t0, double dt, double k_ref) {
    BpConst k;
    k.inv_bin = (float)(2.0 / (HHSAR_C_LIGHT * dt));
    k.x0 = (float)(t0 / dt);
    k.rev = (float)(k_ref / 3.141592653589793);
    k.xmax = (float)(n_t - 1);
    k.n_t = (int)n_t;
    return k;
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_bpa_cartesian(const double *origin, const double *step, const int64_t *dims,
                                   int64_t vox_begin, int64_t vox_end, const float *el_xyz,
                                   int64_t m, const void *envelopes, int64_t n_t, double t0,
                                   double dt, double k_ref, void *out, int64_t *oow_total,
                                   void *stream) {
    HHSAR_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "bpa_cartesian: empty dims");
    HHSAR_REQUIRE(n_t >= 2, "bpa_cartesian: n_t must be >= 2");
    HHSAR_REQUIRE(m >= 0 && m < (1ll << 31), "bpa_cartesian: bad element count");
    const int64_t total = dims[0] * dims[1] * dims[2];
    if (vox_end < 0 || vox_end > total) vox_end = total;
    HHSAR_REQUIRE(vox_begin >= 0 && vox_begin <= vox_end, "bpa_cartesian: bad voxel range");
    if (vox_begin == vox_end) return HHSAR_OK;
    const int nx = (int)dims[0], ny = (int)dims[1], nz = (int)dims[2];
    cudaStream_t s = as_stream(stream);
    if (m == 0) {
        cudaMemsetAsync(out, 0, (vox_end - vox_begin) * sizeof(float2), s);
        return check_launch("bpa_cartesian memset");
    }
    {
        BpFast k;
        const BpConst c = make_bp_const(n_t, t0, dt, k_ref);
        k.inv_bin = c.inv_bin;
        k.x0 = c.x0;
        k.rev = c.rev;
        k.xmax = c.xmax;
        k.n_t = c.n_t;
        k.cbin = -0.5f - c.x0;
        k.kfrac = MAGIC - c.x0;
        k.alpha_d = k_ref * HHSAR_C_LIGHT * dt;
        k.alpha = (float)k.alpha_d;
        k.kc_t0 = k_ref * HHSAR_C_LIGHT * t0;
        float2 *rot = nullptr;
        if (cudaMallocAsync(&rot, n_t * sizeof(float2), s) != cudaSuccess)
            return set_error(HHSAR_ECUDA, "bpa_cartesian: table allocation failed");
        bp_rot_kernel<<<(unsigned)((n_t + 255) / 256), 256, 0, s>>>(rot, (int)n_t, k.kc_t0,
                                                                    k.alpha_d);
        const TileArgs a{origin, step, nx, ny, nz, vox_begin, vox_end,
                         reinterpret_cast<const float4 *>(el_xyz), (int)m,
                         reinterpret_cast<const float2 *>(envelopes), k,
                         reinterpret_cast<float2 *>(out), oow_total, rot, s};
        // 4 voxels per thread, 5 CTAs/SM, packed fp32x2 voxel pairs
        // (measured fastest of the VX / CTAs-per-SM / pair variants on B200)
        const int rc = launch_tile<4, 5, true>(a);
        cudaFreeAsync(rot, s);
        return rc;
    }
}

extern "C" int hhsar_bp_gather(const double *points, int64_t n, const double *el_pos, int64_t m,
                               const void *envelopes, int64_t n_t, double t0, double dt,
                               double k_ref, void *out, int64_t *oow, void *stream) {
    HHSAR_REQUIRE(n >= 0 && m >= 0 && m < (1ll << 31), "bp_gather: bad sizes");
    HHSAR_REQUIRE(n_t >= 2, "bp_gather: n_t must be >= 2");
    if (n == 0) return HHSAR_OK;
    cudaStream_t s = as_stream(stream);
    if (m == 0) {
        cudaMemsetAsync(out, 0, n * sizeof(float2), s);
        cudaMemsetAsync(oow, 0, n * sizeof(int64_t), s);
        return check_launch("bp_gather memset");
    }
    float4 *el4 = nullptr;
    if (cudaMallocAsync(&el4, m * sizeof(float4), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "bp_gather: allocation failed");
    el_to_f32x4<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(el_pos, m, el4);
    bp_gather_kernel<<<(unsigned)((n + BP_THREADS - 1) / BP_THREADS), BP_THREADS, 0, s>>>(
        points, n, el4, (int)m, reinterpret_cast<const float2 *>(envelopes),
        make_bp_const(n_t, t0, dt, k_ref), reinterpret_cast<float2 *>(out), oow);
    cudaFreeAsync(el4, s);
    return check_launch("bp_gather_kernel");
}
