// k_search: initial_poses + local_search (search.cpp:84-193) on sm_100a.
//
// One warp owns one (ligand, restart) work item; warps pull items from a
// global atomic counter (persistent grid, CTAs of 4 warps, as many CTAs per
// SM as registers and shared memory allow).  Per local_search iteration the
// warp evaluates the 12 + 2m neighbours of search.cpp:152-176:
//
//   * neighbour x heavy-atom samples are flattened into one item list and
//     spread over the 32 lanes (rigid neighbours: every heavy atom; torsion
//     neighbour (t, +-): only the heavy atoms of D_t, the atoms whose
//     coordinates can depend on torsion t -- every other atom follows a
//     bit-identical trajectory, so its sample equals the current pose's);
//   * each neighbour's geo_score is then summed by one lane in heavy-atom
//     order (grid.cpp:97-101), reading the per-atom values back from shared
//     memory -- the reference's sequential double sum, bit for bit;
//   * the strictly best neighbour (first wins on ties, search.cpp:138) is a
//     warp shuffle reduction over the scores.
//
// The neighbourhood is processed in groups of at most G neighbours (rigid
// group first, then torsion groups in order), keeping a running best, so the
// per-warp buffer holds G rows instead of 12 + 2m.  Torsion-neighbour
// matrices depend only on the torsion state and the step, so they are
// rebuilt only after a torsion move or a step halving; the pivot only after
// a move.  All arithmetic is FP64 in the reference's evaluation order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../../include/vs_crtrig.h"
#include "../../../include/vs_dock.h"
#include "kernels.cuh"

namespace vsd {

namespace {

#ifndef VS_SEARCH_WARPS
#define VS_SEARCH_WARPS 2  // warps per CTA: small CTAs pack shared memory tighter (measured)
#endif
constexpr int kWarps = VS_SEARCH_WARPS;
#ifndef VS_SEARCH_GROUP
#define VS_SEARCH_GROUP 12
#endif
// Development bounds checks (build with -DVS_DEBUG_CHECKS): trap on an
// out-of-range shared-memory / scratch index instead of corrupting state.
#ifdef VS_DEBUG_CHECKS
#define VS_CHECK(c) \
  do {              \
    if (!(c)) __trap(); \
  } while (0)
#else
#define VS_CHECK(c) \
  do {              \
  } while (0)
#endif
#ifndef VS_ROW_SELECT
#define VS_ROW_SELECT 1  // torsion rows read non-D_t atoms from vcur instead of completing the rows
#endif
#ifndef VS_TORSH_SMEM
#define VS_TORSH_SMEM 1  // heavy atoms' torsioned frame also in shared memory (0: read it from the
                         // global frame -- measured 2% slower; frees 3n doubles per warp)
#endif
#if VS_TORSH_SMEM
#define TORSH(h, a) (torsh + 3 * (h))
#else
#define TORSH(h, a) (hx + 3 * (a))  // the warp's global frame (L1)
#endif
constexpr int kPalDoubles = 32;  // palette / code-pair table at the start of shared memory
constexpr int kRow = 18;  // spin-neighbour row: R (9), pad, t (3), pad, q (4)
constexpr int kGroup = VS_SEARCH_GROUP;  // neighbours per group (>= 12, even; 12 measured best)
constexpr double kPi = 3.14159265358979323846;
constexpr double kLatticeStep = 2.0 * kPi / 36;

__device__ __forceinline__ d3 ld3(const double *p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double *p, d3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

// 12-double blocks (rotation + translation / pivot) at 16-byte aligned
// shared-memory addresses, read with 128-bit loads.
__device__ __forceinline__ void ld12a(const double *p, double r[12]) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
  #pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double2 v = q[i];
    r[2 * i] = v.x;
    r[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ d3 torsion_apply_a(const double *m, d3 x) {
  double r[12];
  ld12a(m, r);
  return torsion_apply(r, x);
}
// Rotation (9 doubles) and translation (3) at two 16-byte aligned addresses.
__device__ __forceinline__ d3 rigid_col_rt(const double *R, const double *T, d3 v, int col) {
  double r[9], t[3];
  const double2 *q = reinterpret_cast<const double2 *>(R);
  #pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double2 w = q[i];
    r[2 * i] = w.x;
    r[2 * i + 1] = w.y;
  }
  r[8] = R[8];
  const double2 w = *reinterpret_cast<const double2 *>(T);
  t[0] = w.x;
  t[1] = w.y;
  t[2] = T[2];
  return rigid_col(r, t, v, col);
}

// sin/cos of a as double-double: hi parts to sc[0], sc[1], lo parts to
// lo[0], lo[1].  Out of line: the search only needs it at a restart's start
// (arbitrary angles) and next to zeros of sin/cos (vs_crtrig sincos_shift).
__device__ __noinline__ void sincos_dd_dev(double a, double *sc, double *lo) {
  vs_crtrig::dd s, c;
  vs_crtrig::sincos_dd(a, &s, &c);
  sc[0] = s.hi;
  sc[1] = c.hi;
  lo[0] = s.lo;
  lo[1] = c.lo;
}

__constant__ double c_lattice_sc_s[72];
__constant__ double c_lattice_lo_s[72];  // lo parts of the double-double lattice sin/cos

// Development-only phase profile (build with -DVS_PHASE_PROF): per-warp
// clock64() time spent in each phase of the search, summed over warps.
#ifdef VS_PHASE_PROF
__device__ unsigned long long g_phase[24];
#define PH_DECL                        \
  unsigned long long ph_t = clock64(); \
  unsigned long long ph_acc[24] = {0};
#define PH(k)                                 \
  {                                           \
    __syncwarp();                             \
    const unsigned long long ph_now = clock64(); \
    ph_acc[k] += ph_now - ph_t;               \
    ph_t = ph_now;                            \
  }
#define PH_FLUSH \
  if (lane == 0) \
    for (int i = 0; i < 24; ++i) atomicAdd(&g_phase[i], ph_acc[i]);
#else
#define PH_DECL
#define PH(k)
#define PH_FLUSH
#endif
__device__ __forceinline__ double c_lattice_sc_dev(int i) { return c_lattice_sc_s[i]; }

enum {
  S_Q = 0,      // current rotation (x, y, z, w)
  S_R = 4,      // current rotation matrix (16-byte aligned)
  S_T = 14,     // current translation (16-byte aligned)
  S_PIV = 17,   // pivot
  S_GEO = 20,   // current geo_score
  S_STEPT = 21,
  S_STEPR = 22,
  S_STEPQ = 23,
  S_ERR = 24,
  S_X = 25,     // screen: max |coordinate| of the heavy atoms' FP32 torsioned frame
  S_N = 26
};

}  // namespace

struct search_args {
  batch_dev b;
  pocket_dev p;
  packed_grid pg;
  search_cfg c;
  flat_out f;
  item_out o;
  const double *pose_in;  // local_search mode: [n][8] q, t, geo; NULL in dock mode
  const double *ang_in;
  const double *conf_in;
  int *work;
  int n_lig;             // ligands of this launch (each: k restarts)
  const int *lig_index;  // bucket launches: launch ligand -> batch ligand (NULL: identity)
  double *hscr;          // global scratch: per resident warp 3 * (Nmax + nmax * mmax), then per CTA 14 * mmax
  int scr_warps;         // warp slots in the scratch
  int Nmax, nmax, mmax, dmax;
  int warp_doubles;
  int cta_doubles;       // CTA-shared ligand staging (after the palette)
  int o_tors, o_Mcur, o_Mvar, o_Rj, o_vb, o_vbest, o_vcur, o_cache, o_ang, o_sccur, o_state, o_ints;
  // FP32 screen (SCR): heavy frame, torsion-neighbour matrices + their error
  // constants, the 13 rigid maps (12 neighbours + current pose), the exact
  // candidate row, FP32 current samples, FP32 stage-t prefixes
  int o_t32, o_A32, o_vc32, o_crow;
  size_t scr_stride;     // doubles of global scratch per warp
};

// Offset (in doubles) of variant v's matrix for torsion u >= t(v) inside the
// triangular Mvar block: variants (t, +), (t, -) each hold m - t matrices.
__device__ __forceinline__ int mvar_off(int v, int u, int m) {
  const int t = v >> 1, s = v & 1;
  return 12 * (2 * (t * m - (t * (t - 1)) / 2) + s * (m - t) + (u - t));
}

// Matrices of torsions t..m-1 for the pose whose angles equal the current
// ones except torsion t (sin/cos st, ct); endpoints are carried from the
// base coordinates through the current matrices (u' < t) and the new ones
// (t <= u' < u): the per-atom composition of apply_torsions
// (transform.cpp:73-81).  Single lane.  out(u) = out + 12 * (u - t).
__device__ __noinline__ bool chain_mats(int t, double st, double ct, int m, const double *ep, const uint32_t *epm,
                                        const double *Mcur, const double *sccur, double *out) {
  #pragma unroll 1
  for (int u = t; u < m; ++u) {
    d3 ea = ld3(ep + 6 * u), eb = ld3(ep + 6 * u + 3);
    const uint32_t ma = epm[2 * u], mb = epm[2 * u + 1];
    #pragma unroll 1
    for (int w = 0; w < u; ++w) {
      const double *M = w < t ? Mcur + 12 * w : out + 12 * (w - t);
      if ((ma >> w) & 1u) ea = torsion_apply_a(M, ea);
      if ((mb >> w) & 1u) eb = torsion_apply_a(M, eb);
    }
    const double s = u == t ? st : sccur[2 * u];
    const double c = u == t ? ct : sccur[2 * u + 1];
    if (!torsion_setup(ea, eb, s, c, out + 12 * (u - t))) return false;
  }
  return true;
}

// Torsion-neighbour matrices of variants vbase + lane (search.cpp:168-176:
// (matrices of torsions u < ufrom are still valid: after a move of torsion
// ufrom only the matrices from ufrom on change)
// torsion t = v / 2 moved by +-step), warp-cooperative: all lanes walk the
// torsions u in the same order, so the endpoint masks (ep/epm: base
// coordinates and torsion masks of torsion u's bond atoms) and the branches
// on them are warp-uniform; lane v carries u's endpoints through Mcur
// (w < t) and through its own new matrices (t <= w < u), then builds matrix
// u once u >= t -- chain_mats' arithmetic, lanes in lockstep instead of
// diverging on different chain lengths.  Returns nonzero on a degenerate axis.
__device__ __noinline__ int chain_warp(int vbase, int ufrom, int m, const double *ep, const uint32_t *epm,
                                       const double *Mcur, const double *sccur, const double *cache, double *Mvar,
                                       int lane) {
  const int v = vbase + lane;
  const bool act = v < 2 * m;
  const int t = act ? (v >> 1) : m;
  double *out = Mvar + (act ? mvar_off(v, t, m) : 0);
  int bad = 0;
#ifdef VS_PHASE_PROF
  unsigned long long cs_acc = 0;
#endif
  #pragma unroll 1
  for (int u = max(vbase >> 1, ufrom); u < m; ++u) {
    d3 ea = ld3(ep + 6 * u), eb = ld3(ep + 6 * u + 3);
    const uint32_t ma = epm[2 * u], mb = epm[2 * u + 1];
    #pragma unroll 1
    for (uint32_t bb = (ma | mb) & ((1u << u) - 1u); bb; bb &= bb - 1u) {
      const int w = __ffs(bb) - 1;
      const double *M = w < t ? Mcur + 12 * w : out + 12 * (w - t);
      // both endpoints in one block (shared matrix loads, overlapping
      // chains), then keep the ones torsion w moves
      double r[12];
      ld12a(M, r);
      const d3 na = torsion_apply(r, ea), nb = torsion_apply(r, eb);
      if ((ma >> w) & 1u) ea = na;
      if ((mb >> w) & 1u) eb = nb;
    }
#ifdef VS_PHASE_PROF
    __syncwarp();
    const unsigned long long cs0 = clock64();
#endif
    if (u >= t) {
      const double s = u == t ? cache[2 * v] : sccur[2 * u];
      const double c = u == t ? cache[2 * v + 1] : sccur[2 * u + 1];
      if (!torsion_setup(ea, eb, s, c, out + 12 * (u - t))) bad = 1;
    }
#ifdef VS_PHASE_PROF
    __syncwarp();
    cs_acc += clock64() - cs0;
#endif
  }
#ifdef VS_PHASE_PROF
  if (lane == 0) atomicAdd(&g_phase[15], cs_acc);
#endif
  return bad;
}

// The same chains with two lanes per variant, one per axis endpoint
// (lane = 2 (v - vbase) + e, 16 variants per call): every carried transform
// is one 3-vector per lane instead of two, halving the chain's FP64
// instructions; the pair exchanges its endpoints by shuffles before the
// Rodrigues build, which both lanes evaluate and store (identical bits).
#ifndef VS_ROW_UNROLL
#define VS_ROW_UNROLL 2  // neighbour row sums: loads in flight ahead of the sequential adds (measured with
                         // VS_CENTROID_UNROLL 2: 1 -> 724 ms, 2 -> 696 ms, 4 -> 702 ms, 8 -> 726 ms search per step;
                         // code-layout sensitive: the hot loop sits at the 32 KB instruction-cache limit)
#endif
constexpr int kRowUnroll = VS_ROW_UNROLL;

#ifndef VS_CHAIN_SPLIT
#define VS_CHAIN_SPLIT 1
#endif
__device__ __noinline__ int chain_warp2(int vbase32, int ufrom, int m, const double *ep, const uint32_t *epm,
                                        const double *Mcur, const double *sccur, const double *cache, double *Mvar,
                                        int lane) {
  int bad = 0;
  const int e = lane & 1;
  #pragma unroll 1
  for (int vbase = vbase32; vbase < 2 * m && vbase < vbase32 + 32; vbase += 16) {
    const int v = vbase + (lane >> 1);
    const bool act = v < 2 * m;
    const int t = act ? (v >> 1) : m;
    double *out = Mvar + (act ? mvar_off(v, t, m) : 0);
    #pragma unroll 1
    for (int u = max(vbase >> 1, ufrom); u < m; ++u) {
      d3 x = ld3(ep + 6 * u + 3 * e);
      const uint32_t mk = epm[2 * u + e], mab = epm[2 * u] | epm[2 * u + 1];
      #pragma unroll 1
      for (uint32_t bb = mab & ((1u << u) - 1u); bb; bb &= bb - 1u) {
        const int w = __ffs(bb) - 1;
        const double *M = w < t ? Mcur + 12 * w : out + 12 * (w - t);
        double r[12];
        ld12a(M, r);
        const d3 nx = torsion_apply(r, x);
        if ((mk >> w) & 1u) x = nx;
      }
      const d3 y{__shfl_xor_sync(0xffffffffu, x.x, 1), __shfl_xor_sync(0xffffffffu, x.y, 1),
                 __shfl_xor_sync(0xffffffffu, x.z, 1)};
      if (u >= t) {
        const double s = u == t ? cache[2 * v] : sccur[2 * u];
        const double c = u == t ? cache[2 * v + 1] : sccur[2 * u + 1];
        // both lanes of the pair store the same bits
        if (!torsion_setup(e ? y : x, e ? x : y, s, c, out + 12 * (u - t))) bad = 1;
      }
      __syncwarp();  // the pair's new matrix is visible to both lanes
    }
  }
  return bad;
}

// Torsioned frame (search.cpp:115) of the hydrogens into the warp's global
// scratch `hx` (atom order; apply_torsions per atom, transform.cpp:73-81).
// The search keeps only heavy atoms in shared memory: hydrogens matter only
// for pivots and outputs.
__device__ __noinline__ void hydrogen_frame(double *hx, int N, const double *base, const uint32_t *tm,
                                            const uint8_t *heavy, const double *Mcur, uint32_t moved, int lane) {
  #pragma unroll 1
  for (int a = lane; a < N; a += 32) {
    if (heavy[a] || (moved != 0xffffffffu && !(tm[a] & moved))) continue;  // all ones: every hydrogen
    d3 x = ld3(base + 3 * a);
    #pragma unroll 1
    for (uint32_t bb = tm[a]; bb; bb &= bb - 1u) x = torsion_apply_a(Mcur + 12 * (__ffs(bb) - 1), x);
    st3(hx + 3 * a, x);
  }
}

// Stage-t prefix positions of the torsion items (search.cpp:168-176): pair p
// = (t, h in D_t) of the stored list gets h's base coordinates carried
// through the current matrices of torsions u < t (the part of its chain that
// is the same for (t,+) and (t,-) and for every step level), pairs from
// `pfrom` on.  Recomputed only when a torsion move changes Mcur.
__device__ __noinline__ void prefix_frame(double *pc, const uint32_t *tit, int pfrom, int npairs, const double *bh,
                                          const uint32_t *tmh, const double *Mcur, int lane) {
  #pragma unroll 1
  for (int p = pfrom + lane; p < npairs; p += 32) {
    const uint32_t e = tit[p];
    const int h = e & 255, t = (e >> 9) & 31;
    d3 x = ld3(bh + 3 * h);
    #pragma unroll 1
    for (uint32_t bb = tmh[h] & ((1u << t) - 1u); bb; bb &= bb - 1u)
      x = torsion_apply_a(Mcur + 12 * (__ffs(bb) - 1), x);
    st3(pc + 3 * p, x);
  }
}

// ---------------------------------------------------------------------------
// FP32 screen.  Every neighbour's geo_score is first
// bracketed in FP32 with a proven error bound; only the neighbours whose
// bracket reaches the decision threshold are evaluated exactly in FP64 (the
// reference's arithmetic, unchanged), so the adopted neighbour -- and every
// bit of the trajectory -- is the reference's.
//
// Error model (u = 2^-24; vectors in the 2-norm unless marked inf):
//  * rigid map l = A x + b (A = fl32(R / h), b = fl32((t - o) / h), x =
//    fl32(frame)), three FMAs per axis: |l~ - l| <= u (5.01 sqrt3 X / h +
//    4.01 |b|inf) per axis (X = |x|inf bound), padded to 5.1 / 4.1; the
//    reference's own FP64 rounding (<1e-13 cells) is covered by +1e-9;
//  * torsion chain y = R (x - p) + p in FP32 per applied matrix: the error
//    grows by sqrt3 u (7.94 |d|inf + 5.01 |p|inf) (padded to 8.7 / 5.75) and
//    is carried through rotations unamplified; the prefix's own rounding adds
//    sqrt3 u |x|inf; the rigid map then scales it by 1 / h;
//  * sample: trilinear interpolation is Lipschitz with sum-over-axes constant
//    G = 3 (vmax - vmin) per cell unit, so |f(l~) - f(l)| <= G dl; FP32
//    lerp rounding <= 7 u V (+ table rounding) = `eval`; in a cell whose 4^3
//    node neighbourhood is uniform (!NU) the value is exactly the constant;
//    within dl of a box face the -10 jump J is added;
//  * row: s~ = fl32(S) + sum (v~ - fl32(vcur)) over the moved atoms (the
//    others sample exactly as the current pose), FP32 summation error
//    <= (k + 2) u (|S| + sum |d|), per-item conversions <= 3 u V; the
//    reference's two FP64 sums differ from the real ones by < 1e-11.
// ---------------------------------------------------------------------------
constexpr float kU32 = 5.9604645e-8f;  // 2^-24
constexpr float kSqrt3 = 1.7320508f;

__device__ __forceinline__ float screen_sample(const screen_grid &sg, const float *tab, float lx, float ly, float lz,
                                               float dl, float &e) {
  constexpr float M = 12582912.0f;  // 1.5 * 2^23: fadd.rm gives M + floor(l) for |l| < 2^22
  const float tx = __fadd_rd(lx, M), ty = __fadd_rd(ly, M), tz = __fadd_rd(lz, M);
  const float flx = tx - M, fly = ty - M, flz = tz - M;
  const float fx = lx - flx, fy = ly - fly, fz = lz - flz;  // exact for l >= 0
  // linear cell index ix + dx (iy + dy iz), exact while M + index < 2^24;
  // out-of-box points are clamped into the array and overridden below
  const float fi = fmaf(flz, sg.fdxy, fmaf(fly, sg.fdx, tx));
  const uint32_t idx = min((uint32_t)(__float_as_int(fi) - 0x4B400000), sg.last);
  const uint32_t w = __ldg(sg.w + idx);
  const char *tb = reinterpret_cast<const char *>(tab);
  const float2 c0 = *reinterpret_cast<const float2 *>(tb + (w & 0xffu));
  const float2 c1 = *reinterpret_cast<const float2 *>(tb + ((w >> 8) & 0xffu));
  const float2 c2 = *reinterpret_cast<const float2 *>(tb + ((w >> 16) & 0xffu));
  const float2 c3 = *reinterpret_cast<const float2 *>(tb + ((w >> 24) & 0x7fu));
  const float X0 = fmaf(fx, c0.y, c0.x), X1 = fmaf(fx, c1.y, c1.x);
  const float X2 = fmaf(fx, c2.y, c2.x), X3 = fmaf(fx, c3.y, c3.x);
  const float Y0 = fmaf(fy, X1 - X0, X0), Y1 = fmaf(fy, X3 - X2, X2);
  float v = fmaf(fz, Y1 - Y0, Y0);
  // signed distance to the nearest node-box face (inf-norm, > 0 inside);
  // l - (dims - 1) is exact near the face (Sterbenz)
  const float lo = fminf(fminf(lx, ly), lz);
  const float hi = fmaxf(fmaxf(lx - sg.dx1, ly - sg.dy1), lz - sg.dz1);
  const float mg = fminf(lo, -hi);
  const float g = fmaf(sg.G, dl, sg.eval);
  float ee = (int)w < 0 ? g : sg.uni;
  ee = mg <= dl ? sg.J + g : ee;  // within dl of a face: either side
  const bool out = mg < -dl;      // outside for the reference too: exactly -10
  e = out ? 0.0f : ee;
  return out ? -10.0f : v;
}

// One FP32 rigid map slot (16 floats): A = R / h (9), b = (t - o) / h (3),
// the per-axis bound dl of a rigid item whose frame |x|inf <= X, |b|inf.
__device__ __forceinline__ void screen_slot(const double *R, const double *T, const grid_view &g, double inv_h,
                                            double X, float *out) {
  #pragma unroll 1
  for (int i = 0; i < 9; ++i) out[i] = (float)(R[i] * inv_h);
  out[9] = (float)((T[0] - g.ox) * inv_h);
  out[10] = (float)((T[1] - g.oy) * inv_h);
  out[11] = (float)((T[2] - g.oz) * inv_h);
  const float B = fmaxf(fmaxf(fabsf(out[9]), fabsf(out[10])), fabsf(out[11]));
  const float base = kU32 * 4.1f * B + 1e-9f;
  out[12] = fmaf(kU32 * 5.1f * kSqrt3 * (float)inv_h * 1.0001f, (float)X * 1.0001f, base);
  out[13] = base;  // torsion items add their own frame term
}

__device__ __forceinline__ void screen_map(const float *S, float x0, float x1, float x2, float &lx, float &ly,
                                           float &lz) {
  const float4 a0 = *reinterpret_cast<const float4 *>(S);
  const float4 a1 = *reinterpret_cast<const float4 *>(S + 4);
  const float4 a2 = *reinterpret_cast<const float4 *>(S + 8);
  lx = fmaf(a0.z, x2, fmaf(a0.y, x1, fmaf(a0.x, x0, a2.y)));
  ly = fmaf(a1.y, x2, fmaf(a1.x, x1, fmaf(a0.w, x0, a2.z)));
  lz = fmaf(a2.x, x2, fmaf(a1.w, x1, fmaf(a1.z, x0, a2.w)));
}

// The whole conformation of the current pose into `out` (3N, atom order):
// the torsioned frame `hx` (global scratch, every atom), then apply_rigid
// (transform.cpp:31) when `rigid`.
// hl != NULL (dock path outputs): only the heavy atoms, compact (heavy atom h
// at 3h, atom hl[h]) -- all that cluster_and_select and chem_score read; the
// best pose's hydrogens are rematerialised by the select (kernels.cu
// best_conformation).
__device__ __noinline__ void full_conformation(double *out, const double *S, int N, const double *hx, bool rigid,
                                               int lane, const uint32_t *hl = nullptr) {
  #pragma unroll 1
  for (int i = lane; i < N; i += 32) {
    const int a = hl ? (int)hl[i] : i;
    const d3 x = ld3(hx + 3 * a);
    st3(out + 3 * i, rigid ? rigid_col_rt(S + S_R, S + S_T, x, a) : x);
  }
}

// Pivot = centroid of apply_rigid(tors, T) (search.cpp:124): the warp writes
// the transformed conformation to `scratch`, then three lanes run the
// Eigen-order row sums (dmath.cuh centroid_row).  `rows`: the coordinates
// that can have changed since the last pivot (a translation along one axis
// leaves the other coordinates of every atom, hence their rows, bit-identical;
// row 2 is the long sequential sum, so x/y moves skip it).
#ifndef VS_PIVOT_ROWS
#define VS_PIVOT_ROWS 1
#endif
__device__ __forceinline__ void compute_pivot(double *scratch, double *S, int N, const double *hx, bool rigid,
                                              int lane, unsigned rows = 7u) {
  full_conformation(scratch, S, N, hx, rigid, lane);
  __syncwarp();
  if (lane < 3 && ((rows >> lane) & 1u)) S[S_PIV + lane] = centroid_row(scratch, N, lane);
  __syncwarp();
}

__device__ __forceinline__ float frame_max32(const float *t32, int n, int lane) {
  float x = 0.0f;
  #pragma unroll 1
  for (int i = lane; i < 3 * n; i += 32) x = fmaxf(x, fabsf(t32[i]));
  #pragma unroll
  for (int off = 16; off > 0; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, off));
  return x;
}

#ifndef VS_SEARCH_MINB
#define VS_SEARCH_MINB (16 / kWarps)  // A/B only: a higher count caps the registers (96 at 10: +9% search time)
#endif
#ifndef VS_SCREEN_MINB
#define VS_SCREEN_MINB 8
#endif
constexpr int kMaxWarpsSM = 24;  // warp slots per SM in the global scratch

template <int MODE, bool SCR>
__global__ void __launch_bounds__(32 * kWarps, SCR ? VS_SCREEN_MINB : VS_SEARCH_MINB) k_search(search_args A) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) float s_pair[32];  // screen pair table: 16 x (a, b - a)
  if (SCR && threadIdx.x < 32) s_pair[threadIdx.x] = A.p.scr.pair[threadIdx.x];
  // palette (CTA-wide): MODE 2 reads the 16 values; MODE 1 a table of code
  // pairs, entry i = (palette[i & 3], palette[i >> 2]), so two corners of a
  // cell come with one 128-bit load
  double *pal = sm;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < kPalDoubles)
    pal[threadIdx.x] = MODE == 0 ? 0.0
                       : MODE == 1 ? A.p.palette[(threadIdx.x & 1) ? ((threadIdx.x >> 1) >> 2) : ((threadIdx.x >> 1) & 3)]
                                   : (threadIdx.x < 16 ? A.p.palette[threadIdx.x] : 0.0);
  // CTA-shared staging of the current ligand (all warps of the CTA run its
  // restarts): heavy-atom base coordinates, torsion endpoints, masks, items
  double *s_bh = sm + kPalDoubles;        // 3 * nmax: base coordinates of heavy atom h
  double *s_ep = s_bh + 3 * A.nmax;       // 6 * mmax: base coordinates of torsion u's endpoints
  uint32_t *s_tmh = reinterpret_cast<uint32_t *>(s_ep + 6 * A.mmax);  // nmax: torsion mask | parity << 31
  uint32_t *s_dm = s_tmh + A.nmax;        // nmax: D_t membership of heavy atom h
  uint32_t *s_hl = s_dm + A.nmax;         // nmax: atom index of heavy atom h
  uint32_t *s_epm = s_hl + A.nmax;        // 2 * mmax: torsion masks of the endpoints
  int *s_doff = reinterpret_cast<int *>(s_epm + 2 * A.mmax);  // mmax
  int *s_dcnt = s_doff + A.mmax;          // mmax
  uint32_t *s_tit = reinterpret_cast<uint32_t *>(s_dcnt + A.mmax);  // dmax: (t, h in D_t) pairs, h | 2t << 8
  __shared__ int sh_lig, sh_r;
  double *W = sm + kPalDoubles + A.cta_doubles + (size_t)warp * A.warp_doubles;
#if VS_TORSH_SMEM
  double *torsh = W + A.o_tors;  // 3 * nmax: torsioned frame of the heavy atoms (search.cpp:115)
#endif
  // per-warp global scratch: the hydrogens' torsioned frame (3 * Nmax) and
  // the stage-t prefix positions of the torsion items (3 * nmax * mmax)
  double *hx = A.hscr + (size_t)(blockIdx.x * kWarps + warp) * A.scr_stride;
  double *pc = hx + 3 * A.Nmax;
  // per-CTA global slot (dock path): the start matrices of flatten's angles
  // and their sin/cos, computed once per ligand for all its restarts
  double *M0 = A.hscr + (size_t)A.scr_warps * A.scr_stride + (size_t)blockIdx.x * 14 * A.mmax;
  double *sc0 = M0 + 12 * A.mmax;
  VS_CHECK((int)(blockIdx.x * kWarps + warp) < A.scr_warps);
  double *Mcur = W + A.o_Mcur;
  double *Mvar = W + A.o_Mvar;
  float *t32 = reinterpret_cast<float *>(W + A.o_t32);
  float *A32 = reinterpret_cast<float *>(W + A.o_A32);
  float *vc32 = reinterpret_cast<float *>(W + A.o_vc32);
  int *crow = reinterpret_cast<int *>(W + A.o_crow);  // screen: rigid candidate rows
  const screen_grid &sg = A.p.scr;
  float Xf = 0.0f;  // screen: |frame|inf bound of the rigid items
  unsigned mgn = 1u;  // screen: ceil(2^32 / n), it / n == umulhi(it, mgn) for the rigid items
  double *Rj = W + A.o_Rj;       // 6 spin neighbours x kRow: R at 0, t at 10, q at 14 (16-byte aligned)
  double *Tj = Rj + 6 * kRow;    // 6 translation neighbours' t, stride 4
  double *vb = W + A.o_vb;
  double *vbest = W + A.o_vbest;
  double *vcur = W + A.o_vcur;
  double *cache = W + A.o_cache;
  double *cachelo = cache + 4 * A.mmax;
  double *ang = W + A.o_ang;
  double *sccur = W + A.o_sccur;
  double *sclo = sccur + 2 * A.mmax;
  double *S = W + A.o_state;
  int *cvalid = reinterpret_cast<int *>(W + A.o_ints);

  const batch_dev &b = A.b;
  const grid_view &g = A.p.g;
  const packed_grid &pg = A.pg;
  const bool ls_mode = A.pose_in != nullptr;
  const bool dock_path = !ls_mode && A.ang_in == nullptr;  // start angles = flatten's lattice angles
  const int k = ls_mode ? 1 : A.c.k;
  const int nmax = A.nmax;
  PH_DECL

  while (true) {  // one ligand per CTA pass
    __syncthreads();  // previous ligand finished by every warp
    PH(22)
    if (threadIdx.x == 0) {
      sh_lig = atomicAdd(A.work, 1);
      sh_r = 0;
    }
    __syncthreads();
    const int li = sh_lig;
    if (li >= A.n_lig) break;
    const int l = A.lig_index ? A.lig_index[li] : li;
    const lig_meta meta = b.meta[l];
    if (meta.status != VS_LIG_OK) {
      #pragma unroll 1
      for (int r = threadIdx.x; r < k; r += blockDim.x) A.o.status[l * k + r] = meta.status;
      continue;
    }
    const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
    if (SCR) mgn = n > 1 ? (unsigned)(0xffffffffu / (unsigned)n) + 1u : 1u;
    const int a0 = b.atom_off[l], t0 = b.tors_off[l];
    const double *base = b.xyz + 3 * (size_t)a0;
    const uint32_t *tm = b.atom_tmask + a0;
    const uint8_t *hv = b.heavy + a0;
    {
      const uint16_t *hl = b.heavy_list + a0;
      const uint16_t *ta = b.tors_a + t0, *tb = b.tors_b + t0;
      const uint32_t *titems = b.titems + 2 * b.ditem_base[l];
      #pragma unroll 1
      for (int h = threadIdx.x; h < n; h += blockDim.x) {
        const int a = hl[h];
        st3(s_bh + 3 * h, ld3(base + 3 * a));
        s_tmh[h] = tm[a] | ((uint32_t)(a & 1) << 31);
        s_dm[h] = b.heavy_dmask[a0 + h];
        s_hl[h] = (uint32_t)a;
      }
      #pragma unroll 1
      for (int u = threadIdx.x; u < m; u += blockDim.x) {
        const int ea = ta[u], eb = tb[u];
        st3(s_ep + 6 * u, ld3(base + 3 * ea));
        st3(s_ep + 6 * u + 3, ld3(base + 3 * eb));
        s_epm[2 * u] = tm[ea];
        s_epm[2 * u + 1] = tm[eb];
        s_doff[u] = b.d_off[t0 + u];
        s_dcnt[u] = b.d_count[t0 + u];
      }
      // the (t,+) half of k_setup's item list: (t,-) items pair with them
      #pragma unroll 1
      for (int u = threadIdx.x; u < m; u += blockDim.x) {
        const int off = b.d_off[t0 + u], cnt = b.d_count[t0 + u];
        #pragma unroll 1
        for (int i = 0; i < cnt; ++i) s_tit[off + i] = titems[2 * off + i];
      }
      if (dock_path) {
        #pragma unroll 1
        for (int u = threadIdx.x; u < m; u += blockDim.x) {
          const int li = A.f.idx[t0 + u];
          sc0[2 * u] = c_lattice_sc_dev(2 * li);
          sc0[2 * u + 1] = c_lattice_sc_dev(2 * li + 1);
        }
      }
    }
    __syncthreads();
    if (dock_path) {
      // flatten already rejected ligands whose axes degenerate at these angles
      if (threadIdx.x == 0 && m > 0) chain_mats(0, sc0[0], sc0[1], m, s_ep, s_epm, M0, sc0, M0);
      __syncthreads();
    }
    const int J = 12 + 2 * m;
    PH(23)

  while (true) {  // restarts of this ligand, one per warp at a time
    int r = 0;
    if (lane == 0) r = atomicAdd(&sh_r, 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= k) break;
    const int item = l * k + r;  // global item index of the outputs
    unsigned long long evals = 0;

    // ---- per-restart tables
    #pragma unroll 1
    for (int v = lane; v < 2 * m; v += 32) cvalid[v] = 0;
    if (A.ang_in) {  // local_search / initial_poses entry points: arbitrary angles
      #pragma unroll 1
      for (int u = lane; u < m; u += 32) {
        ang[u] = A.ang_in[t0 + u];
        sincos_dd_dev(ang[u], &sccur[2 * u], &sclo[2 * u]);
      }
    } else {
      #pragma unroll 1
      for (int u = lane; u < m; u += 32) {
        const int li = A.f.idx[t0 + u];
        ang[u] = li * kLatticeStep;  // angles_of, search.cpp:40
        sccur[2 * u] = c_lattice_sc_dev(2 * li);
        sccur[2 * u + 1] = c_lattice_sc_dev(2 * li + 1);
        sclo[2 * u] = c_lattice_lo_s[2 * li];
        sclo[2 * u + 1] = c_lattice_lo_s[2 * li + 1];
      }
    }
    if (lane == 0) S[S_ERR] = 0.0;
    __syncwarp();
    if (dock_path) {
      // start matrices from the CTA slot; the torsioned frame is flatten's
      // conformation (the same per-atom operations, bit for bit)
      #pragma unroll 1
      for (int i = lane; i < 12 * m; i += 32) Mcur[i] = M0[i];
      #pragma unroll 1
      for (int i = lane; i < 3 * N; i += 32) hx[i] = A.f.xyz[3 * (size_t)a0 + i];
#if VS_TORSH_SMEM
      if (!SCR) {
        #pragma unroll 1
        for (int h = lane; h < n; h += 32) st3(torsh + 3 * h, ld3(A.f.xyz + 3 * ((size_t)a0 + s_hl[h])));
      }
#endif
      if (SCR) {
        #pragma unroll 1
        for (int h = lane; h < n; h += 32) {
          const d3 x = ld3(A.f.xyz + 3 * ((size_t)a0 + s_hl[h]));
          t32[3 * h] = (float)x.x;
          t32[3 * h + 1] = (float)x.y;
          t32[3 * h + 2] = (float)x.z;
        }
      }
    } else {
      if (lane == 0 && m > 0 && !chain_mats(0, sccur[0], sccur[1], m, s_ep, s_epm, Mcur, sccur, Mcur))
        S[S_ERR] = 1.0;
      __syncwarp();
      if (S[S_ERR] != 0.0) {
        if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
        continue;
      }
      // torsioned frame (search.cpp:115)
      #pragma unroll 1
      for (int h = lane; h < n; h += 32) {
        d3 x = ld3(s_bh + 3 * h);
        #pragma unroll 1
        for (uint32_t bb = s_tmh[h] & 0x7fffffffu; bb; bb &= bb - 1u)
          x = torsion_apply_a(Mcur + 12 * (__ffs(bb) - 1), x);
#if VS_TORSH_SMEM
        if (!SCR) st3(torsh + 3 * h, x);
#endif
        if (SCR) {
          t32[3 * h] = (float)x.x;
          t32[3 * h + 1] = (float)x.y;
          t32[3 * h + 2] = (float)x.z;
        }
        st3(hx + 3 * s_hl[h], x);  // every atom's frame also in hx (pivots, outputs)
      }
      hydrogen_frame(hx, N, base, tm, hv, Mcur, 0xffffffffu, lane);
    }
    __syncwarp();
    prefix_frame(pc, s_tit, 0, meta.d_total, s_bh, s_tmh, Mcur, lane);
    __syncwarp();
    if (SCR) Xf = frame_max32(t32, n, lane);
    // initial_poses entry point: the flat centroid of these angles
    // (search.cpp:89-90) instead of flatten's
    if (!ls_mode && A.ang_in) {
      __syncwarp();
      compute_pivot(vb, S, N, hx, false, lane);
    }
    // ---- start pose: initial_poses (search.cpp:95-103) or the given one
    if (lane == 0) {
      quat q;
      double t[3];
      if (ls_mode) {
        const double *pi = A.pose_in + 8 * l;
        q = {pi[0], pi[1], pi[2], pi[3]};
        t[0] = pi[4];
        t[1] = pi[5];
        t[2] = pi[6];
      } else {
        const double *fq = A.c.fibq + 4 * r;
        q = {fq[0], fq[1], fq[2], fq[3]};
        const d3 rc = quat_rotate(q, A.ang_in ? ld3(S + S_PIV) : ld3(A.f.centroid + 3 * l));
        t[0] = A.p.center[0] - rc.x;
        t[1] = A.p.center[1] - rc.y;
        t[2] = A.p.center[2] - rc.z;
      }
      S[S_Q] = q.x;
      S[S_Q + 1] = q.y;
      S[S_Q + 2] = q.z;
      S[S_Q + 3] = q.w;
      S[S_T] = t[0];
      S[S_T + 1] = t[1];
      S[S_T + 2] = t[2];
      quat_matrix(q, S + S_R);
      S[S_STEPT] = A.c.step_t;
      S[S_STEPR] = A.c.step_r;
      S[S_STEPQ] = A.c.step_q;
    }
    __syncwarp();
    #pragma unroll 1
    for (int h = lane; h < n; h += 32) {
      const int a = s_hl[h];
      bool out;
      vcur[h] = field_value_fast<MODE>(g, pg, pal, rigid_col_rt(S + S_R, S + S_T, ld3(SCR ? hx + 3 * a : TORSH(h, a)), a),
                                       out);
      if (SCR) vc32[h] = (float)vcur[h];
    }
    __syncwarp();
    if (lane == 0) {
      if (ls_mode) {
        S[S_GEO] = A.pose_in[8 * l + 7];
      } else {
        double acc = 0.0;
        #pragma unroll 1
        for (int h = 0; h < n; ++h) acc += vcur[h];
        S[S_GEO] = acc;
      }
    }
    if (!ls_mode) evals += (unsigned long long)n;
    // pivot of the start pose: centroid of its conformation (search.cpp:124)
    if (ls_mode) {
      if (lane < 3) S[S_PIV + lane] = centroid_row(A.conf_in + 3 * (size_t)a0, N, lane);
      __syncwarp();
    } else {
      compute_pivot(vb, S, N, hx, true, lane);
    }

    PH(0)
    // ---- local_search (search.cpp:121-191)
    int level = 0, n_iter = 0, n_adopt = 0;
    bool failed = false, mvar_valid = false, moved = false;
    int chain_from = 0;  // first torsion whose neighbour matrices are stale
    for (int iter = 0; iter < A.c.max_iter && S[S_STEPT] >= A.c.min_t; ++iter) {
      const double step_t = S[S_STEPT], step_q = S[S_STEPQ];
      // rigid neighbour transforms (lanes 0-11) and, when stale, the
      // torsion-neighbour matrices (lanes 12..; one lane per neighbour)
#ifdef VS_PHASE_PROF
      const bool ph_rebuild = !mvar_valid;
#endif
#ifdef VS_PHASE_PROF
      unsigned int pr_sc = 0, pr_ch = 0, pr_rg = 0;
      unsigned long long pr0 = clock64();
#endif
      // rigid neighbour transforms (lanes 0-11)
      if (lane < 12) {
        if (lane < 6) {  // translations (search.cpp:152-158): rotation stays S_R
          const int axis = lane >> 1;
          const double sign = (lane & 1) ? -1.0 : 1.0;
          double *X = Tj + 4 * lane;
          for (int q = 0; q < 3; ++q) X[q] = S[S_T + q];
          X[axis] = S[S_T + axis] + sign * step_t;
        } else {  // rotations about the pivot (search.cpp:159-167)
          double *X = Rj + kRow * (lane - 6);
          // tables end at n_levels (<= 4096): deeper levels have step 0, equal to the last entry
          const double *sq = A.c.spin + 4 * (6 * min(level, A.c.n_levels - 1) + (lane - 6));
          const quat spin{sq[0], sq[1], sq[2], sq[3]};
          const d3 piv = ld3(S + S_PIV);
          const d3 spin_t = sub3(piv, quat_rotate(spin, piv));
          const quat cur{S[S_Q], S[S_Q + 1], S[S_Q + 2], S[S_Q + 3]};
          const quat qn = quat_normalized(quat_mul(spin, cur));  // compose, transform.cpp:18-19
          const d3 tt = add3(quat_rotate(spin, ld3(S + S_T)), spin_t);
          quat_matrix(qn, X);
          X[10] = tt.x;
          X[11] = tt.y;
          X[12] = tt.z;
          X[14] = qn.x;
          X[15] = qn.y;
          X[16] = qn.z;
          X[17] = qn.w;
        }
      }
      if (SCR) {
        __syncwarp();
        // FP32 maps of the 12 rigid neighbours (slots 0-11) and the current
        // pose (slot 12, torsion neighbours)
        if (lane < 13) {
          const double *R = (lane < 6 || lane == 12) ? S + S_R : Rj + kRow * (lane - 6);
          const double *T = lane < 6 ? Tj + 4 * lane : (lane == 12 ? S + S_T : R + 10);
          screen_slot(R, T, g, pg.inv_h, Xf, A32 + 16 * lane);
        }
      }
#ifdef VS_PHASE_PROF
      __syncwarp();
      pr_rg = (unsigned int)(clock64() - pr0);
      pr0 = clock64();
#endif
      // torsion-neighbour matrices when stale (after a torsion move or a
      // step halving): sin/cos of the moved angles, then the chains
      if (!mvar_valid) {
        #pragma unroll 1
        for (int vb0 = 0; vb0 < 2 * m; vb0 += 32) {
          const int v = vb0 + lane;
          if (v < 2 * m && !cvalid[v]) {
            // sin/cos of ang[t] +- step_q from the current double-double
            // values and the level's step table (vs_crtrig.h sincos_shift)
            const int t = v >> 1;
            const double *st = A.c.stepsc + 4 * min(level, A.c.n_levels - 1);
            const bool neg = v & 1;
            const vs_crtrig::dd sd{neg ? -st[0] : st[0], neg ? -st[1] : st[1]}, cd{st[2], st[3]};
            double an;
            vs_crtrig::dd sn, cn;
            if (!vs_crtrig::sincos_shift(ang[t], vs_crtrig::dd{sccur[2 * t], sclo[2 * t]},
                                         vs_crtrig::dd{sccur[2 * t + 1], sclo[2 * t + 1]}, neg ? -step_q : step_q, sd,
                                         cd, &an, &sn, &cn)) {
              sincos_dd_dev(an, &cache[2 * v], &cachelo[2 * v]);
            } else {
              cache[2 * v] = sn.hi;
              cache[2 * v + 1] = cn.hi;
              cachelo[2 * v] = sn.lo;
              cachelo[2 * v + 1] = cn.lo;
            }
            cvalid[v] = 1;
          }
          __syncwarp();
#ifdef VS_PHASE_PROF
          pr_sc += (unsigned int)(clock64() - pr0);
          pr0 = clock64();
#endif
#if VS_CHAIN_SPLIT
          if (chain_warp2(vb0, chain_from, m, s_ep, s_epm, Mcur, sccur, cache, Mvar, lane)) S[S_ERR] = 1.0;
#else
          if (chain_warp(vb0, chain_from, m, s_ep, s_epm, Mcur, sccur, cache, Mvar, lane)) S[S_ERR] = 1.0;
#endif
#ifdef VS_PHASE_PROF
          __syncwarp();
          pr_ch += (unsigned int)(clock64() - pr0);
          pr0 = clock64();
#endif
        }
      }
#ifdef VS_PHASE_PROF
      if (ph_rebuild) {
        ph_acc[12] += pr_sc;
        ph_acc[13] += pr_ch;
        ph_acc[14] += pr_rg;
      }
#endif
      mvar_valid = true;
      __syncwarp();
      PH(ph_rebuild ? 9 : 1)
#ifdef VS_PHASE_PROF
      ph_acc[10] += ph_rebuild ? 1 : 0;
      ph_acc[11] += 1;
#endif
      if (S[S_ERR] != 0.0) {
        failed = true;
        break;
      }
      // neighbour groups: rigid first, then torsion neighbours in order
      double bv = S[S_GEO];
      int bj = -1;
      int tg = 0;  // next torsion to schedule
      const float S32 = (float)bv, aS = fabsf(S32);
      for (int grp = 0; grp == 0 || tg < m; ++grp) {
        int j0, jn, tlo = 0, thi = 0, items;
        if (grp == 0) {
          j0 = 0;
          jn = 12;
          items = 12 * n;
        } else {
          tlo = tg;
          thi = min(m, tlo + kGroup / 2);
          tg = thi;
          j0 = 12 + 2 * tlo;
          jn = 2 * (thi - tlo);
          items = 2 * (s_doff[thi - 1] + s_dcnt[thi - 1] - s_doff[tlo]);
        }
        const int *rmap = nullptr;  // screen: compact row ci -> rigid neighbour j
        if constexpr (SCR) {
          if (grp == 0) {
            // ---- FP32 screen of the 12 rigid neighbours: per item (v~ -
            // fl32(vcur), bound), then a proven bracket per row; only rows
            // whose bracket reaches max(current score, best lower bound) are
            // sampled exactly below (search.cpp:138 is decided in FP64)
            float2 *vs2 = reinterpret_cast<float2 *>(vb);
            #pragma unroll 1
            for (int it = lane; it < items; it += 32) {
              const int j = n == 1 ? it : (int)__umulhi((unsigned)it, mgn), h = it - j * n;
              const float *Sj = A32 + 16 * j;
              float lx, ly, lz, e;
              screen_map(Sj, t32[3 * h], t32[3 * h + 1], t32[3 * h + 2], lx, ly, lz);
              const float val = screen_sample(sg, s_pair, lx, ly, lz, Sj[12], e);
              vs2[it] = make_float2(val - vc32[h], e);
            }
            __syncwarp();
            PH(2)
            float ub = -__int_as_float(0x7f800000), lb = ub;
            if (lane < 12) {
              float sd = 0.0f, sa = 0.0f, se = 0.0f;
              #pragma unroll 4
              for (int i = 0; i < n; ++i) {
                const float2 q = vs2[lane * n + i];
                sd += q.x;
                sa += fabsf(q.x);
                se += q.y;
              }
              const float st = S32 + sd;
              const float E = fmaf(kU32, fmaf((float)(n + 2), aS + sa, sg.v3 * (float)n), se + 1e-9f) * 1.001f;
              ub = __fadd_ru(st, E);
              lb = __fadd_rd(st, -E);
              if (isnan(ub) || isnan(lb)) {  // non-finite inputs: sample exactly (NaN is never adopted)
                ub = __int_as_float(0x7f800000);
                lb = -ub;
              }
            }
            float gl = lb;
            #pragma unroll
            for (int off = 16; off > 0; off >>= 1) gl = fmaxf(gl, __shfl_xor_sync(0xffffffffu, gl, off));
            const unsigned cand = __ballot_sync(0xffffffffu, lane < 12 && (double)ub >= fmax(bv, (double)gl));
#ifdef VS_PHASE_PROF
            ph_acc[16] += __popc(cand);
            ph_acc[17] += 12;
#endif
            if (!cand) {
              PH(4)
              continue;  // no rigid neighbour can beat the current pose or another's lower bound
            }
            if ((cand >> lane) & 1u) crow[__popc(cand & ((1u << lane) - 1u))] = lane;
            __syncwarp();
            jn = __popc(cand);
            items = jn * n;
            rmap = crow;
          }
        }
        // Rigid and torsion neighbours run in separate compact loops, one
        // sample in flight per lane: the search is instruction-fetch bound
        // when warps at different phases share an SM (measured: two samples
        // per lane, even without an intervening store, tripled the
        // no-instruction stalls), so the hot code is kept small.
        // One sample loop for both kinds of group (the hot code must stay
        // small: the search is instruction-fetch bound when warps at
        // different phases share an SM).  Rigid item it = (transform j, heavy
        // atom h), walked incrementally; torsion item it = (t, h) pair it / 2
        // of the stored list with sign it & 1, its chain from the base
        // coordinates through the current / the variant's matrices.
        {
          const bool rig = grp == 0;
          const uint32_t *ti = s_tit + s_doff[tlo];
          const double *pcg = pc + 3 * s_doff[tlo];
          int rj = 0, rh = lane;
          if (rig && n > 0) {  // (n == 0: a hydrogen-only ligand docked with k == 1 has no items)
            #pragma unroll 1
            while (rh >= n) {
              rh -= n;
              ++rj;
            }
          }
          #pragma unroll 1
          for (int it = lane; it < items; it += 32) {
            int row, h, col;
            const double *R, *T;
            d3 x;
            if (rig) {
              h = rh;
              row = rj;
              col = s_hl[h];
              const int jr = rmap ? rmap[rj] : rj;
              R = jr < 6 ? S + S_R : Rj + kRow * (jr - 6);
              T = jr < 6 ? Tj + 4 * jr : R + 10;
              x = ld3(SCR ? hx + 3 * col : TORSH(h, col));
              rh += 32;
              #pragma unroll 1
              while (rh >= n) {
                rh -= n;
                ++rj;
              }
            } else {
              VS_CHECK(s_doff[tlo] + (it >> 1) < A.dmax);
              const uint32_t e = ti[it >> 1];
              const int v = ((e >> 8) & 63) | (it & 1), t = v >> 1;
              h = e & 255;
              x = ld3(pcg + 3 * (it >> 1));  // stage-t prefix (prefix_frame)
              const uint32_t mask = s_tmh[h];
              col = (int)(mask >> 31);
              const double *Mv = Mvar + mvar_off(v, t, m) - 12 * t;  // matrix u >= t at Mv + 12u
              VS_CHECK(t < m && mvar_off(v, m - 1, m) + 12 <= 12 * A.mmax * (A.mmax + 1) && h < n);
              #pragma unroll 1
              for (uint32_t bb = (mask & 0x7fffffffu) >> t << t; bb; bb &= bb - 1u)
                x = torsion_apply_a(Mv + 12 * (__ffs(bb) - 1), x);
              row = v - 2 * tlo;
              R = S + S_R;
              T = S + S_T;
            }
            bool out;
            VS_CHECK(row >= 0 && row < kGroup && h >= 0 && h < nmax);
            vb[row * nmax + h] = field_value_fast<MODE>(g, pg, pal, rigid_col_rt(R, T, x, col), out);
          }
        }
#if !VS_ROW_SELECT
        if (grp != 0) {
          // heavy atoms outside D_t sample exactly as in the current pose:
          // complete the torsion rows with the current values
          #pragma unroll 1
          for (int rr = 0; rr < jn; ++rr) {
            const int t = tlo + (rr >> 1);
            #pragma unroll 1
            for (int h = lane; h < n; h += 32)
              if (!((s_dm[h] >> t) & 1u)) vb[rr * nmax + h] = vcur[h];
          }
        }
#endif
        __syncwarp();
        PH(grp == 0 ? 2 : 3)
        // geo_score of each neighbour in the group (grid.cpp:97-101)
        double gacc = 0.0;
        if (lane < jn) {
          const double *row = vb + lane * nmax;
          double acc = 0.0;
#if VS_ROW_SELECT
          if (grp != 0) {
            // heavy atoms outside D_t sample exactly as in the current pose:
            // their values come from vcur (the row holds only D_t's samples)
            const uint32_t tb = 1u << (tlo + (lane >> 1));
            #pragma unroll kRowUnroll
            for (int h = 0; h < n; ++h) acc += (s_dm[h] & tb) ? row[h] : vcur[h];
          } else
#endif
          {
            #pragma unroll kRowUnroll
            for (int h = 0; h < n; ++h) acc += row[h];
          }
          gacc = acc;
        }
        // first strict maximum of the group, then against the running best
        // a NaN score is never adopted (score > best is false, search.cpp:138):
        // map it to -inf so every lane's reduction agrees
        double gv = (lane < jn && !isnan(gacc)) ? gacc : -__longlong_as_double(0x7ff0000000000000LL);
        int gj = lane < jn ? lane : 0x7fffffff;
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, gv, off);
          const int oj = __shfl_xor_sync(0xffffffffu, gj, off);
          if (ov > gv || (ov == gv && oj < gj)) {
            gv = ov;
            gj = oj;
          }
        }
        if (gv > bv) {  // search.cpp:138: strictly better than everything before
          bv = gv;
          bj = j0 + (rmap ? rmap[gj] : gj);
          const double *row = vb + gj * nmax;
#if VS_ROW_SELECT
          const uint32_t tb = grp != 0 ? 1u << (tlo + (gj >> 1)) : 0xffffffffu;
          #pragma unroll 1
          for (int h = lane; h < n; h += 32) vbest[h] = (grp == 0 || (s_dm[h] & tb)) ? row[h] : vcur[h];
#else
          #pragma unroll 1
          for (int h = lane; h < n; h += 32) vbest[h] = row[h];
#endif
        }
        __syncwarp();
        PH(4)
      }
      evals += (unsigned long long)n * J;
      ++n_iter;
      if (bj >= 0) {
        ++n_adopt;
        moved = true;
        if (bj < 6) {
          if (lane < 3) S[S_T + lane] = Tj[4 * bj + lane];
        } else if (bj < 12) {
          const double *X = Rj + kRow * (bj - 6);
          if (lane < 9) S[S_R + lane] = X[lane];
          else if (lane < 12) S[S_T + lane - 9] = X[lane + 1];
          else if (lane < 16) S[S_Q + lane - 12] = X[lane + 2];
        } else {
          const int v = bj - 12, t = v >> 1;
          const double sign = (v & 1) ? -1.0 : 1.0;
          #pragma unroll 1
          for (int i = lane; i < 12 * (m - t); i += 32) Mcur[12 * t + i] = Mvar[mvar_off(v, t, m) + i];
          if (lane == 0) {
            ang[t] = ang[t] + sign * step_q;
            sccur[2 * t] = cache[2 * v];
            sccur[2 * t + 1] = cache[2 * v + 1];
            sclo[2 * t] = cachelo[2 * v];
            sclo[2 * t + 1] = cachelo[2 * v + 1];
          }
          if (lane < 2) cvalid[2 * t + lane] = 0;
          mvar_valid = false;
          chain_from = t;
          __syncwarp();
          // only atoms whose coordinates depend on torsion t move: heavy
          // atoms of D_t continue from their cached stage-t prefixes through
          // the new matrices u >= t; hydrogens moved by t or by a torsion
          // whose axis depends on t are re-torsioned from base
          uint32_t dep = 1u << t;
          #pragma unroll 1
          for (int u = t + 1; u < m; ++u)
            if ((s_epm[2 * u] | s_epm[2 * u + 1]) & dep) dep |= 1u << u;
          #pragma unroll 1
          for (int i = lane; i < s_dcnt[t]; i += 32) {
            const int p = s_doff[t] + i;
            const int h = s_tit[p] & 255;
            d3 x = ld3(pc + 3 * p);
            #pragma unroll 1
            for (uint32_t bb = (s_tmh[h] & 0x7fffffffu) >> t << t; bb; bb &= bb - 1u)
              x = torsion_apply_a(Mcur + 12 * (__ffs(bb) - 1), x);
#if VS_TORSH_SMEM
            if (!SCR) st3(torsh + 3 * h, x);
#endif
            if (SCR) {
              t32[3 * h] = (float)x.x;
              t32[3 * h + 1] = (float)x.y;
              t32[3 * h + 2] = (float)x.z;
            }
            st3(hx + 3 * s_hl[h], x);
          }
          PH(19)
          hydrogen_frame(hx, N, base, tm, hv, Mcur, dep, lane);
          PH(20)
          prefix_frame(pc, s_tit, s_doff[t] + s_dcnt[t], meta.d_total, s_bh, s_tmh, Mcur, lane);
          PH(21)
          if (SCR) {
            __syncwarp();
            Xf = frame_max32(t32, n, lane);
          }
        }
        #pragma unroll 1
        for (int h = lane; h < n; h += 32) {
          vcur[h] = vbest[h];
          if (SCR) vc32[h] = (float)vbest[h];
        }
        if (lane == 0) S[S_GEO] = bv;
        __syncwarp();
        // new pivot = centroid of the adopted conformation (vb is free here)
        compute_pivot(vb, S, N, hx, true, lane, VS_PIVOT_ROWS && bj < 6 ? 1u << (bj >> 1) : 7u);
        PH(bj < 12 ? 5 : 6)
      } else {
        if (lane == 0) {
          S[S_STEPT] = S[S_STEPT] * 0.5;
          S[S_STEPR] = S[S_STEPR] * 0.5;
          S[S_STEPQ] = S[S_STEPQ] * 0.5;
        }
        #pragma unroll 1
        for (int v = lane; v < 2 * m; v += 32) cvalid[v] = 0;
        mvar_valid = false;
        chain_from = 0;
        ++level;
        PH(7)
      }
      __syncwarp();
    }
    if (failed) {
      if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
      continue;
    }
    // ---- outputs: the pose's conformation = apply_rigid(tors, T); in
    // local_search mode an unmoved pose returns its input conformation.
    const size_t ck = 3 * ((size_t)a0 * k + (size_t)r * N);
    if (ls_mode && !moved) {
      #pragma unroll 1
      for (int i = lane; i < 3 * N; i += 32) A.o.conf[ck + i] = A.conf_in[3 * (size_t)a0 + i];
    } else {
      full_conformation(A.o.conf + ck, S, A.o.heavy_conf ? n : N, hx, true, lane, A.o.heavy_conf ? s_hl : nullptr);
    }
    const size_t tk = (size_t)t0 * k + (size_t)r * m;
    #pragma unroll 1
    for (int u = lane; u < m; u += 32) A.o.ang[tk + u] = ang[u];
    if (lane < 4)
      A.o.T[7 * (size_t)item + lane] = S[S_Q + lane];
    else if (lane < 7)
      A.o.T[7 * (size_t)item + lane] = S[S_T + lane - 4];
    if (lane == 0) {
      A.o.geo[item] = S[S_GEO];
      A.o.evals[item] = evals;
      A.o.status[item] = VS_LIG_OK;
      if (A.o.iters) A.o.iters[item] = n_iter;
      if (A.o.adopts) A.o.adopts[item] = n_adopt;
    }
    __syncwarp();
    PH(8)
  }  // restarts
  }  // ligands
  PH_FLUSH
}

namespace {

struct Layout {
  int o_tors, o_Mcur, o_Mvar, o_Rj, o_vb, o_vbest, o_vcur, o_cache, o_ang, o_sccur, o_state, o_ints, total;
  int o_t32, o_A32, o_vc32, o_crow;
  int cta;  // CTA-shared ligand staging, doubles
};

Layout layout(int Nm, int nm, int mm, int dm, bool scr) {
  Layout L{};
  L.cta = 3 * nm + 6 * mm + (3 * nm + 4 * mm + dm + 1) / 2 + 1;
  L.cta = (L.cta + 1) & ~1;
  int o = 0;
  auto take = [&](int n) {
    const int at = o;
    o += (n + 1) & ~1;  // keep 16-byte alignment
    return at;
  };
  L.o_tors = take(VS_TORSH_SMEM && !scr ? 3 * nm : 0);
  L.o_Mcur = take(12 * mm);
  L.o_Mvar = take(12 * mm * (mm + 1));
  L.o_Rj = take(kRow * 6 + 4 * 6);
  L.o_vb = take(kGroup * nm > 3 * Nm ? kGroup * nm : 3 * Nm);  // also the pivot scratch / screen items (float2)
  L.o_vbest = take(nm);
  L.o_vcur = take(nm);
  L.o_cache = take(8 * mm);  // sin/cos of the 2m variant angles: hi parts, then lo parts
  L.o_ang = take(mm);
  L.o_sccur = take(4 * mm);  // sin/cos of the current angles: hi parts, then lo parts
  L.o_state = take(S_N);
  L.o_ints = take((2 * mm + 1) / 2 + 1);
  if (scr) {
    L.o_t32 = take((3 * nm + 1) / 2);  // FP32 heavy-atom frame
    L.o_A32 = take(13 * 8);            // 13 FP32 rigid maps x 16 floats
    L.o_vc32 = take((nm + 1) / 2);     // FP32 current samples
    L.o_crow = take(6);                // candidate rows (12 ints)
  }
  L.total = o;
  return L;
}

// Global scratch per warp, in doubles: hydrogen frame (3 Nmax) and stage-t
// prefixes (3 nmax mmax), 16-byte aligned.
size_t scr_stride(int Nm, int nm, int mm) { return (3 * (size_t)Nm + 3 * (size_t)nm * mm + 1) & ~(size_t)1; }

bool use_screen(const search_args &A) { return A.pg.mode == 1 && A.p.scr.w != nullptr; }

cudaError_t run_search(search_args &A, int num_sms, cudaStream_t s, int *launches) {
  const bool scr = use_screen(A);
  const Layout L = layout(A.Nmax, A.nmax, A.mmax, A.dmax, scr);
  A.cta_doubles = L.cta;
  A.o_tors = L.o_tors;
  A.o_Mcur = L.o_Mcur;
  A.o_Mvar = L.o_Mvar;
  A.o_Rj = L.o_Rj;
  A.o_vb = L.o_vb;
  A.o_vbest = L.o_vbest;
  A.o_vcur = L.o_vcur;
  A.o_cache = L.o_cache;
  A.o_ang = L.o_ang;
  A.o_sccur = L.o_sccur;
  A.o_state = L.o_state;
  A.o_ints = L.o_ints;
  A.o_t32 = L.o_t32;
  A.o_A32 = L.o_A32;
  A.o_vc32 = L.o_vc32;
  A.o_crow = L.o_crow;
  A.warp_doubles = L.total;
  A.scr_stride = scr_stride(A.Nmax, A.nmax, A.mmax);
  const int o = L.total;
  const size_t smem = (size_t)(kPalDoubles + L.cta + o * kWarps) * sizeof(double);
  if (smem > 227 * 1024 - 256) return cudaErrorInvalidValue;
  const void *fn = scr ? (const void *)k_search<1, true>
                       : (A.pg.mode == 1 ? (const void *)k_search<1, false>
                                         : (A.pg.mode == 2 ? (const void *)k_search<2, false>
                                                           : (const void *)k_search<0, false>));
  std::lock_guard<std::mutex> lock(launch_mutex());  // attribute + launch, atomically w.r.t. other workers
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kWarps, smem);
  if (per_sm < 1) per_sm = 1;
  // the global scratch holds kMaxWarpsSM warps per SM (search_scratch_bytes)
  if (per_sm > kMaxWarpsSM / kWarps) per_sm = kMaxWarpsSM / kWarps;
#ifdef VS_PROF_CTAS_PER_SM
  per_sm = VS_PROF_CTAS_PER_SM;  // development: phase timing without co-resident warps
#endif
  if (const char *cap = std::getenv("VS_SEARCH_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(cap)));
  int blocks = num_sms * per_sm;
  if (blocks > A.n_lig) blocks = A.n_lig;
  if (blocks < 1) blocks = 1;
  if (std::getenv("VSDOCK_DEBUG"))
    std::fprintf(stderr, "k_search%s: %d ligands, N<=%d n<=%d m<=%d d<=%d, smem %zu B/CTA, %d CTAs/SM, %d CTAs\n",
                 scr ? " (screen)" : "", A.n_lig, A.Nmax, A.nmax, A.mmax, A.dmax, smem, per_sm, blocks);
  if (scr)
    k_search<1, true><<<blocks, 32 * kWarps, smem, s>>>(A);
  else if (A.pg.mode == 1)
    k_search<1, false><<<blocks, 32 * kWarps, smem, s>>>(A);
  else if (A.pg.mode == 2)
    k_search<2, false><<<blocks, 32 * kWarps, smem, s>>>(A);
  else
    k_search<0, false><<<blocks, 32 * kWarps, smem, s>>>(A);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

void set_lattice_table_search(const double *sc72, const double *lo72) {
  cudaMemcpyToSymbol(c_lattice_sc_s, sc72, sizeof(double) * 72);
  cudaMemcpyToSymbol(c_lattice_lo_s, lo72, sizeof(double) * 72);
}

#ifdef VS_PHASE_PROF
extern "C" int vs_debug_phase_read(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(g_phase, z, sizeof z);
  }
  return 0;
}
#endif

// Global scratch of the search: per resident warp slot (kMaxWarpsSM per SM)
// scr_stride doubles, then a 14 mmax-double slot per CTA.
size_t search_scratch_bytes(int nmax_atoms, int nmax_heavy, int mmax, int num_sms) {
  const int N = nmax_atoms > 0 ? nmax_atoms : 1, n = nmax_heavy > 0 ? nmax_heavy : 1, m = mmax > 0 ? mmax : 1;
  const size_t warps = (size_t)num_sms * kMaxWarpsSM;
  return (warps * scr_stride(N, n, m) + warps * 14 * (size_t)m) * sizeof(double);
}

int search_warps_per_cta() { return kWarps; }

size_t search_smem_bytes(int N, int n, int m, int dtot, bool screen) {
  const Layout L = layout(N > 0 ? N : 1, n > 0 ? n : 1, m > 0 ? m : 1, dtot > 0 ? dtot : 1, screen);
  return (size_t)(kPalDoubles + L.cta + L.total * kWarps) * sizeof(double) + (screen ? 128 : 0);
}

cudaError_t launch_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const flat_out &f,
                          const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                          int num_sms, cudaStream_t s, int *launches, void *args_buf, const int *lig_index,
                          int n_lig, int dmax) {
  search_args A{};
  A.hscr = static_cast<double *>(args_buf);
  A.scr_warps = num_sms * kMaxWarpsSM;
  A.b = b;
  A.p = p;
  A.pg = p.packed;
  A.c = c;
  A.f = f;
  A.o = o;
  A.work = work_counter;
  A.lig_index = lig_index;
  A.n_lig = lig_index ? n_lig : b.n_lig;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  A.dmax = dmax > 0 ? dmax : A.nmax * A.mmax;
  if (A.n_lig == 0) return cudaSuccess;
  return run_search(A, num_sms, s, launches);
}

cudaError_t launch_initial_poses(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *angles,
                                 const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                                 int num_sms, cudaStream_t s, void *args_buf) {
  search_args A{};
  A.hscr = static_cast<double *>(args_buf);
  A.scr_warps = num_sms * kMaxWarpsSM;
  A.b = b;
  A.p = p;
  A.pg = p.packed;
  A.c = c;
  A.c.max_iter = 0;  // poses only: no local_search iteration
  A.o = o;
  A.ang_in = angles;
  A.work = work_counter;
  A.n_lig = b.n_lig;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  A.dmax = A.nmax * A.mmax;  // upper bound of sum_t |D_t|
  if (A.n_lig == 0) return cudaSuccess;
  return run_search(A, num_sms, s, nullptr);
}

cudaError_t launch_local_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *pose_in,
                                const double *ang_in, const double *conf_in, const item_out &o, int *work_counter,
                                int nmax_atoms, int nmax_heavy, int mmax, int num_sms, cudaStream_t s,
                                void *args_buf) {
  search_args A{};
  A.hscr = static_cast<double *>(args_buf);
  A.scr_warps = num_sms * kMaxWarpsSM;
  A.b = b;
  A.p = p;
  A.pg = p.packed;
  A.c = c;
  A.o = o;
  A.pose_in = pose_in;
  A.ang_in = ang_in;
  A.conf_in = conf_in;
  A.work = work_counter;
  A.n_lig = b.n_lig;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  A.dmax = A.nmax * A.mmax;  // upper bound of sum_t |D_t|
  if (A.n_lig == 0) return cudaSuccess;
  return run_search(A, num_sms, s, nullptr);
}

void preload_kernels_search() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_search<0, false>);
  cudaFuncGetAttributes(&a, k_search<1, false>);
  cudaFuncGetAttributes(&a, k_search<2, false>);
  cudaFuncGetAttributes(&a, k_search<1, true>);
}

}  // namespace vsd

