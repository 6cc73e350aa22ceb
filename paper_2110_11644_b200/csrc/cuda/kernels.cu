// sm_100a kernels of the batched dock-and-score path.
//
//   k_setup        per ligand: validation, heavy-atom list, right-set masks,
//                  torsion dependency closures D_t (thread per ligand)
//   k_flatten_dep  flatten (search.cpp:27-69): CTA per ligand, 8 lanes per
//                  10-degree candidate, candidate-dependent atoms only, exact
//                  sequential sums for near ties (k_flatten: legacy layout,
//                  used for ligands too large for its shared memory)
//   k_search       initial_poses + local_search (search.cpp:84-193): one
//                  warp per (ligand, restart), persistent, atomic work queue
//   k_select       cluster_and_select + chem_score + argmax
//                  (search.cpp:195-275, chem.cpp:31-46): CTA per ligand
//   k_field/k_geo/k_chem/k_build_pocket  the sub-APIs (grid.cpp, chem.cpp)
//
// Everything is FP64 in the reference's evaluation order (dmath.cuh), so for
// the same torsion sin/cos the results are bit-identical to the CPU oracle.
// Compiled with -fmad=false.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "../../../include/vs_crtrig.h"
#include "../../../include/vs_dock.h"
#include "kernels.cuh"

namespace vsd {

// CR sin/cos of the 36 flatten lattice angles idx * (2 pi / 36)
// (search.cpp:33,40), computed on the host with vs_crtrig.
__constant__ double c_lattice_sc[72];

// A kernel's max-dynamic-shared-memory attribute is process-wide state:
// CUDA workers on other host threads launching the same kernel with another
// size must not change it between this thread's set and launch.
std::mutex &launch_mutex() {
  static std::mutex mu;
  return mu;
}

void set_lattice_table(const double *sc72, const double *lo72) {
  cudaMemcpyToSymbol(c_lattice_sc, sc72, sizeof(double) * 72);
  set_lattice_table_search(sc72, lo72);
}

__device__ __forceinline__ d3 ld3(const double *p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double *p, d3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

// ============================================================== k_setup
__global__ void k_setup(batch_dev b, int restarts) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= b.n_lig) return;
  const int a0 = b.atom_off[l], N = b.atom_off[l + 1] - a0;
  const int b0 = b.bond_off[l], nb = b.bond_off[l + 1] - b0;
  const int t0 = b.tors_off[l], m = b.tors_off[l + 1] - t0;
  lig_meta meta{N, 0, m, VS_LIG_OK, 0, 0, 0};
  if (b.pre_status && b.pre_status[l] != 0) {  // a record that failed to decode (vs_dock_records)
    meta.status = VS_LIG_BAD_RECORD;
    b.meta[l] = meta;
    return;
  }
  // apply_torsion's index checks (transform.cpp:56-57, 66-67) fire in the
  // first flatten pass, before any coordinate is used.
  if (m > VS_MAX_TORSIONS) meta.status = VS_LIG_TOO_LARGE;
  for (int t = 0; t < m && meta.status == VS_LIG_OK; ++t) {
    const int bi = b.tors_bond[t0 + t];
    if (bi >= nb) {
      meta.status = VS_LIG_BAD_TORSION;
      break;
    }
    if (b.bond_a[b0 + bi] >= N || b.bond_b[b0 + bi] >= N) meta.status = VS_LIG_BAD_TORSION;
    for (int r = b.right_off[t0 + t]; r < b.right_off[t0 + t + 1]; ++r)
      if (b.right_atoms[r] >= N) meta.status = VS_LIG_BAD_TORSION;
  }
  if (meta.status == VS_LIG_OK && N == 0) meta.status = VS_LIG_EMPTY;  // centroid, transform.cpp:50
  if (meta.status == VS_LIG_OK && N > VS_MAX_ATOMS) meta.status = VS_LIG_TOO_LARGE;
  if (meta.status != VS_LIG_OK) {
    b.meta[l] = meta;
    return;
  }
  int n = 0;
  for (int a = 0; a < N; ++a) {
    b.atom_tmask[a0 + a] = 0u;
    if (b.heavy[a0 + a]) b.heavy_list[a0 + n++] = (uint16_t)a;
  }
  meta.n_heavy = n;
  if (n > VS_MAX_HEAVY) {
    meta.status = VS_LIG_TOO_LARGE;
    b.meta[l] = meta;
    return;
  }
  if (n == 0 && restarts >= 2) {  // heavy_atom_rmsd, transform.cpp:111
    meta.status = VS_LIG_NO_HEAVY;
    b.meta[l] = meta;
    return;
  }
  for (int h = 0; h < n; ++h) b.heavy_dmask[a0 + h] = 0u;
  for (int t = 0; t < m; ++t)
    for (int r = b.right_off[t0 + t]; r < b.right_off[t0 + t + 1]; ++r) {
      b.atom_tmask[a0 + b.right_atoms[r]] |= 1u << t;
      meta.r_all += 1;
      meta.r_heavy += b.heavy[a0 + b.right_atoms[r]] ? 1 : 0;
    }
  for (int t = 0; t < m; ++t) {
    const int bi = b.tors_bond[t0 + t];
    b.tors_a[t0 + t] = b.bond_a[b0 + bi];
    b.tors_b[t0 + t] = b.bond_b[b0 + bi];
  }
  // D_t: atoms whose coordinates can depend on torsion t's angle.  Start
  // from right_set(t); a later torsion u joins when either endpoint is
  // already in the set (its axis moves), adding right_set(u).  Atoms outside
  // D_t follow bit-identical trajectories whatever angle t takes.
  int off = 0;
  const int base = b.ditem_base[l];
  for (int t = 0; t < m; ++t) {
    uint32_t dset = 1u << t;  // torsions whose right sets are in D_t
    for (int u = t + 1; u < m; ++u) {
      const int ea = b.tors_a[t0 + u], eb = b.tors_b[t0 + u];
      if ((b.atom_tmask[a0 + ea] & dset) || (b.atom_tmask[a0 + eb] & dset)) dset |= 1u << u;
    }
    int cnt = 0;
    for (int h = 0; h < n; ++h) {
      if (b.atom_tmask[a0 + b.heavy_list[a0 + h]] & dset) {
        b.heavy_dmask[a0 + h] |= 1u << t;
        b.ditems[base + off + cnt] = (uint16_t)h;
        ++cnt;
      }
    }
    // Order D_t by the atoms' remaining torsion chain (right-set membership
    // of torsions >= t), so that neighbouring search lanes apply the same
    // rotations (less divergence).  Stable insertion sort, lists are short.
    uint16_t *dl = b.ditems + base + off;
    for (int i = 1; i < cnt; ++i) {
      const uint16_t hv = dl[i];
      const uint32_t key = b.atom_tmask[a0 + b.heavy_list[a0 + hv]] >> t;
      int j = i - 1;
      while (j >= 0 && (b.atom_tmask[a0 + b.heavy_list[a0 + dl[j]]] >> t) > key) {
        dl[j + 1] = dl[j];
        --j;
      }
      dl[j + 1] = hv;
    }
    b.d_count[t0 + t] = cnt;
    b.d_off[t0 + t] = off;
    // the 2*cnt search items of neighbours (t,+) and (t,-), in that order;
    // bits 14+ index the atom's stage-t position in the search's prefix list
    for (int s = 0; s < 2; ++s)
      for (int i = 0; i < cnt; ++i)
        b.titems[2 * base + 2 * off + s * cnt + i] =
            (uint32_t)dl[i] | ((uint32_t)(2 * t + s) << 8) | ((uint32_t)(off + i) << 14);
    off += cnt;
  }
  meta.d_total = off;
  b.meta[l] = meta;
}

cudaError_t launch_setup(const batch_dev &b, int restarts, cudaStream_t s) {
  if (b.n_lig == 0) return cudaSuccess;
  k_setup<<<(b.n_lig + 127) / 128, 128, 0, s>>>(b, restarts);
  return cudaGetLastError();
}

// ============================================================== k_flatten
// One CTA per ligand; thread o evaluates candidate offset o of the current
// torsion (search.cpp:50-58).  The prefix state P (torsions < t applied with
// the current lattice indices, all atoms) is shared; each candidate applies
// torsions t..m-1 to its private copy (layout [atom][xyz][candidate]) and
// sums all pair distances sequentially (transform.cpp:83-90).
constexpr int kFlatThreads = 64;
#ifndef VS_FLAT_UNROLL
#define VS_FLAT_UNROLL 4
#endif
constexpr int kFlatUnroll = VS_FLAT_UNROLL;  // independent pair distances in flight per thread

__device__ __forceinline__ void lattice_sc(int idx, double &s, double &c) {
  s = c_lattice_sc[2 * idx];
  c = c_lattice_sc[2 * idx + 1];
}

__global__ void __launch_bounds__(kFlatThreads) k_flatten(batch_dev b, int max_sweeps, flat_out f, int cand_per_round,
                                                          const int *lig_index) {
  extern __shared__ double sm[];
  const int l = lig_index ? lig_index[blockIdx.x] : blockIdx.x;
  const int tid = threadIdx.x;
  const lig_meta meta = b.meta[l];
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const int N = meta.n_atoms, m = meta.m;
  if (meta.status != VS_LIG_OK) return;
  const int CB = cand_per_round;
  double *P = sm;                  // N*3
  double *cand = P + 3 * N;        // N*3*CB
  double *spread = cand + 3 * N * CB;  // 36
  double *mat = spread + 36;       // 12 (prefix advance)
  __shared__ int idx[VS_MAX_TORSIONS + 1];
  __shared__ int changed, bad, sweeps_done;
  const double *base = b.xyz + 3 * (size_t)a0;
  const uint32_t *tm = b.atom_tmask + a0;
  const int b0 = b.bond_off[l];
  if (tid < m) idx[tid] = 0;
  if (tid == 0) {
    bad = 0;
    sweeps_done = 0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps && m > 0; ++sweep) {
    __syncthreads();  // every thread has read the previous sweep's `changed`
    if (tid == 0) sweeps_done = sweep + 1;
    for (int i = tid; i < 3 * N; i += blockDim.x) P[i] = base[i];
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int t = 0; t < m; ++t) {
      for (int r0 = 0; r0 < 36; r0 += CB) {
        const int o = r0 + tid;
        if (tid < CB && o < 36) {
          double *C = cand + tid;  // element (a, c) at C[(3a + c) * CB]
          for (int a = 0; a < N; ++a)
            for (int c = 0; c < 3; ++c) C[(3 * a + c) * CB] = P[3 * a + c];
          bool ok = true;
          for (int u = t; u < m; ++u) {
            const int bi = b.tors_bond[t0 + u];
            const int ea = b.bond_a[b0 + bi], eb = b.bond_b[b0 + bi];
            const int li = u == t ? (idx[t] + o) % 36 : idx[u];
            double s, c;
            lattice_sc(li, s, c);
            double M[12];
            const d3 pa{C[(3 * ea) * CB], C[(3 * ea + 1) * CB], C[(3 * ea + 2) * CB]};
            const d3 pb{C[(3 * eb) * CB], C[(3 * eb + 1) * CB], C[(3 * eb + 2) * CB]};
            if (!torsion_setup(pa, pb, s, c, M)) {
              ok = false;
              break;
            }
            for (int a = 0; a < N; ++a) {
              if (!((tm[a] >> u) & 1u)) continue;
              const d3 x{C[(3 * a) * CB], C[(3 * a + 1) * CB], C[(3 * a + 2) * CB]};
              const d3 y = torsion_apply(M, x);
              C[(3 * a) * CB] = y.x;
              C[(3 * a + 1) * CB] = y.y;
              C[(3 * a + 2) * CB] = y.z;
            }
          }
          if (!ok) bad = 1;
          double sum = 0.0;
          for (int i = 0; i + 1 < N; ++i) {
            const d3 xi{C[(3 * i) * CB], C[(3 * i + 1) * CB], C[(3 * i + 2) * CB]};
            int j = i + 1;
            for (; j + kFlatUnroll - 1 < N; j += kFlatUnroll) {
              double d[kFlatUnroll];
#pragma unroll
              for (int q = 0; q < kFlatUnroll; ++q) {
                const d3 xj{C[(3 * (j + q)) * CB], C[(3 * (j + q) + 1) * CB], C[(3 * (j + q) + 2) * CB]};
                d[q] = dsqrt_dist2(sqn3(sub3(xi, xj)));
              }
#pragma unroll
              for (int q = 0; q < kFlatUnroll; ++q) sum += d[q];
            }
            for (; j < N; ++j) {
              const d3 xj{C[(3 * j) * CB], C[(3 * j + 1) * CB], C[(3 * j + 2) * CB]};
              sum += dsqrt_dist2(sqn3(sub3(xi, xj)));
            }
          }
          spread[o] = sum;
        }
        __syncthreads();
      }
      if (tid == 0) {
        int best_off = 0;
        double best = -__longlong_as_double(0x7ff0000000000000LL);
        for (int o = 0; o < 36; ++o)
          if (spread[o] > best) {
            best = spread[o];
            best_off = o;
          }
        if (best_off != 0) {
          idx[t] = (idx[t] + best_off) % 36;
          changed = 1;
        }
        // prefix advance: torsion t with its (possibly new) index
        const int bi = b.tors_bond[t0 + t];
        const int ea = b.bond_a[b0 + bi], eb = b.bond_b[b0 + bi];
        double s, c;
        lattice_sc(idx[t], s, c);
        if (!torsion_setup(ld3(P + 3 * ea), ld3(P + 3 * eb), s, c, mat)) bad = 1;
      }
      __syncthreads();
      if (bad) break;
      for (int a = tid; a < N; a += blockDim.x)
        if ((tm[a] >> t) & 1u) st3(P + 3 * a, torsion_apply(mat, ld3(P + 3 * a)));
      __syncthreads();
    }
    if (bad || !changed) break;
  }
  if (bad) {
    if (tid == 0) b.meta[l].status = VS_LIG_DEGENERATE_AXIS;
    return;
  }
  // flat conformation = apply_torsions(base, angles_of(index)) (search.cpp:67-68)
  for (int i = tid; i < 3 * N; i += blockDim.x) P[i] = base[i];
  __syncthreads();
  for (int t = 0; t < m; ++t) {
    if (tid == 0) {
      const int bi = b.tors_bond[t0 + t];
      const int ea = b.bond_a[b0 + bi], eb = b.bond_b[b0 + bi];
      double s, c;
      lattice_sc(idx[t], s, c);
      if (!torsion_setup(ld3(P + 3 * ea), ld3(P + 3 * eb), s, c, mat)) bad = 1;
    }
    __syncthreads();
    if (bad) break;
    for (int a = tid; a < N; a += blockDim.x)
      if ((tm[a] >> t) & 1u) st3(P + 3 * a, torsion_apply(mat, ld3(P + 3 * a)));
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) b.meta[l].status = VS_LIG_DEGENERATE_AXIS;
    return;
  }
  for (int i = tid; i < 3 * N; i += blockDim.x) f.xyz[3 * (size_t)a0 + i] = P[i];
  if (tid < m) f.idx[t0 + tid] = idx[tid];
  if (tid < 3) f.centroid[3 * l + tid] = centroid_row(P, N, tid);
  if (tid == 0) f.sweeps[l] = sweeps_done;
}

// ============================================================== k_flatten_dep
// The same flatten, organised around what the 36 candidates of torsion t
// actually change.  The spread sums only feed an argmax (search.cpp:52-58), so
// a candidate needs its exact sequential sum (transform.cpp:83-90) only when
// another candidate comes within rounding distance of it:
//   * D_t = atoms whose final position depends on the candidate: moved by t or
//     by a later torsion whose axis moves with the candidate (closure over
//     u > t).  Every other atom ends where all candidates put it; that common
//     position (Q) and the matrices of the candidate-independent torsions are
//     computed once per t by warp 0 -- the same operations on the same values
//     as in every candidate of the legacy kernel, so bit-identical.
//   * 8 lanes per candidate (288 threads = 36 x 8, no idle lane) transform the
//     D_t atoms and sum the distances of the pairs that touch D_t, in any
//     order ("A_o"); pairs of two common atoms add the same I to every
//     candidate and are only bounded (I <= (n_I - 1) * sum |q - q_0|).
//   * The reference's choice is the first argmax of R_o = fl_seq(I + T_o).
//     With n pairs, |R_o - (I + T_o)| <= gamma_n (I + T_o) and our A_o carries
//     at most the same plus the 2^-50 of the filter square root (and 2^-500
//     absolute per pair: near-coincident atoms sample 0), so
//     A_best - A_o > ((2 I_bound + A_best + A_o) * 2^-48 + 2^-499) * n proves
//     R_best > R_o (the 2^-48 = 32 u covers 2 gamma_n + 2^-49 from n = 1 on).  Candidates that fail the test (near ties: symmetric
//     groups, ~2% of decisions) get the exact sequential sum of the legacy
//     kernel, and the argmax is taken over those exact values.
// The decision, and so every output, is bit-identical to the legacy kernel.
#ifdef VS_FLAT_PROF  // development only: thread 0's clock64() time per phase (tools/flat_prof.py)
__device__ unsigned long long g_fphase[16];  // 0-6 phases, 7 CTAs, 8 decisions, 9 exact near-tie paths
#define FP_MARK(k)                             \
  if (tid == 0) {                              \
    const unsigned long long fp_n = clock64(); \
    fp_acc[k] += fp_n - fp_t;                  \
    fp_t = fp_n;                               \
  }
#else
#define FP_MARK(k)
#endif
// Development bounds checks (build with -DVS_DEBUG_CHECKS): trap instead of
// reading or writing out of range.
#ifdef VS_DEBUG_CHECKS
#define VS_KCHECK(c) \
  do {               \
    if (!(c)) __trap(); \
  } while (0)
#else
#define VS_KCHECK(c) \
  do {               \
  } while (0)
#endif
constexpr int kFC = 36;         // candidates per torsion (10-degree lattice offsets)
constexpr int kFL = 8;          // lanes per candidate
constexpr int kFT = kFC * kFL;  // 288 threads = 9 full warps

// sqrt for the filter sums: MUFU seed + one third-order step, relative error
// below 2^-50 (no final rounding correction; the bound above allows for it).
__device__ __forceinline__ double dsqrt_filter(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double e = fma(x, -(y0 * y0), 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double y1 = fma(p, y0 * e, y0);
  return x < 0x1p-1000 ? 0.0 : x * y1;
}

size_t flatten_dep_smem(int nmax, int mmax) {
  return (size_t)(3 * nmax + 3 * nmax + 4 * nmax + 3 * nmax * kFC + 18 * mmax + 3 * kFC) * sizeof(double) +
         (size_t)(5 * nmax + mmax) * sizeof(int);
}

#ifndef VS_FLAT_RIGID_DD
#define VS_FLAT_RIGID_DD 16  // D_t sizes from which the D_t x D_t sums come from candidate 0 + a bound (0: off)
#endif

// Rigid-subtree mode helpers of k_flatten_dep (out of line: their registers
// stay out of the kernel's 72).  Thread `tid`'s share (stride kFT) of
// candidate 0's D_t x D_t filter sum.
__device__ __noinline__ double flat_dd0_share(const double *C, int nd, int tid) {
  double dd = 0.0;
  int r = 0, k = tid, len = nd - 1;
  while (r < nd - 1 && k >= len) {
    k -= len;
    ++r;
    len = nd - 1 - r;
  }
  d3 xi{0.0, 0.0, 0.0};
  if (r < nd - 1) xi = d3{C[(3 * r) * kFC], C[(3 * r + 1) * kFC], C[(3 * r + 2) * kFC]};
  while (r < nd - 1) {
    VS_KCHECK(r + 1 + k < nd);
    const double *q = C + 3 * (r + 1 + k) * kFC;
    dd += dsqrt_filter(sqn3(sub3(xi, d3{q[0], q[kFC], q[2 * kFC]})));
    k += kFT;
    if (k >= len) {
      do {
        k -= len;
        ++r;
        len = nd - 1 - r;
      } while (r < nd - 1 && k >= len);
      if (r < nd - 1) xi = d3{C[(3 * r) * kFC], C[(3 * r + 1) * kFC], C[(3 * r + 2) * kFC]};
    }
  }
  return dd;
}

// Lane g's share of sum_i |r_i| for candidate o: r_i = y_i(o) - (R (y_i(0) -
// p) + p), R the rotation about torsion t's axis (stage-t endpoints, the same
// for every candidate) by o x 10 degrees; each |r_i| taken as its 1-norm plus
// 2^-46 X_i for the rounding of its evaluation (<= 60 u X_i).  Writes eps >=
// ||R^T R - I||_F plus its own rounding (lane g = 0).  A degenerate axis gives
// +inf (no exclusion).
__device__ __noinline__ double flat_rigid_residual(const double *C, const double *Co, const double *P, int ax, int o,
                                                   int nd, int g, double *eps) {
  double M[12], sn, cs;
  lattice_sc(o, sn, cs);
  if (!torsion_setup(ld3(P + 3 * (ax & 0xffff)), ld3(P + 3 * (ax >> 16)), sn, cs, M))
    return __longlong_as_double(0x7ff0000000000000LL);
  const double pm = fmax(fabs(M[9]), fmax(fabs(M[10]), fabs(M[11])));
  double rs = 0.0;
  VS_KCHECK(o > 0 && o < kFC && nd <= VS_MAX_ATOMS);
  for (int r = g; r < nd; r += kFL) {
    const d3 y0{C[(3 * r) * kFC], C[(3 * r + 1) * kFC], C[(3 * r + 2) * kFC]};
    const d3 yo{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
    const d3 e = sub3(yo, torsion_apply(M, y0));
    const double xm = fmax(fmax(fmax(fabs(y0.x), fabs(y0.y)), fmax(fabs(y0.z), fabs(yo.x))),
                           fmax(fmax(fabs(yo.y), fabs(yo.z)), pm));
    rs += (fabs(e.x) + fabs(e.y)) + fabs(e.z) + xm * 0x1p-46;
  }
  if (g == 0) {
    double f = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int c = a; c < 3; ++c) {
        const double v = (M[a] * M[c] + M[3 + a] * M[3 + c]) + M[6 + a] * M[6 + c];
        f += (a == c ? 1.0 : 2.0) * fabs(v - (a == c ? 1.0 : 0.0));
      }
    *eps = f + 0x1p-47;
  }
  return rs;
}

#ifndef VS_FLAT_ROWS
#define VS_FLAT_ROWS 1  // cross pairs: whole rows per lane (4 distances in flight) before the strided walk
#endif
#ifndef VS_FLAT_MINB
#define VS_FLAT_MINB 3  // 3 CTAs (27 warps) per SM: 72 registers; without the cap 92 (2 CTAs) measured 35% slower,
                        // 4 (56 registers, 412 B spills) 3.5% slower
#endif
__global__ void __launch_bounds__(kFT, VS_FLAT_MINB) k_flatten_dep(batch_dev b, int max_sweeps, flat_out f, int nmax,
                                                                   int mmax, const int *lig_index) {
  extern __shared__ double sm[];
  const int l = lig_index ? lig_index[blockIdx.x] : blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const lig_meta meta = b.meta[l];
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const int N = meta.n_atoms, m = meta.m;
  if (meta.status != VS_LIG_OK) return;
  double *P = sm;                   // [N][3] stage-t prefix (torsions < t applied)
  double *Q = P + 3 * nmax;         // [N][3] common positions (candidate-independent torsions applied)
  double *Qc = Q + 3 * nmax;        // [n_I][4] Q of the common atoms, compacted
  double *C = Qc + 4 * nmax;        // [rank][xyz][36] candidate positions of the D_t atoms
  double *Ms = C + 3 * nmax * kFC;  // [u][12] matrices of the candidate-independent torsions
  double *AX = Ms + 12 * mmax;      // [u][6] stage-u axis endpoints of the dependent torsions
  double *spread = AX + 6 * mmax;   // [36] filter sums A_o
  double *devb = spread + kFC;      // [36] rigid-subtree mode: (nd - 1) * sum of residuals of candidate o
  double *epsb = devb + kFC;        // [36] rigid-subtree mode: orthogonality defect of candidate o's map
  int *dl = reinterpret_cast<int *>(epsb + kFC);              // rank -> atom
  int *nl = dl + nmax;                                        // common atoms, ascending
  int *slot = nl + nmax;                                      // atom -> rank, -1 for common atoms
  uint32_t *tms = reinterpret_cast<uint32_t *>(slot + nmax);  // right-set masks of the atoms
  uint32_t *tmr = tms + nmax;                                 // right-set mask of rank r
  int *tax = reinterpret_cast<int *>(tmr + nmax);             // torsion u's axis atoms, ea | eb << 16
  __shared__ int idx[VS_MAX_TORSIONS + 1];
  __shared__ int changed, bad, sweeps_done, s_nd, s_nn, s_ver, s_skip;
  __shared__ int stamp[VS_MAX_TORSIONS + 1];
  __shared__ uint32_t s_dt, s_du;
  __shared__ double s_ib, s_dd0;
  __shared__ int s_rig;
  const double *base = b.xyz + 3 * (size_t)a0;
  const int o = tid >> 3, g = tid & 7;
  double *Co = C + o;  // element (r, c) of this lane's candidate at Co[(3r + c) * kFC]
  const double npairs = 0.5 * (double)N * (double)(N - 1);
  const double ninf = -__longlong_as_double(0x7ff0000000000000LL);
  if (tid < m) {
    idx[tid] = 0;
    stamp[tid] = -1;
    const int bi = b.tors_bond[t0 + tid], b0 = b.bond_off[l];
    tax[tid] = b.bond_a[b0 + bi] | (b.bond_b[b0 + bi] << 16);
  }
  for (int a = tid; a < N; a += blockDim.x) tms[a] = b.atom_tmask[a0 + a];
  if (tid == 0) {
    bad = 0;
    sweeps_done = 0;
    s_ver = 0;
  }
  __syncthreads();
#ifdef VS_FLAT_PROF
  unsigned long long fp_acc[8] = {0}, fp_t = clock64();
#endif
  for (int sweep = 0; sweep < max_sweeps && m > 0; ++sweep) {
    if (sweep) __syncthreads();  // every thread has read the previous sweep's `changed`
    if (tid == 0) {
      sweeps_done = sweep + 1;
      changed = 0;
    }
    for (int i = tid; i < 3 * N; i += blockDim.x) P[i] = base[i];
    __syncthreads();
    for (int t = 0; t < m; ++t) {
      // ---- A (warp 0): D_t, the common positions, the shared matrices.
      // If no lattice index changed since torsion t's last decision, its 36
      // candidates are the same conformations as then, cyclically shifted so
      // that the previous winner sits at offset 0: the first argmax is 0 and
      // the evaluation is skipped (only the prefix advances).
      if (tid < 32 && stamp[t] == s_ver) {
        if (lane == 0) s_skip = 1;
      } else if (tid < 32) {
        if (lane == 0) s_skip = 0;
        uint32_t dt = 1u << t;
        for (int u = t + 1; u < m; ++u) {
          const int ax = tax[u];
          if ((tms[ax & 0xffff] | tms[ax >> 16]) & dt) dt |= 1u << u;
        }
        int nd = 0, nn = 0;
        uint32_t du = 0;
        for (int c0 = 0; c0 < N; c0 += 32) {
          const int a = c0 + lane;
          const bool in = a < N;
          const uint32_t ma = in ? tms[a] : 0u;
          const bool dep = in && (ma & dt);
          const unsigned bd = __ballot_sync(0xffffffffu, dep), bn = __ballot_sync(0xffffffffu, in && !dep);
          const unsigned below = (1u << lane) - 1u;
          if (dep) {
            const int r = nd + __popc(bd & below);
            dl[r] = a;
            slot[a] = r;
            tmr[r] = ma;
            du |= ma;
          } else if (in) {
            nl[nn + __popc(bn & below)] = a;
            slot[a] = -1;
          }
          nd += __popc(bd);
          nn += __popc(bn);
        }
        du = __reduce_or_sync(0xffffffffu, du);
        for (int i = lane; i < 3 * N; i += 32) Q[i] = P[i];
        __syncwarp();
        for (int u = t + 1; u < m; ++u) {
          const int ax = tax[u], ea = ax & 0xffff, eb = ax >> 16;
          if ((dt >> u) & 1u) {
            if (lane < 3) {
              AX[6 * u + lane] = Q[3 * ea + lane];
              AX[6 * u + 3 + lane] = Q[3 * eb + lane];
            }
          } else {
            double M[12], s, c;
            lattice_sc(idx[u], s, c);
            if (!torsion_setup(ld3(Q + 3 * ea), ld3(Q + 3 * eb), s, c, M) && lane == 0) bad = 1;
            if (lane == 0)
#pragma unroll
              for (int k = 0; k < 12; ++k) Ms[12 * u + k] = M[k];
            __syncwarp();  // everyone has read the endpoints
            for (int a = lane; a < N; a += 32)
              if ((tms[a] >> u) & 1u) st3(Q + 3 * a, torsion_apply(M, ld3(Q + 3 * a)));
          }
          __syncwarp();
        }
        // compacted common positions and the bound on their pair sum
        double acc = 0.0;
        const d3 q0 = nn > 0 ? ld3(Q + 3 * nl[0]) : d3{0.0, 0.0, 0.0};
        for (int k = lane; k < nn; k += 32) {
          const d3 q = ld3(Q + 3 * nl[k]);
          Qc[4 * k] = q.x;
          Qc[4 * k + 1] = q.y;
          Qc[4 * k + 2] = q.z;
          acc += dsqrt_filter(sqn3(sub3(q, q0)));
        }
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
        if (lane == 0) {
          s_nd = nd;
          s_nn = nn;
          s_dt = dt;
          s_du = du;
          s_ib = acc * (double)(nn > 0 ? nn - 1 : 0) * (1.0 + 0x1p-40);
          s_rig = VS_FLAT_RIGID_DD > 0 && nd >= VS_FLAT_RIGID_DD;
          s_dd0 = 0.0;
        }
      }
      __syncthreads();
      FP_MARK(0)
      if (bad) break;
      const bool skipping = s_skip;
      if (!skipping) {
        // ---- B: this lane's share of its candidate's D_t atoms through t..m-1
        const int nd = s_nd, nn = s_nn;
        const uint32_t dt = s_dt, du = s_du;
        for (int r = g; r < nd; r += kFL) {
          const int a = dl[r];
#pragma unroll
          for (int c = 0; c < 3; ++c) Co[(3 * r + c) * kFC] = P[3 * a + c];
        }
        __syncwarp();
        for (int u = t; u < m; ++u) {
          if (!(((du | dt) >> u) & 1u)) continue;  // candidate-independent and moves no D_t atom
          double M[12];
          if ((dt >> u) & 1u) {
            const int ax = tax[u], ea = ax & 0xffff, eb = ax >> 16;
            d3 pa, pb;
            if (u == t) {
              pa = ld3(P + 3 * ea);
              pb = ld3(P + 3 * eb);
            } else {
              const int sa = slot[ea], sb = slot[eb];
              pa = sa >= 0 ? d3{Co[(3 * sa) * kFC], Co[(3 * sa + 1) * kFC], Co[(3 * sa + 2) * kFC]} : ld3(AX + 6 * u);
              pb = sb >= 0 ? d3{Co[(3 * sb) * kFC], Co[(3 * sb + 1) * kFC], Co[(3 * sb + 2) * kFC]}
                           : ld3(AX + 6 * u + 3);
            }
            double s, c;
            lattice_sc(u == t ? (idx[t] + o) % 36 : idx[u], s, c);
            if (!torsion_setup(pa, pb, s, c, M)) bad = 1;
          } else {
#pragma unroll
            for (int k = 0; k < 12; ++k) M[k] = Ms[12 * u + k];
          }
          __syncwarp();  // endpoints read before anyone moves them
          for (int r = g; r < nd; r += kFL)
            if ((tmr[r] >> u) & 1u) {
              double *x = Co + 3 * r * kFC;
              const d3 y = torsion_apply(M, d3{x[0], x[kFC], x[2 * kFC]});
              x[0] = y.x;
              x[kFC] = y.y;
              x[2 * kFC] = y.z;
            }
          __syncwarp();
        }
        FP_MARK(1)
        // ---- C: filter sum over the pairs that touch D_t, in two flattened
        // walks strided by the 8 lanes of the candidate: (rank r, common k),
        // then (rank r, rank s > r).
        {
          double acc = 0.0;
#if VS_FLAT_ROWS
          // full rows first: lane g takes ranks g, g + 8, ... of the first
          // 8 * floor(nd / 8) and walks all nn common atoms, four at a time
          const int nd8 = nd & ~(kFL - 1);
          if (nn > 0)
            for (int r = g; r < nd8; r += kFL) {
              const d3 xi{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
              int k = 0;
              for (; k + 4 <= nn; k += 4) {
                double d[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const double *q = Qc + 4 * (k + e);
                  d[e] = dsqrt_filter(sqn3(sub3(xi, d3{q[0], q[1], q[2]})));
                }
                acc += (d[0] + d[1]) + (d[2] + d[3]);
              }
              for (; k < nn; ++k) {
                const double *q = Qc + 4 * k;
                acc += dsqrt_filter(sqn3(sub3(xi, d3{q[0], q[1], q[2]})));
              }
            }
#else
          const int nd8 = 0;
#endif
          if (nn > 0) {
            int r = nd8 + g / nn, k = g - (g / nn) * nn;
            d3 xi{0.0, 0.0, 0.0};
            if (r < nd) xi = d3{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
            while (r < nd) {
              const double *q = Qc + 4 * k;
              acc += dsqrt_filter(sqn3(sub3(xi, d3{q[0], q[1], q[2]})));
              k += kFL;
              if (k >= nn) {
                do {
                  k -= nn;
                  ++r;
                } while (k >= nn);
                if (r < nd) xi = d3{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
              }
            }
          }
          if (!s_rig) {
            {
              int r = 0, k = g, len = nd - 1;
              while (r < nd - 1 && k >= len) {
                k -= len;
                ++r;
                len = nd - 1 - r;
              }
              d3 xi{0.0, 0.0, 0.0};
              if (r < nd - 1) xi = d3{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
              while (r < nd - 1) {
                const double *q = Co + 3 * (r + 1 + k) * kFC;
                acc += dsqrt_filter(sqn3(sub3(xi, d3{q[0], q[kFC], q[2 * kFC]})));
                k += kFL;
                if (k >= len) {
                  do {
                    k -= len;
                    ++r;
                    len = nd - 1 - r;
                  } while (r < nd - 1 && k >= len);
                  if (r < nd - 1) xi = d3{Co[(3 * r) * kFC], Co[(3 * r + 1) * kFC], Co[(3 * r + 2) * kFC]};
                }
              }
            }
          } else {
            // Rigid-subtree mode.  In exact arithmetic every candidate moves
            // D_t as one rigid body (the right subtree of t; nested axes ride
            // along), so its D_t x D_t sum is candidate 0's: all 288 threads
            // sum candidate 0's triangle into s_dd0, and each candidate bounds
            // how far it is from a rigid image of candidate 0.  With y(o) =
            // R (y(0) - p) + p + r (R: the rotation about t's axis by o x 10
            // degrees, built here; r: the residuals),
            //   |DD_o - DD_0| <= eps DD_0 + (nd - 1) sum_i |r_i|,
            // eps >= the orthogonality defect of R.  D tests with these.
            double dd = flat_dd0_share(C, nd, tid);
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, sh);
            if (lane == 0) atomicAdd(&s_dd0, dd);
            double eps = 0.0;
            double rs = o != 0 ? flat_rigid_residual(C, Co, P, tax[t], o, nd, g, &eps) : 0.0;
            rs += __shfl_xor_sync(0xffffffffu, rs, 1);
            rs += __shfl_xor_sync(0xffffffffu, rs, 2);
            rs += __shfl_xor_sync(0xffffffffu, rs, 4);
            if (g == 0) {
              devb[o] = rs * (double)(nd - 1) * (1.0 + 0x1p-40);
              epsb[o] = eps;
            }
          }
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          acc += __shfl_xor_sync(0xffffffffu, acc, 4);
          if (g == 0) spread[o] = acc;
        }
      }  // !skipping
      FP_MARK(2)
      __syncthreads();  // (skipping: every thread has read bad and s_skip)
      FP_MARK(3)
      // ---- D (warp 0): certain winner, or the exact sums of the candidates
      // within rounding of it; then the prefix advance (search.cpp:52-60)
      if (tid < 32) {
        int best_off = 0;
        if (!skipping) {
          // first argmax (the reference's strict > from -inf; NaN never wins)
          // rigid-subtree mode: A_o = spread + DD_0, and T_o lies within dev_o of it
          const bool rig = s_rig;
          const double dd0 = rig ? s_dd0 : 0.0;
          const double v0 = spread[lane] + dd0, v1 = lane + 32 < kFC ? spread[lane + 32] + dd0 : ninf;
          double bv = v0 == v0 ? v0 : ninf;
          int bo = lane;
          if (v1 > bv) {
            bv = v1;
            bo = lane + 32;
          }
#pragma unroll
          for (int sh = 16; sh; sh >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, sh);
            const int oo = __shfl_xor_sync(0xffffffffu, bo, sh);
            if (ov > bv || (ov == bv && oo < bo)) {
              bv = ov;
              bo = oo;
            }
          }
          if (bv == ninf) bo = 0;
          const double ib2 = 2.0 * s_ib;
          const double ddu = dd0 * (1.0 + 0x1p-30);  // >= the exact DD_0: filter sum + 2^-50 per distance + gamma(<= 32640 terms) < 2^-37
          auto dev = [&](int q) { return rig ? devb[q] + epsb[q] * ddu : 0.0; };
          const double db = dev(bo), d0 = dev(lane), d1 = lane + 32 < kFC ? dev(lane + 32) : 0.0;
          const bool n0 = lane != bo &&
                          !(bv - v0 > db + d0 + ((ib2 + bv + db + v0 + d0) * 0x1p-48 + 0x1p-499) * npairs);
          const bool n1 = lane + 32 < kFC && lane + 32 != bo &&
                          !(bv - v1 > db + d1 + ((ib2 + bv + db + v1 + d1) * 0x1p-48 + 0x1p-499) * npairs);
          unsigned long long w = (unsigned long long)__ballot_sync(0xffffffffu, n0) |
                                 ((unsigned long long)__ballot_sync(0xffffffffu, n1) << 32);
#ifdef VS_FLAT_FORCE_EXACT  // testing only: exact sums for every candidate
          w = (1ull << kFC) - 1;
#endif
          w |= 1ull << bo;
#ifdef VS_FLAT_NO_EXACT  // timing experiments only: trust the filter blindly
          w = 1ull << bo;
#endif
          best_off = bo;
          FP_MARK(4)
#ifdef VS_FLAT_PROF
          if (lane == 0) {
            atomicAdd(&g_fphase[8], 1ull);
            if (__popcll(w) > 1) atomicAdd(&g_fphase[9], 1ull);
          }
#endif
          if (__popcll(w) > 1) {
            // exact sequential sums (transform.cpp:83-90) of the near-tied
            // candidates, first argmax among them
            double ev = ninf;
            int eo = lane;
            for (int q = lane; q < kFC; q += 32) {
              if (!((w >> q) & 1ull)) continue;
              const double *Ct = C + q;
              double sum = 0.0;
              for (int i = 0; i + 1 < N; ++i) {
                const int si = slot[i];
                const d3 xi = si >= 0 ? d3{Ct[(3 * si) * kFC], Ct[(3 * si + 1) * kFC], Ct[(3 * si + 2) * kFC]}
                                      : ld3(Q + 3 * i);
                int j = i + 1;
                for (; j + 3 < N; j += 4) {  // four distances in flight, added in order
                  double d[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const int sj = slot[j + e];
                    const d3 xj = sj >= 0 ? d3{Ct[(3 * sj) * kFC], Ct[(3 * sj + 1) * kFC], Ct[(3 * sj + 2) * kFC]}
                                          : ld3(Q + 3 * (j + e));
                    d[e] = dsqrt_dist2(sqn3(sub3(xi, xj)));
                  }
                  sum += d[0];
                  sum += d[1];
                  sum += d[2];
                  sum += d[3];
                }
                for (; j < N; ++j) {
                  const int sj = slot[j];
                  const d3 xj = sj >= 0 ? d3{Ct[(3 * sj) * kFC], Ct[(3 * sj + 1) * kFC], Ct[(3 * sj + 2) * kFC]}
                                        : ld3(Q + 3 * j);
                  sum += dsqrt_dist2(sqn3(sub3(xi, xj)));
                }
              }
              if (sum > ev) {
                ev = sum;
                eo = q;
              }
            }
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, ev, sh);
              const int oo = __shfl_xor_sync(0xffffffffu, eo, sh);
              if (ov > ev || (ov == ev && oo < eo)) {
                ev = ov;
                eo = oo;
              }
            }
            best_off = ev == ninf ? 0 : eo;
          }
          FP_MARK(5)
        }  // !skipping
        const int nidx = (idx[t] + best_off) % 36;
        __syncwarp();
        if (lane == 0) {
          if (best_off != 0) {
            idx[t] = nidx;
            changed = 1;
            ++s_ver;
          }
          stamp[t] = s_ver;
        }
        const int ax = tax[t];
        double M[12], s, c;
        lattice_sc(nidx, s, c);
        if (!torsion_setup(ld3(P + 3 * (ax & 0xffff)), ld3(P + 3 * (ax >> 16)), s, c, M) && lane == 0) bad = 1;
        __syncwarp();  // endpoints read before the right set moves
        for (int a = lane; a < N; a += 32)
          if ((tms[a] >> t) & 1u) st3(P + 3 * a, torsion_apply(M, ld3(P + 3 * a)));
        __syncwarp();
      }
      FP_MARK(6)
    }
    __syncthreads();
    if (bad || !changed) break;
  }
#ifdef VS_FLAT_PROF
  if (tid == 0) {
    for (int k = 0; k < 7; ++k) atomicAdd(&g_fphase[k], fp_acc[k]);
    atomicAdd(&g_fphase[7], 1ull);
  }
#endif
  if (bad) {
    if (tid == 0) b.meta[l].status = VS_LIG_DEGENERATE_AXIS;
    return;
  }
  // flat conformation = apply_torsions(base, angles_of(index)) (search.cpp:67-68)
  if (tid < 32) {
    for (int i = lane; i < 3 * N; i += 32) P[i] = base[i];
    __syncwarp();
    for (int t = 0; t < m; ++t) {
      const int ax = tax[t];
      double M[12], s, c;
      lattice_sc(idx[t], s, c);
      if (!torsion_setup(ld3(P + 3 * (ax & 0xffff)), ld3(P + 3 * (ax >> 16)), s, c, M) && lane == 0) bad = 1;
      __syncwarp();
      for (int a = lane; a < N; a += 32)
        if ((tms[a] >> t) & 1u) st3(P + 3 * a, torsion_apply(M, ld3(P + 3 * a)));
      __syncwarp();
    }
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) b.meta[l].status = VS_LIG_DEGENERATE_AXIS;
    return;
  }
  for (int i = tid; i < 3 * N; i += blockDim.x) f.xyz[3 * (size_t)a0 + i] = P[i];
  if (tid < m) f.idx[t0 + tid] = idx[tid];
  if (tid < 3) f.centroid[3 * l + tid] = centroid_row(P, N, tid);
  if (tid == 0) f.sweeps[l] = sweeps_done;
}

#ifdef VS_FLAT_PROF
extern "C" int vs_debug_flat_phase_read(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_fphase, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_fphase, z, sizeof z);
  }
  return 0;
}
#endif

#ifndef VS_FLAT_LEGACY
#define VS_FLAT_LEGACY 0  // A/B only: 1 = always the legacy kernel
#endif

cudaError_t launch_flatten(const batch_dev &b, int max_sweeps, const flat_out &f, int nmax_atoms, int mmax,
                           cudaStream_t s, const int *lig_index, int n_lig) {
  const int n = lig_index ? n_lig : b.n_lig;
  if (n == 0) return cudaSuccess;
  const int mm = mmax < 1 ? 1 : mmax;
  const size_t dsmem = flatten_dep_smem(nmax_atoms, mm);
  if (!VS_FLAT_LEGACY && dsmem <= 200 * 1024) {
    std::lock_guard<std::mutex> lock(launch_mutex());
    cudaFuncSetAttribute(k_flatten_dep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    k_flatten_dep<<<n, kFT, dsmem, s>>>(b, max_sweeps, f, nmax_atoms, mm, lig_index);
    return cudaGetLastError();
  }
  int cb = 36;
  auto bytes = [&](int c) { return (size_t)(3 * nmax_atoms * (1 + c) + 36 + 12) * sizeof(double); };
  while (cb > 1 && bytes(cb) > 200 * 1024) cb = (cb + 1) / 2;
  const size_t smem = bytes(cb);
  std::lock_guard<std::mutex> lock(launch_mutex());
  cudaFuncSetAttribute(k_flatten, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_flatten<<<n, kFlatThreads, smem, s>>>(b, max_sweeps, f, cb, lig_index);
  return cudaGetLastError();
}

// ============================================================== chem
// chem_score (chem.cpp:31-46) of one heavy atom against the protein, in
// protein order.  Pairs at d >= 4.5 add nothing in the reference, so only
// the atoms of the cell list (a superset of those within 4.5 A, sorted by
// protein index) are visited; outside the cell grid every atom is.
__device__ __forceinline__ double chem_weight(int a, int b) {
  if (a == 2 || b == 2) return 0.05;
  if (a == 0 && b == 0) return 0.4;
  if (a == 1 && b == 1) return 1.0;
  return 0.1;
}
__device__ __forceinline__ int chem_class_of(uint8_t e) { return e == 0 ? 0 : ((e == 1 || e == 2) ? 1 : 2); }

#ifndef VS_CHEM_REC2
#define VS_CHEM_REC2 1
#endif
#ifndef VS_CHEM_REC4
#define VS_CHEM_REC4 0  // A/B: four records in flight
#endif
__device__ __forceinline__ void chem_atom(const pocket_dev &p, d3 x, int ci, double &total, int &clashes,
                                          int &pairs) {
  int lo = 0, hi = p.n_protein;
  bool culled = false;
  const int cx = (int)floor((x.x - p.cmin[0]) / p.cs);
  const int cy = (int)floor((x.y - p.cmin[1]) / p.cs);
  const int cz = (int)floor((x.z - p.cmin[2]) / p.cs);
  if (p.cell_start && cx >= 0 && cy >= 0 && cz >= 0 && cx < p.cdims[0] && cy < p.cdims[1] && cz < p.cdims[2]) {
    const int cell = cx + p.cdims[0] * (cy + p.cdims[1] * cz);
    lo = p.cell_start[cell];
    hi = p.cell_start[cell + 1];
    culled = true;
  }
  // one protein atom (protein order, chem.cpp:31-46); `pc` its class
  auto pair = [&](d3 pp, int pc) {
    // (an exact d2 >= 20.25 early-out before the sqrt measured 6% slower:
    // the lanes are different poses, so the branch only adds divergence)
    const double d = dsqrt(sqn3(sub3(x, pp)));
    if (d >= 4.5) return;
    ++pairs;
    const double ramp = d <= 3.5 ? 1.0 : (4.5 - d) / (4.5 - 3.5);
    total += chem_weight(ci, pc) * ramp;
    if (d < 2.0) {
      total -= 5.0;
      ++clashes;
    }
  };
  int q = lo;
  if (culled) {
    // culled cell: 32-byte records in list order (two in flight with VS_CHEM_REC2)
    const double2 *rec = p.cell_rec;
#if VS_CHEM_REC4
    for (; q + 4 <= hi; q += 4) {
      double2 a[4], bb[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = __ldg(rec + 2 * (q + e));
        bb[e] = __ldg(rec + 2 * (q + e) + 1);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) pair(d3{a[e].x, a[e].y, bb[e].x}, (int)bb[e].y);
    }
#endif
#if VS_CHEM_REC2
    for (; q + 2 <= hi; q += 2) {
      const double2 a0 = __ldg(rec + 2 * q), b0 = __ldg(rec + 2 * q + 1);
      const double2 a1 = __ldg(rec + 2 * q + 2), b1 = __ldg(rec + 2 * q + 3);
      pair(d3{a0.x, a0.y, b0.x}, (int)b0.y);
      pair(d3{a1.x, a1.y, b1.x}, (int)b1.y);
    }
#endif
    for (; q < hi; ++q) {
      const double2 a0 = __ldg(rec + 2 * q), b0 = __ldg(rec + 2 * q + 1);
      pair(d3{a0.x, a0.y, b0.x}, (int)b0.y);
    }
    return;
  }
  for (; q < hi; ++q)  // no culling cells: every protein atom
    pair(d3{__ldg(p.pxyz + 3 * q), __ldg(p.pxyz + 3 * q + 1), __ldg(p.pxyz + 3 * q + 2)}, p.pclass[q]);
}

// chem_score of a compact heavy-atom conformation (heavy atom h at 3h).
__device__ double chem_pose(const pocket_dev &p, const double *conf, const uint16_t *hl, const uint8_t *elem, int n,
                            int &clashes, int &pairs) {
  double total = 0.0;
  clashes = 0;
  pairs = 0;
  for (int h = 0; h < n; ++h) chem_atom(p, ld3(conf + 3 * h), chem_class_of(elem[hl[h]]), total, clashes, pairs);
  return total;
}

// The best pose's full conformation (atom order) from its compact heavy-atom
// conformation, its angles and its transform: heavy atoms copied (the bits
// k_search produced), hydrogens rematerialised as apply_rigid(
// apply_torsions(base, angles), T) (pose.hpp:20-22; transform.cpp:73-81,
// 31): lane 0 rebuilds the torsion matrices from the base coordinates and
// the correctly rounded sin/cos of the final angles -- the values and
// operations of k_search's chains -- then the lanes carry the hydrogens.
// M: 12 m doubles of scratch.  Warp-cooperative.
__device__ void best_conformation(const batch_dev &b, int l, const double *hc, const double *ang, const double *T7,
                                  double *M, double *out, int lane) {
  const lig_meta meta = b.meta[l];
  const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const double *base = b.xyz + 3 * (size_t)a0;
  const uint32_t *tm = b.atom_tmask + a0;
  const uint16_t *hl = b.heavy_list + a0;
  VS_KCHECK(m <= VS_MAX_TORSIONS && n <= N && N <= VS_MAX_ATOMS);
  if (lane == 0)
    for (int t = 0; t < m; ++t) {
      const int ia = b.tors_a[t0 + t], ib = b.tors_b[t0 + t];
      VS_KCHECK(ia < N && ib < N);
      d3 pa = ld3(base + 3 * ia), pb = ld3(base + 3 * ib);
      const uint32_t ma = tm[ia], mb = tm[ib];
      for (int w = 0; w < t; ++w) {
        if ((ma >> w) & 1u) pa = torsion_apply(M + 12 * w, pa);
        if ((mb >> w) & 1u) pb = torsion_apply(M + 12 * w, pb);
      }
      double sn, cs;
      vs_crtrig::sincos_cr(ang[t], &sn, &cs);
      torsion_setup(pa, pb, sn, cs, M + 12 * t);  // k_search built this axis: not degenerate
    }
  __syncwarp();
  double R[9];
  quat_matrix(quat{T7[0], T7[1], T7[2], T7[3]}, R);
  const double tr[3] = {T7[4], T7[5], T7[6]};
  for (int h = lane; h < n; h += 32) st3(out + 3 * (size_t)hl[h], ld3(hc + 3 * h));
  for (int a = lane; a < N; a += 32) {
    if (b.heavy[a0 + a]) continue;
    d3 x = ld3(base + 3 * a);
    for (uint32_t bb = tm[a]; bb; bb &= bb - 1u) x = torsion_apply(M + 12 * (__ffs(bb) - 1), x);
    st3(out + 3 * (size_t)a, rigid_col(R, tr, x, a));
  }
}

__device__ __forceinline__ int f_sweeps_of(const dock_out &d, int l) { return d.sweeps ? d.sweeps[l] : 0; }

// ============================================================== k_select
// cluster_and_select + chem_score + best (search.cpp:195-275).  One CTA per
// ligand.
constexpr int kSelThreads = 128;

// Per-ligand select state (ints): order, leaders, followers (3k), chem
// (k doubles, 8-byte aligned), clash, pairs (2k).
__host__ __device__ inline size_t select_state_ints(int k) { return (size_t)3 * k + (k & 1) + 2 + 2 * (size_t)k + 2 * k + 4; }

__global__ void __launch_bounds__(kSelThreads) k_select(batch_dev b, pocket_dev p, search_cfg c, item_out o, dock_out d,
                                                        int *gs) {
  extern __shared__ int sdyn[];
  const int l = blockIdx.x, tid = threadIdx.x;
  const int k = c.k;
  // shared memory, or a per-ligand slice of global scratch for restart
  // counts whose state exceeds it
  int *si = gs ? gs + select_state_ints(k) * (size_t)l : sdyn;
  int *order = si;            // k
  int *leaders = order + k;   // k
  int *followers = leaders + k;
  double *chem = reinterpret_cast<double *>(followers + k + (k & 1) + 2);  // rescored
  int *clash = reinterpret_cast<int *>(chem + k);
  int *pairs = clash + k;
  __shared__ int n_lead, n_follow, status, first_match;
  __shared__ unsigned long long rmsd_terms;
  vs_dock_result *res = reinterpret_cast<vs_dock_result *>(d.results) + l;
  lig_meta meta = b.meta[l];
  if (tid == 0) {
    status = meta.status;
    n_lead = 0;
    n_follow = 0;
    rmsd_terms = 0ull;
  }
  __syncthreads();
  if (status == VS_LIG_OK)
    for (int r = tid; r < k; r += blockDim.x)
      if (o.status[(size_t)l * k + r] != VS_LIG_OK) atomicMax(&status, o.status[(size_t)l * k + r]);
  __syncthreads();
  if (status != VS_LIG_OK) {
    if (tid == 0) {
      vs_dock_result z{};
      z.status = status;
      *res = z;
      if (d.best_idx) d.best_idx[l] = -1;
    }
    return;
  }
  const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const uint16_t *hl = b.heavy_list + a0;
  const double *geo = o.geo + (size_t)l * k;
  const double *confs = o.conf + 3 * (size_t)a0 * k;  // pose r at + 3*r*N, heavy atoms compact
  // stable sort by descending geo_score (search.cpp:201-206)
  for (int i = tid; i < k; i += blockDim.x) {
    const double gi = geo[i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double gj = geo[j];
      rank += (gj > gi || (gj == gi && j < i)) ? 1 : 0;
    }
    order[rank] = i;
  }
  __syncthreads();
  // greedy leader clustering (search.cpp:208-223)
  for (int vi = 0; vi < k; ++vi) {
    const int idx = order[vi];
    if (tid == 0) first_match = 0x7fffffff;
    __syncthreads();
    const int nl = n_lead;
    const double *ci = confs + 3 * (size_t)idx * N;
    for (int li = tid; li < nl; li += blockDim.x) {
      const double *cl = confs + 3 * (size_t)leaders[li] * N;
      double sum = 0.0;
      for (int h = 0; h < n; ++h) sum += sqn3(sub3(ld3(ci + 3 * h), ld3(cl + 3 * h)));
      if (dsqrt(sum / (double)n) <= c.rmsd_threshold) atomicMin(&first_match, li);
    }
    __syncthreads();
    if (tid == 0) {
      // the reference stops at the first leader within threshold
      rmsd_terms += (unsigned long long)n * (first_match != 0x7fffffff ? first_match + 1 : nl);
      if (first_match != 0x7fffffff)
        followers[n_follow++] = idx;
      else
        leaders[n_lead++] = idx;
    }
    __syncthreads();
  }
  const int top = c.rescored < k ? c.rescored : k;
  // survivors: leaders then followers, truncated (search.cpp:225-235)
  for (int s = tid; s < top; s += blockDim.x) {
    const int idx = s < n_lead ? leaders[s] : followers[s - n_lead];
    int cl = 0, pr = 0;
    chem[s] = chem_pose(p, confs + 3 * (size_t)idx * N, hl, b.elem + a0, n, cl, pr);
    clash[s] = cl;
    pairs[s] = pr;
  }
  __syncthreads();
  __shared__ int best_s;
  if (tid == 0) {
    int best = 0;
    double bc = -__longlong_as_double(0x7ff0000000000000LL);
    for (int s = 0; s < top; ++s)
      if (chem[s] > bc) {
        bc = chem[s];
        best = s;
      }
    best_s = best;
  }
  __syncthreads();
  const int bs = best_s;
  const int bidx = bs < n_lead ? leaders[bs] : followers[bs - n_lead];
  const double *bconf = confs + 3 * (size_t)bidx * N;
  if (tid == 0 && d.best_idx) d.best_idx[l] = bidx;
  if (d.best_ang)
    for (int u = tid; u < m; u += blockDim.x) d.best_ang[t0 + u] = o.ang[(size_t)t0 * k + (size_t)bidx * m + u];
  __shared__ int oob;
  if (tid == 0) oob = 0;
  __syncthreads();
  for (int h = tid; h < n; h += blockDim.x) {
    bool out;
    field_value(p.g, ld3(bconf + 3 * h), out);
    if (out) atomicAdd(&oob, 1);
  }
  __syncthreads();
  if (tid == 0) {
    vs_dock_result rr{};
    const double best = chem[bs];
    rr.status = isfinite(best) ? VS_LIG_OK : VS_LIG_NONFINITE;
    rr.n_survivors = top;
    rr.best_score = best;
    const size_t item = (size_t)l * k + bidx;
    rr.best_geo_score = o.geo[item];
    for (int q = 0; q < 4; ++q) rr.rotation[q] = o.T[7 * item + q];
    for (int q = 0; q < 3; ++q) rr.translation[q] = o.T[7 * item + 4 + q];
    rr.poses_evaluated = (uint64_t)k;
    unsigned long long ev = 0;
    for (int r = 0; r < k; ++r) ev += o.evals[(size_t)l * k + r];
    rr.scoring_evals = ev;
    rr.clash_pairs = clash[bs];
    rr.oob_samples = oob;
    *res = rr;
    if (d.counters) {
      // Appendix B counter model, reproduced from the run's integers.
      unsigned long long iters = 0, adopts = 0, pchem = 0;
      for (int r = 0; r < k; ++r) {
        iters += (unsigned long long)o.iters[(size_t)l * k + r];
        adopts += (unsigned long long)o.adopts[(size_t)l * k + r];
      }
      for (int s = 0; s < top; ++s) pchem += (unsigned long long)pairs[s];
      const unsigned long long NN = N, nn = n, mm = m, kk = k, J = 12 + 2 * mm;
      const unsigned long long cand = 36ull * mm * (unsigned long long)f_sweeps_of(d, l);
      unsigned long long *cn = d.counters + 9 * (size_t)l;
      cn[0] = ev;
      cn[1] = kk * NN + iters * J * nn + adopts * NN;
      cn[2] = cand * (unsigned long long)meta.r_all + iters * 2ull * mm * (unsigned long long)meta.r_heavy;
      cn[3] = cand * mm + 2ull * mm + kk * mm + iters * 2ull * mm * mm;
      cn[4] = cand * (NN * (NN - 1) / 2);
      cn[5] = pchem;
      cn[6] = rmsd_terms;
      cn[7] = (unsigned long long)clash[bs];
      cn[8] = (unsigned long long)oob;
    }
  }
}

// The same for k <= 32 restarts with one warp per ligand (lane = restart /
// leader / survivor): no CTA barriers, 4 independent ligands per CTA.
#ifndef VS_SEL_WARPS
#define VS_SEL_WARPS 4
#endif
constexpr int kSelWarps = VS_SEL_WARPS;  // ligands (warps) per select CTA
#ifndef VS_SEL_UNROLL
#define VS_SEL_UNROLL 8  // RMSD loads in flight (measured: 1 and 4 -> 20.6 ms, 8 -> 19.7 ms select per step)
#endif
constexpr int kSelUnroll = VS_SEL_UNROLL;

__global__ void __launch_bounds__(32 * kSelWarps) k_select_warp(batch_dev b, pocket_dev p, search_cfg c, item_out o,
                                                               dock_out d) {
  __shared__ int s_order[kSelWarps][32], s_lead[kSelWarps][32], s_foll[kSelWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int l = blockIdx.x * kSelWarps + w;
  if (l >= b.n_lig) return;
  const int k = c.k;
  int *order = s_order[w], *leaders = s_lead[w], *followers = s_foll[w];
  vs_dock_result *res = reinterpret_cast<vs_dock_result *>(d.results) + l;
  const lig_meta meta = b.meta[l];
  int status = meta.status;
  if (status == VS_LIG_OK) {
    const int st = lane < k ? o.status[(size_t)l * k + lane] : VS_LIG_OK;
    status = __reduce_max_sync(0xffffffffu, st);
  }
  if (status != VS_LIG_OK) {
    if (lane == 0) {
      vs_dock_result z{};
      z.status = status;
      *res = z;
      if (d.best_idx) d.best_idx[l] = -1;
    }
    return;
  }
  const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const uint16_t *hl = b.heavy_list + a0;
  const double *geo = o.geo + (size_t)l * k;
  const double *confs = o.conf + 3 * (size_t)a0 * k;  // pose r at + 3*r*N, heavy atoms compact
  // stable sort by descending geo_score (search.cpp:201-206)
  if (lane < k) {
    const double gi = geo[lane];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double gj = geo[j];
      rank += (gj > gi || (gj == gi && j < lane)) ? 1 : 0;
    }
    order[rank] = lane;
  }
  __syncwarp();
  // greedy leader clustering (search.cpp:208-223): lane li tests leader li
  int n_lead = 0, n_follow = 0;
  unsigned long long rmsd_terms = 0ull;
  #pragma unroll 1
  for (int vi = 0; vi < k; ++vi) {
    const int idx = order[vi];
    const double *ci = confs + 3 * (size_t)idx * N;
    bool match = false;
    if (lane < n_lead) {
      const double *cl = confs + 3 * (size_t)leaders[lane] * N;
      double sum = 0.0;
      // unrolled: the L2 loads of several atoms are in flight ahead of the
      // sequential sum (whose order is unchanged)
      #pragma unroll kSelUnroll
      for (int h = 0; h < n; ++h) sum += sqn3(sub3(ld3(ci + 3 * h), ld3(cl + 3 * h)));
      match = dsqrt(sum / (double)n) <= c.rmsd_threshold;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, match);
    // the reference stops at the first leader within threshold
    rmsd_terms += (unsigned long long)n * (bal ? (unsigned)__ffs(bal) : (unsigned)n_lead);
    if (lane == 0) {
      if (bal)
        followers[n_follow] = idx;
      else
        leaders[n_lead] = idx;
    }
    if (bal) ++n_follow;
    else ++n_lead;
    __syncwarp();
  }
  const int top = c.rescored < k ? c.rescored : k;
  // survivors: leaders then followers, truncated (search.cpp:225-235)
  double chem = -__longlong_as_double(0x7ff0000000000000LL);
  int clash = 0, pairs = 0;
  if (lane < top) {
    const int idx = lane < n_lead ? leaders[lane] : followers[lane - n_lead];
    chem = chem_pose(p, confs + 3 * (size_t)idx * N, hl, b.elem + a0, n, clash, pairs);
  }
  // strict argmax, first survivor on ties (search.cpp:255-265); NaN never
  // beats anything, as in the sequential `chem > best` scan
  double bc = isnan(chem) ? -__longlong_as_double(0x7ff0000000000000LL) : chem;
  int bs = lane < top ? lane : 0x7fffffff;
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bc, off);
    const int os = __shfl_xor_sync(0xffffffffu, bs, off);
    if (ov > bc || (ov == bc && os < bs)) {
      bc = ov;
      bs = os;
    }
  }
  if (!(bc > -__longlong_as_double(0x7ff0000000000000LL))) bs = 0;  // all -inf/nan: the first survivor
  const int best_clash = __shfl_sync(0xffffffffu, clash, bs & 31);
  const double best = __shfl_sync(0xffffffffu, chem, bs & 31);
  unsigned long long pchem = lane < top ? (unsigned long long)pairs : 0ull;
  for (int off = 16; off > 0; off >>= 1) pchem += __shfl_xor_sync(0xffffffffu, pchem, off);
  const int bidx = bs < n_lead ? leaders[bs] : followers[bs - n_lead];
  const double *bconf = confs + 3 * (size_t)bidx * N;
  if (lane == 0 && d.best_idx) d.best_idx[l] = bidx;
  if (d.best_ang)
    for (int u = lane; u < m; u += 32) d.best_ang[t0 + u] = o.ang[(size_t)t0 * k + (size_t)bidx * m + u];
  int oob = 0;
  for (int h = lane; h < n; h += 32) {
    bool out;
    field_value(p.g, ld3(bconf + 3 * h), out);
    oob += out ? 1 : 0;
  }
  oob = __reduce_add_sync(0xffffffffu, oob);
  unsigned long long ev = lane < k ? o.evals[(size_t)l * k + lane] : 0ull;
  unsigned long long iters = lane < k && o.iters ? (unsigned long long)o.iters[(size_t)l * k + lane] : 0ull;
  unsigned long long adopts = lane < k && o.adopts ? (unsigned long long)o.adopts[(size_t)l * k + lane] : 0ull;
  for (int off = 16; off > 0; off >>= 1) {
    ev += __shfl_xor_sync(0xffffffffu, ev, off);
    iters += __shfl_xor_sync(0xffffffffu, iters, off);
    adopts += __shfl_xor_sync(0xffffffffu, adopts, off);
  }
  if (lane == 0) {
    vs_dock_result rr{};
    rr.status = isfinite(best) ? VS_LIG_OK : VS_LIG_NONFINITE;
    rr.n_survivors = top;
    rr.best_score = best;
    const size_t item = (size_t)l * k + bidx;
    rr.best_geo_score = o.geo[item];
    for (int q = 0; q < 4; ++q) rr.rotation[q] = o.T[7 * item + q];
    for (int q = 0; q < 3; ++q) rr.translation[q] = o.T[7 * item + 4 + q];
    rr.poses_evaluated = (uint64_t)k;
    rr.scoring_evals = ev;
    rr.clash_pairs = best_clash;
    rr.oob_samples = oob;
    *res = rr;
    if (d.counters) {
      // Appendix B counter model, reproduced from the run's integers.
      const unsigned long long NN = N, nn = n, mm = m, kk = k, J = 12 + 2 * mm;
      const unsigned long long cand = 36ull * mm * (unsigned long long)f_sweeps_of(d, l);
      unsigned long long *cn = d.counters + 9 * (size_t)l;
      cn[0] = ev;
      cn[1] = kk * NN + iters * J * nn + adopts * NN;
      cn[2] = cand * (unsigned long long)meta.r_all + iters * 2ull * mm * (unsigned long long)meta.r_heavy;
      cn[3] = cand * mm + 2ull * mm + kk * mm + iters * 2ull * mm * mm;
      cn[4] = cand * (NN * (NN - 1) / 2);
      cn[5] = pchem;
      cn[6] = rmsd_terms;
      cn[7] = (unsigned long long)best_clash;
      cn[8] = (unsigned long long)oob;
    }
  }
}

// The best pose's full conformation (best_conformation), one warp per ligand,
// after the select (its own kernel: the rematerialisation's registers would
// halve the select's occupancy).
__global__ void __launch_bounds__(32 * kSelWarps) k_best_conf(batch_dev b, search_cfg c, item_out o, dock_out d) {
  __shared__ double s_M[kSelWarps][12 * VS_MAX_TORSIONS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int l = blockIdx.x * kSelWarps + w;
  if (l >= b.n_lig) return;
  const int bidx = d.best_idx[l];
  if (bidx < 0) return;
  VS_KCHECK(bidx < c.k);
  const int k = c.k, m = b.meta[l].m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const size_t item = (size_t)l * k + bidx;
  best_conformation(b, l, o.conf + 3 * ((size_t)a0 * k + (size_t)bidx * b.meta[l].n_atoms),
                    o.ang + (size_t)t0 * k + (size_t)bidx * m, o.T + 7 * item, s_M[w], d.best_conf + 3 * (size_t)a0,
                    lane);
}

constexpr size_t kSelSmemMax = 160 * 1024;

size_t select_scratch_bytes(int n_lig, int k) {
  return k > 32 && select_state_ints(k) * sizeof(int) > kSelSmemMax
             ? select_state_ints(k) * sizeof(int) * (size_t)(n_lig > 0 ? n_lig : 1)
             : 0;
}

cudaError_t launch_select(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const item_out &o,
                          const dock_out &d, int nmax_atoms, cudaStream_t s, int *sel_scratch) {
  (void)nmax_atoms;
  if (b.n_lig == 0) return cudaSuccess;
  if (!o.heavy_conf) return cudaErrorInvalidValue;  // the selects read compact heavy-atom conformations
  const int k = c.k;
  if (d.best_conf && !d.best_idx) return cudaErrorInvalidValue;
  if (k <= 32) {
    k_select_warp<<<(b.n_lig + kSelWarps - 1) / kSelWarps, 32 * kSelWarps, 0, s>>>(b, p, c, o, d);
  } else if (select_state_ints(k) * sizeof(int) <= kSelSmemMax) {
    const size_t smem = select_state_ints(k) * sizeof(int);
    std::lock_guard<std::mutex> lock(launch_mutex());
    cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_select<<<b.n_lig, kSelThreads, smem, s>>>(b, p, c, o, d, nullptr);
  } else {
    if (!sel_scratch) return cudaErrorInvalidValue;  // select_scratch_bytes of global scratch
    k_select<<<b.n_lig, kSelThreads, 0, s>>>(b, p, c, o, d, sel_scratch);
  }
  if (d.best_conf) k_best_conf<<<(b.n_lig + kSelWarps - 1) / kSelWarps, 32 * kSelWarps, 0, s>>>(b, c, o, d);
  return cudaGetLastError();
}

// cluster_and_select (search.cpp:195-236) of np given poses of ligand 0:
// one CTA, the same greedy leader rule as k_select.
__global__ void __launch_bounds__(kSelThreads) k_cluster(batch_dev b, int np, const double *geo, const double *confs,
                                                         double threshold, int top, int *order_out, int *count_out) {
  extern __shared__ int ci[];
  int *order = ci, *leaders = ci + np, *followers = ci + 2 * np;
  __shared__ int n_lead, n_follow, joined;
  const int tid = threadIdx.x;
  const lig_meta meta = b.meta[0];
  const int N = meta.n_atoms, n = meta.n_heavy;
  const uint16_t *hl = b.heavy_list;
  if (tid == 0) {
    n_lead = 0;
    n_follow = 0;
  }
  for (int i = tid; i < np; i += blockDim.x) {
    const double gi = geo[i];
    int rank = 0;
    for (int j = 0; j < np; ++j) rank += (geo[j] > gi || (geo[j] == gi && j < i)) ? 1 : 0;
    order[rank] = i;
  }
  __syncthreads();
  for (int vi = 0; vi < np; ++vi) {
    const int idx = order[vi];
    if (tid == 0) joined = 0;
    __syncthreads();
    const int nl = n_lead;
    for (int li = tid; li < nl; li += blockDim.x) {
      double sum = 0.0;
      for (int h = 0; h < n; ++h) {
        const int a = hl[h];
        sum += sqn3(sub3(ld3(confs + 3 * ((size_t)idx * N + a)), ld3(confs + 3 * ((size_t)leaders[li] * N + a))));
      }
      if (dsqrt(sum / (double)n) <= threshold) joined = 1;
    }
    __syncthreads();
    if (tid == 0) {
      if (joined)
        followers[n_follow++] = idx;
      else
        leaders[n_lead++] = idx;
    }
    __syncthreads();
  }
  const int cnt = top < np ? top : np;
  for (int s = tid; s < cnt; s += blockDim.x) order_out[s] = s < n_lead ? leaders[s] : followers[s - n_lead];
  if (tid == 0) *count_out = cnt;
}

cudaError_t launch_cluster(const batch_dev &b, int np, const double *geo, const double *confs, double threshold,
                           int top, int *order_out, int *count_out, cudaStream_t s) {
  const size_t smem = sizeof(int) * 3 * (size_t)np;
  std::lock_guard<std::mutex> lock(launch_mutex());
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cluster<<<1, kSelThreads, smem, s>>>(b, np, geo, confs, threshold, top, order_out, count_out);
  return cudaGetLastError();
}

// ============================================================== sub-APIs
__global__ void k_field(pocket_dev p, int64_t n, const double *xyz, double *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool o;
  out[i] = field_value(p.g, ld3(xyz + 3 * i), o);
}
cudaError_t launch_field_values(const pocket_dev &p, int64_t n, const double *xyz, double *out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_field<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, xyz, out);
  return cudaGetLastError();
}

// geo_score (grid.cpp:93-104): warp per ligand, lanes sample, lane 0 sums
// in heavy-atom order.
__global__ void k_geo(batch_dev b, pocket_dev p, const double *conf, double *out, unsigned long long *evals) {
  __shared__ double vals[4][VS_MAX_HEAVY];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.x * 4 + warp;
  if (l >= b.n_lig) return;
  const lig_meta meta = b.meta[l];
  const int a0 = b.atom_off[l];
  const int n = meta.status == VS_LIG_OK || meta.status == VS_LIG_NO_HEAVY ? meta.n_heavy : 0;
  for (int h = lane; h < n; h += 32) {
    bool o;
    const int a = b.heavy_list[a0 + h];
    vals[warp][h] = field_value(p.g, ld3(conf + 3 * ((size_t)a0 + a)), o);
  }
  __syncwarp();
  if (lane == 0) {
    double acc = 0.0;
    for (int h = 0; h < n; ++h) acc += vals[warp][h];
    out[l] = acc;
    if (evals) evals[l] = (unsigned long long)n;
  }
}
cudaError_t launch_geo_score(const batch_dev &b, const pocket_dev &p, const double *conf, double *out,
                             unsigned long long *evals, cudaStream_t s) {
  if (b.n_lig == 0) return cudaSuccess;
  k_geo<<<(b.n_lig + 3) / 4, 128, 0, s>>>(b, p, conf, out, evals);
  return cudaGetLastError();
}

__global__ void k_chem(batch_dev b, pocket_dev p, const double *conf, double *out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= b.n_lig) return;
  const lig_meta meta = b.meta[l];
  const int a0 = b.atom_off[l];
  const int n = meta.status == VS_LIG_OK || meta.status == VS_LIG_NO_HEAVY ? meta.n_heavy : 0;
  int cl = 0, pr = 0;
  out[l] = chem_pose(p, conf + 3 * (size_t)a0, b.heavy_list + a0, b.elem + a0, n, cl, pr);
}
cudaError_t launch_chem_score(const batch_dev &b, const pocket_dev &p, const double *conf, double *out,
                              cudaStream_t s) {
  if (b.n_lig == 0) return cudaSuccess;
  k_chem<<<(b.n_lig + 63) / 64, 64, 0, s>>>(b, p, conf, out);
  return cudaGetLastError();
}

// build_pocket (grid.cpp:15-57): per node, min squared distance to the
// protein heavy atoms (min is order-independent, so the tiled parallel scan
// is exact), then the three-way classification.
__global__ void k_build_pocket(const double *hxyz, int nh, double cx, double cy, double cz, double radius, double ox,
                               double oy, double oz, double h, int d0, int d1, int d2, double *values) {
  __shared__ double tile[3 * 256];
  const int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)d0 * d1 * d2;
  int ix = 0, iy = 0, iz = 0;
  if (node < total) {
    ix = (int)(node % d0);
    iy = (int)((node / d0) % d1);
    iz = (int)(node / ((int64_t)d0 * d1));
  }
  // node_position = origin + spacing * (ix, iy, iz) (pocket.hpp:48-50)
  const d3 x{ox + h * (double)ix, oy + h * (double)iy, oz + h * (double)iz};
  double d2min = __longlong_as_double(0x7ff0000000000000LL);
  for (int base = 0; base < nh; base += 256) {
    const int cnt = min(256, nh - base);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * cnt; i += blockDim.x) tile[i] = hxyz[3 * base + i];
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const double q = sqn3(sub3(x, ld3(tile + 3 * j)));
      d2min = q < d2min ? q : d2min;  // std::min(d2, q)
    }
  }
  if (node >= total) return;
  const double dist = sqrt(d2min);
  double v = 0.0;
  if (dist < 1.5)
    v = -10.0;
  else if (dist <= 4.0 && sqrt(sqn3(sub3(x, d3{cx, cy, cz}))) <= radius)
    v = 1.0;
  values[node] = v;
}
cudaError_t launch_build_pocket(const double *hxyz, int nh, double cx, double cy, double cz, double radius,
                                double ox, double oy, double oz, double h, int d0, int d1, int d2, double *values,
                                cudaStream_t s) {
  const int64_t total = (int64_t)d0 * d1 * d2;
  k_build_pocket<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(hxyz, nh, cx, cy, cz, radius, ox, oy, oz, h, d0, d1,
                                                                 d2, values);
  return cudaGetLastError();
}

// Load this translation unit's kernels on the current device at context
// creation rather than at the first launch (keeps module loading out of the
// CUDA workers' concurrent first launches).
void preload_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_setup);
  cudaFuncGetAttributes(&a, k_flatten);
  cudaFuncGetAttributes(&a, k_flatten_dep);
  cudaFuncGetAttributes(&a, k_select);
  cudaFuncGetAttributes(&a, k_select_warp);
  cudaFuncGetAttributes(&a, k_cluster);
  cudaFuncGetAttributes(&a, k_field);
  cudaFuncGetAttributes(&a, k_geo);
  cudaFuncGetAttributes(&a, k_chem);
  cudaFuncGetAttributes(&a, k_build_pocket);
  preload_kernels_search();
  preload_kernels_codec();
}

}  // namespace vsd

