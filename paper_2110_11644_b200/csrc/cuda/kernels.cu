// sm_100a kernels of the batched dock-and-score path.
//
//   k_setup        per ligand: validation, heavy-atom list, right-set masks,
//                  torsion dependency closures D_t (thread per ligand)
//   k_flatten      flatten (search.cpp:27-69): CTA per ligand, one thread
//                  per 10-degree candidate, sequential distance sums
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

#include "../../../include/vs_crtrig.h"
#include "../../../include/vs_dock.h"
#include "kernels.cuh"

namespace vsd {

// CR sin/cos of the 36 flatten lattice angles idx * (2 pi / 36)
// (search.cpp:33,40), computed on the host with vs_crtrig.
__constant__ double c_lattice_sc[72];
constexpr double kPi = 3.14159265358979323846;
constexpr double kLatticeStep = 2.0 * kPi / 36;

void set_lattice_table(const double *sc72) { cudaMemcpyToSymbol(c_lattice_sc, sc72, sizeof(double) * 72); }

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
  lig_meta meta{N, 0, m, VS_LIG_OK, 0, 0};
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
  // Heavy index of each torsion endpoint (the search tracks heavy atoms).
  for (int t = 0; t < m; ++t) {
    const int bi = b.tors_bond[t0 + t];
    const int ea = b.bond_a[b0 + bi], eb = b.bond_b[b0 + bi];
    int ha = -1, hb = -1;
    for (int h = 0; h < n; ++h) {
      if (b.heavy_list[a0 + h] == ea) ha = h;
      if (b.heavy_list[a0 + h] == eb) hb = h;
    }
    if (ha < 0 || hb < 0) {  // hydrogen torsion endpoint: not produced by detect_torsions
      meta.status = VS_LIG_TOO_LARGE;
      b.meta[l] = meta;
      return;
    }
    b.tors_ha[t0 + t] = (uint16_t)ha;
    b.tors_hb[t0 + t] = (uint16_t)hb;
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
      const int ea = b.heavy_list[a0 + b.tors_ha[t0 + u]], eb = b.heavy_list[a0 + b.tors_hb[t0 + u]];
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
    b.d_count[t0 + t] = cnt;
    b.d_off[t0 + t] = off;
    off += cnt;
  }
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

__device__ __forceinline__ void lattice_sc(int idx, double &s, double &c) {
  s = c_lattice_sc[2 * idx];
  c = c_lattice_sc[2 * idx + 1];
}

__global__ void __launch_bounds__(kFlatThreads) k_flatten(batch_dev b, int max_sweeps, flat_out f, int cand_per_round) {
  extern __shared__ double sm[];
  const int l = blockIdx.x;
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
            for (; j + 3 < N; j += 4) {
              double d[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const d3 xj{C[(3 * (j + q)) * CB], C[(3 * (j + q) + 1) * CB], C[(3 * (j + q) + 2) * CB]};
                d[q] = sqrt(sqn3(sub3(xi, xj)));
              }
              sum += d[0];
              sum += d[1];
              sum += d[2];
              sum += d[3];
            }
            for (; j < N; ++j) {
              const d3 xj{C[(3 * j) * CB], C[(3 * j + 1) * CB], C[(3 * j + 2) * CB]};
              sum += sqrt(sqn3(sub3(xi, xj)));
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

cudaError_t launch_flatten(const batch_dev &b, int max_sweeps, const flat_out &f, int nmax_atoms, int mmax,
                           cudaStream_t s) {
  if (b.n_lig == 0) return cudaSuccess;
  (void)mmax;
  int cb = 36;
  auto bytes = [&](int c) { return (size_t)(3 * nmax_atoms * (1 + c) + 36 + 12) * sizeof(double); };
  while (cb > 1 && bytes(cb) > 200 * 1024) cb = (cb + 1) / 2;
  const size_t smem = bytes(cb);
  cudaFuncSetAttribute(k_flatten, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_flatten<<<b.n_lig, kFlatThreads, smem, s>>>(b, max_sweeps, f, cb);
  return cudaGetLastError();
}

// ============================================================== k_search
// One warp per (ligand, restart).  Per-warp shared memory (doubles):
//   conf[N*3]  current pose, all atoms (pivot = its centroid)
//   tors[N*3]  torsioned, untransformed frame (search.cpp:115)
//   P[m*n*3]   heavy-atom prefix states: P_t = atoms before torsion t
//   Mcur[m*12] current torsion matrices {R, pivot}
//   Mvar[2m*m*12] torsion-neighbour matrices (only u >= t used)
//   Rj[12*16]  rigid neighbours {R, t, q}
//   vb[J*n]    per-neighbour, per-heavy-atom field values
//   vcur[n]    field values of the current pose
//   scores[J], cache[2m*2] (sin,cos of cur +- step), ang[m], sccur[m*2]
//   state[32]  q, t, R, pivot, geo, steps
//   dm[n] (u32), cvalid[2m] (int)
struct search_args {
  batch_dev b;
  pocket_dev p;
  search_cfg c;
  flat_out f;
  item_out o;
  const double *pose_in;   // local_search mode: [items][8] q,t,geo; NULL in dock mode
  const double *ang_in;    // local_search mode: per torsion
  const double *conf_in;   // local_search mode: 3*atoms
  int *work;
  int n_items;
  int Nmax, nmax, mmax, Jmax;
  int warp_doubles;
  int o_conf, o_tors, o_P, o_Mcur, o_Mvar, o_Rj, o_vb, o_vcur, o_scores, o_cache, o_ang, o_sccur, o_state, o_dm,
      o_cvalid;
};

enum { S_Q = 0, S_T = 4, S_R = 7, S_PIV = 16, S_GEO = 19, S_STEPT = 20, S_STEPR = 21, S_STEPQ = 22, S_ERR = 23, S_N = 24 };

// Matrices of torsions u = t..m-1 for a pose whose angles equal the current
// ones except torsion t (sin/cos st/ct): each endpoint is carried from the
// prefix P_t through the already-built rotations (per-atom composition of
// apply_torsions, transform.cpp:73-81).  Single lane.
__device__ bool chain_mats(int t, double st, double ct, int m, const double *P, int nmax, const uint16_t *ha,
                           const uint16_t *hb, const uint16_t *hl, const uint32_t *tm, const double *sccur, double *out) {
  for (int u = t; u < m; ++u) {
    const int hA = ha[u], hB = hb[u];
    d3 ea = ld3(P + 3 * (t * nmax + hA));
    d3 eb = ld3(P + 3 * (t * nmax + hB));
    const uint32_t ma = tm[hl[hA]], mb = tm[hl[hB]];
    for (int w = t; w < u; ++w) {
      if ((ma >> w) & 1u) ea = torsion_apply(out + 12 * w, ea);
      if ((mb >> w) & 1u) eb = torsion_apply(out + 12 * w, eb);
    }
    const double s = u == t ? st : sccur[2 * u];
    const double c = u == t ? ct : sccur[2 * u + 1];
    if (!torsion_setup(ea, eb, s, c, out + 12 * u)) return false;
  }
  return true;
}

// Rebuild P (heavy prefixes) and tors (all atoms) from the base coordinates
// with the current matrices Mcur.  Warp-cooperative over atoms.
__device__ __forceinline__ void rebuild_frames(int lane, int N, int m, int nmax, const double *base, const uint8_t *heavy,
                                               const uint32_t *tm, const double *Mcur, double *P, double *tors,
                                               const int *heavy_index) {
  for (int a = lane; a < N; a += 32) {
    d3 x = ld3(base + 3 * a);
    const int h = heavy_index[a];
    const uint32_t mask = tm[a];
    for (int u = 0; u < m; ++u) {
      if (h >= 0) st3(P + 3 * (u * nmax + h), x);
      if ((mask >> u) & 1u) x = torsion_apply(Mcur + 12 * u, x);
    }
    st3(tors + 3 * a, x);
  }
  (void)heavy;
}

__global__ void __launch_bounds__(128) k_search(search_args A) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double *W = sm + (size_t)warp * A.warp_doubles;
  double *conf = W + A.o_conf;
  double *tors = W + A.o_tors;
  double *P = W + A.o_P;
  double *Mcur = W + A.o_Mcur;
  double *Mvar = W + A.o_Mvar;
  double *Rj = W + A.o_Rj;
  double *vb = W + A.o_vb;
  double *vcur = W + A.o_vcur;
  double *scores = W + A.o_scores;
  double *cache = W + A.o_cache;
  double *ang = W + A.o_ang;
  double *sccur = W + A.o_sccur;
  double *S = W + A.o_state;
  uint32_t *dm = reinterpret_cast<uint32_t *>(W + A.o_dm);
  int *cvalid = reinterpret_cast<int *>(W + A.o_cvalid);
  // heavy index of each atom (-1 for hydrogens) lives after cvalid
  int *hidx = cvalid + 2 * A.mmax + 2;

  const batch_dev &b = A.b;
  const grid_view &g = A.p.g;
  const int k = A.pose_in ? 1 : A.c.k;
  const int nmax = A.nmax;

  while (true) {
    int item = 0;
    if (lane == 0) item = atomicAdd(A.work, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= A.n_items) break;
    const int l = item / k, r = item - l * k;
    const lig_meta meta = b.meta[l];
    if (meta.status != VS_LIG_OK) {
      if (lane == 0) A.o.status[item] = meta.status;
      continue;
    }
    const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
    const int a0 = b.atom_off[l], t0 = b.tors_off[l];
    const double *base = b.xyz + 3 * (size_t)a0;
    const uint16_t *hl = b.heavy_list + a0;
    const uint32_t *tm = b.atom_tmask + a0;
    const uint16_t *ha = b.tors_ha + t0, *hb = b.tors_hb + t0;
    const int *dcnt = b.d_count + t0, *doff = b.d_off + t0;
    const uint16_t *ditems = b.ditems + b.ditem_base[l];
    const int J = 12 + 2 * m;
    unsigned long long evals = 0;

    // ---- per-ligand tables into shared memory
    for (int a = lane; a < N; a += 32) hidx[a] = -1;
    __syncwarp();
    for (int h = lane; h < n; h += 32) {
      hidx[hl[h]] = h;
      dm[h] = b.heavy_dmask[a0 + h];
    }
    for (int v = lane; v < 2 * m; v += 32) cvalid[v] = 0;
    if (A.pose_in) {
      for (int u = lane; u < m; u += 32) {
        ang[u] = A.ang_in[t0 + u];
        vs_crtrig::sincos_cr(ang[u], &sccur[2 * u], &sccur[2 * u + 1]);
      }
    } else {
      for (int u = lane; u < m; u += 32) {
        const int li = A.f.idx[t0 + u];
        ang[u] = li * kLatticeStep;
        sccur[2 * u] = c_lattice_sc[2 * li];
        sccur[2 * u + 1] = c_lattice_sc[2 * li + 1];
      }
    }
    for (int h = lane; h < n; h += 32) st3(P + 3 * h, ld3(base + 3 * hl[h]));  // P_0 = base
    __syncwarp();
    if (lane == 0) {
      S[S_ERR] = 0.0;
      if (m > 0 && !chain_mats(0, sccur[0], sccur[1], m, P, nmax, ha, hb, hl, tm, sccur, Mcur)) S[S_ERR] = 1.0;
    }
    __syncwarp();
    if (S[S_ERR] != 0.0) {
      if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
      continue;
    }
    rebuild_frames(lane, N, m, nmax, base, nullptr, tm, Mcur, P, tors, hidx);
    __syncwarp();

    // ---- initial pose (initial_poses, search.cpp:95-103) or the given one
    if (lane == 0) {
      quat q;
      double t[3];
      if (A.pose_in) {
        const double *pi = A.pose_in + 8 * l;
        q = {pi[0], pi[1], pi[2], pi[3]};
        t[0] = pi[4];
        t[1] = pi[5];
        t[2] = pi[6];
      } else {
        const double *fq = A.c.fibq + 4 * r;
        q = {fq[0], fq[1], fq[2], fq[3]};
        const d3 fc = ld3(A.f.centroid + 3 * l);
        const d3 rc = quat_rotate(q, fc);
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
    }
    __syncwarp();
    // current-pose sample values from apply_rigid(tors, T)
    for (int h = lane; h < n; h += 32) {
      const int a = hl[h];
      bool out;
      vcur[h] = field_value(g, rigid_col(S + S_R, S + S_T, ld3(tors + 3 * a), a), out);
    }
    if (A.pose_in) {
      const double *ci = A.conf_in + 3 * (size_t)a0;
      for (int i = lane; i < 3 * N; i += 32) conf[i] = ci[i];
    } else {
      for (int a = lane; a < N; a += 32) st3(conf + 3 * a, rigid_col(S + S_R, S + S_T, ld3(tors + 3 * a), a));
    }
    __syncwarp();
    if (lane == 0) {
      if (A.pose_in) {
        S[S_GEO] = A.pose_in[8 * l + 7];
      } else {
        double acc = 0.0;
        for (int h = 0; h < n; ++h) acc += vcur[h];
        S[S_GEO] = acc;
      }
      S[S_STEPT] = A.c.step_t;
      S[S_STEPR] = A.c.step_r;
      S[S_STEPQ] = A.c.step_q;
    }
    if (!A.pose_in) evals += (unsigned long long)n;
    __syncwarp();

    // ---- local_search (search.cpp:121-191)
    int level = 0, n_iter = 0, n_adopt = 0;
    bool failed = false;
    for (int iter = 0; iter < A.c.max_iter && S[S_STEPT] >= A.c.min_t; ++iter) {
      if (lane < 3) S[S_PIV + lane] = centroid_row(conf, N, lane);
      __syncwarp();
      const double step_t = S[S_STEPT], step_q = S[S_STEPQ];
      for (int w = lane; w < J; w += 32) {
        if (w < 12) {
          double *X = Rj + 16 * w;
          if (w < 6) {  // translations (search.cpp:152-158)
            const int axis = w >> 1;
            const double sign = (w & 1) ? -1.0 : 1.0;
            for (int q = 0; q < 9; ++q) X[q] = S[S_R + q];
            for (int q = 0; q < 3; ++q) X[9 + q] = S[S_T + q];
            X[9 + axis] = S[S_T + axis] + sign * step_t;
            for (int q = 0; q < 4; ++q) X[12 + q] = S[S_Q + q];
          } else {  // rotations about the pivot (search.cpp:159-167)
            const double *sq = A.c.spin + 4 * (6 * level + (w - 6));
            const quat spin{sq[0], sq[1], sq[2], sq[3]};
            const d3 piv = ld3(S + S_PIV);
            const d3 sp = quat_rotate(spin, piv);
            const d3 spin_t = sub3(piv, sp);
            const quat cur{S[S_Q], S[S_Q + 1], S[S_Q + 2], S[S_Q + 3]};
            const quat qn = quat_normalized(quat_mul(spin, cur));  // compose, transform.cpp:18-19
            const d3 tt = add3(quat_rotate(spin, ld3(S + S_T)), spin_t);
            quat_matrix(qn, X);
            X[9] = tt.x;
            X[10] = tt.y;
            X[11] = tt.z;
            X[12] = qn.x;
            X[13] = qn.y;
            X[14] = qn.z;
            X[15] = qn.w;
          }
        } else {  // torsion neighbours (search.cpp:168-176)
          const int v = w - 12, t = v >> 1;
          const double sign = (v & 1) ? -1.0 : 1.0;
          if (!cvalid[v]) {
            const double a = ang[t] + sign * step_q;
            vs_crtrig::sincos_cr(a, &cache[2 * v], &cache[2 * v + 1]);
            cvalid[v] = 1;
          }
          if (!chain_mats(t, cache[2 * v], cache[2 * v + 1], m, P, nmax, ha, hb, hl, tm, sccur,
                          Mvar + (size_t)12 * A.mmax * v))
            S[S_ERR] = 1.0;
        }
      }
      __syncwarp();
      if (S[S_ERR] != 0.0) {
        failed = true;
        break;
      }
      // neighbour x heavy-atom samples
      int total_d = 0;
      for (int t = 0; t < m; ++t) total_d += dcnt[t];
      const int nR = 12 * n, nT = 2 * total_d;
      for (int it = lane; it < nR + nT; it += 32) {
        if (it < nR) {
          const int j = it / n, h = it - j * n;
          const int a = hl[h];
          const double *X = Rj + 16 * j;
          bool out;
          vb[j * nmax + h] = field_value(g, rigid_col(X, X + 9, ld3(tors + 3 * a), a), out);
        } else {
          const int kk = it - nR;
          int t = 0;
          while (kk >= 2 * (doff[t] + dcnt[t])) ++t;
          const int rem = kk - 2 * doff[t];
          const int s = rem >= dcnt[t] ? 1 : 0;
          const int h = ditems[doff[t] + rem - s * dcnt[t]];
          const int v = 2 * t + s;
          const int a = hl[h];
          const double *Mv = Mvar + (size_t)12 * A.mmax * v;
          d3 x = ld3(P + 3 * (t * nmax + h));
          const uint32_t mask = tm[a];
          for (int u = t; u < m; ++u)
            if ((mask >> u) & 1u) x = torsion_apply(Mv + 12 * u, x);
          bool out;
          vb[(12 + v) * nmax + h] = field_value(g, rigid_col(S + S_R, S + S_T, x, a), out);
        }
      }
      __syncwarp();
      // geo_score of each neighbour: sequential over heavy atoms (grid.cpp:97-101)
      for (int j = lane; j < J; j += 32) {
        double acc = 0.0;
        const double *row = vb + j * nmax;
        if (j < 12) {
          for (int h = 0; h < n; ++h) acc += row[h];
        } else {
          const int t = (j - 12) >> 1;
          for (int h = 0; h < n; ++h) acc += ((dm[h] >> t) & 1u) ? row[h] : vcur[h];
        }
        scores[j] = acc;
      }
      evals += (unsigned long long)n * J;
      __syncwarp();
      // strict-best neighbour, first wins on ties (search.cpp:138)
      double bv = -__longlong_as_double(0x7ff0000000000000LL);
      int bj = 0x7fffffff;
      for (int j = lane; j < J; j += 32)
        if (scores[j] > bv) {
          bv = scores[j];
          bj = j;
        }
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
        if (ov > bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      const bool improved = bv > S[S_GEO];
      ++n_iter;
      n_adopt += improved ? 1 : 0;
      __syncwarp();
      if (improved) {
        if (bj < 12) {
          const double *X = Rj + 16 * bj;
          if (lane < 9) S[S_R + lane] = X[lane];
          else if (lane < 12) S[S_T + lane - 9] = X[lane];
          else if (lane < 16) S[S_Q + lane - 12] = X[lane];
          __syncwarp();
          for (int a = lane; a < N; a += 32) st3(conf + 3 * a, rigid_col(X, X + 9, ld3(tors + 3 * a), a));
          for (int h = lane; h < n; h += 32) vcur[h] = vb[bj * nmax + h];
        } else {
          const int v = bj - 12, t = v >> 1;
          const double sign = (v & 1) ? -1.0 : 1.0;
          const double *Mv = Mvar + (size_t)12 * A.mmax * v;
          for (int i = lane; i < 12 * (m - t); i += 32) Mcur[12 * t + i] = Mv[12 * t + i];
          if (lane == 0) {
            ang[t] = ang[t] + sign * step_q;
            sccur[2 * t] = cache[2 * v];
            sccur[2 * t + 1] = cache[2 * v + 1];
            cvalid[2 * t] = 0;
            cvalid[2 * t + 1] = 0;
          }
          __syncwarp();
          rebuild_frames(lane, N, m, nmax, base, nullptr, tm, Mcur, P, tors, hidx);
          __syncwarp();
          for (int a = lane; a < N; a += 32)
            st3(conf + 3 * a, rigid_col(S + S_R, S + S_T, ld3(tors + 3 * a), a));
          for (int h = lane; h < n; h += 32)
            if ((dm[h] >> t) & 1u) vcur[h] = vb[bj * nmax + h];
        }
        if (lane == 0) S[S_GEO] = bv;
      } else {
        if (lane == 0) {
          S[S_STEPT] = S[S_STEPT] * 0.5;
          S[S_STEPR] = S[S_STEPR] * 0.5;
          S[S_STEPQ] = S[S_STEPQ] * 0.5;
        }
        for (int v = lane; v < 2 * m; v += 32) cvalid[v] = 0;
        ++level;
      }
      __syncwarp();
    }
    if (failed) {
      if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
      continue;
    }
    // ---- outputs
    const size_t ck = (size_t)a0 * k + (size_t)r * N;
    for (int i = lane; i < 3 * N; i += 32) A.o.conf[3 * ck + i] = conf[i];
    const size_t tk = (size_t)t0 * k + (size_t)r * m;
    for (int u = lane; u < m; u += 32) A.o.ang[tk + u] = ang[u];
    if (lane < 4) A.o.T[7 * (size_t)item + lane] = S[S_Q + lane];
    else if (lane < 7) A.o.T[7 * (size_t)item + lane] = S[S_T + lane - 4];
    if (lane == 0) {
      A.o.geo[item] = S[S_GEO];
      A.o.evals[item] = evals;
      A.o.status[item] = VS_LIG_OK;
      if (A.o.iters) A.o.iters[item] = n_iter;
      if (A.o.adopts) A.o.adopts[item] = n_adopt;
    }
    __syncwarp();
  }
}

static cudaError_t run_search(search_args &A, int num_sms, cudaStream_t s, int *launches) {
  const int Nm = A.Nmax, nm = A.nmax, mm = A.mmax, Jm = 12 + 2 * mm;
  A.Jmax = Jm;
  int o = 0;
  auto take = [&](int n) {
    const int at = o;
    o += (n + 1) & ~1;  // keep 16-byte alignment
    return at;
  };
  A.o_conf = take(3 * Nm);
  A.o_tors = take(3 * Nm);
  A.o_P = take(3 * mm * nm);
  A.o_Mcur = take(12 * mm);
  A.o_Mvar = take(12 * mm * 2 * mm);
  A.o_Rj = take(16 * 12);
  A.o_vb = take(Jm * nm);
  A.o_vcur = take(nm);
  A.o_scores = take(Jm);
  A.o_cache = take(4 * mm);
  A.o_ang = take(mm);
  A.o_sccur = take(2 * mm);
  A.o_state = take(S_N);
  A.o_dm = take((nm + 1) / 2);
  A.o_cvalid = take((2 * mm + 2 + Nm + 1) / 2 + 1);
  A.warp_doubles = o;
  const int warps = 4;
  const size_t smem = (size_t)o * sizeof(double) * warps;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_search, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search, 32 * warps, smem);
  if (per_sm < 1) per_sm = 1;
  int blocks = num_sms * per_sm;
  const int need = (A.n_items + warps - 1) / warps;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  k_search<<<blocks, 32 * warps, smem, s>>>(A);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const flat_out &f,
                          const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                          int num_sms, cudaStream_t s, int *launches) {
  search_args A{};
  A.b = b;
  A.p = p;
  A.c = c;
  A.f = f;
  A.o = o;
  A.work = work_counter;
  A.n_items = b.n_lig * c.k;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  if (A.n_items == 0) return cudaSuccess;
  return run_search(A, num_sms, s, launches);
}

cudaError_t launch_local_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *pose_in,
                                const double *ang_in, const double *conf_in, const item_out &o, int *work_counter,
                                int nmax_atoms, int nmax_heavy, int mmax, int num_sms, cudaStream_t s) {
  search_args A{};
  A.b = b;
  A.p = p;
  A.c = c;
  A.o = o;
  A.pose_in = pose_in;
  A.ang_in = ang_in;
  A.conf_in = conf_in;
  A.work = work_counter;
  A.n_items = b.n_lig;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  if (A.n_items == 0) return cudaSuccess;
  return run_search(A, num_sms, s, nullptr);
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

__device__ __forceinline__ void chem_atom(const pocket_dev &p, d3 x, int ci, double &total, int &clashes,
                                          int &pairs) {
  int lo = 0, hi = p.n_protein;
  const int *list = nullptr;
  const int cx = (int)floor((x.x - p.cmin[0]) / p.cs);
  const int cy = (int)floor((x.y - p.cmin[1]) / p.cs);
  const int cz = (int)floor((x.z - p.cmin[2]) / p.cs);
  if (p.cell_start && cx >= 0 && cy >= 0 && cz >= 0 && cx < p.cdims[0] && cy < p.cdims[1] && cz < p.cdims[2]) {
    const int cell = cx + p.cdims[0] * (cy + p.cdims[1] * cz);
    lo = p.cell_start[cell];
    hi = p.cell_start[cell + 1];
    list = p.cell_atoms;
  }
  for (int q = lo; q < hi; ++q) {
    const int j = list ? __ldg(list + q) : q;
    const d3 pp{__ldg(p.pxyz + 3 * j), __ldg(p.pxyz + 3 * j + 1), __ldg(p.pxyz + 3 * j + 2)};
    const double d = sqrt(sqn3(sub3(x, pp)));
    if (d >= 4.5) continue;
    ++pairs;
    const double ramp = d <= 3.5 ? 1.0 : (4.5 - d) / (4.5 - 3.5);
    total += chem_weight(ci, p.pclass[j]) * ramp;
    if (d < 2.0) {
      total -= 5.0;
      ++clashes;
    }
  }
}

__device__ double chem_pose(const pocket_dev &p, const double *conf, const uint16_t *hl, const uint8_t *elem, int n,
                            int &clashes, int &pairs) {
  double total = 0.0;
  clashes = 0;
  pairs = 0;
  for (int h = 0; h < n; ++h) {
    const int a = hl[h];
    chem_atom(p, ld3(conf + 3 * a), chem_class_of(elem[a]), total, clashes, pairs);
  }
  return total;
}

__device__ __forceinline__ int f_sweeps_of(const dock_out &d, int l) { return d.sweeps ? d.sweeps[l] : 0; }

// ============================================================== k_select
// cluster_and_select + chem_score + best (search.cpp:195-275).  One CTA per
// ligand.
constexpr int kSelThreads = 128;

__global__ void __launch_bounds__(kSelThreads) k_select(batch_dev b, pocket_dev p, search_cfg c, item_out o, dock_out d) {
  extern __shared__ int si[];
  const int l = blockIdx.x, tid = threadIdx.x;
  const int k = c.k;
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
    }
    return;
  }
  const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const uint16_t *hl = b.heavy_list + a0;
  const double *geo = o.geo + (size_t)l * k;
  const double *confs = o.conf + 3 * (size_t)a0 * k;  // pose r at + 3*r*N
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
      for (int h = 0; h < n; ++h) {
        const int a = hl[h];
        sum += sqn3(sub3(ld3(ci + 3 * a), ld3(cl + 3 * a)));
      }
      if (sqrt(sum / (double)n) <= c.rmsd_threshold) atomicMin(&first_match, li);
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
  if (d.best_conf)
    for (int i = tid; i < 3 * N; i += blockDim.x) d.best_conf[3 * (size_t)a0 + i] = bconf[i];
  if (d.best_ang)
    for (int u = tid; u < m; u += blockDim.x) d.best_ang[t0 + u] = o.ang[(size_t)t0 * k + (size_t)bidx * m + u];
  __shared__ int oob;
  if (tid == 0) oob = 0;
  __syncthreads();
  for (int h = tid; h < n; h += blockDim.x) {
    bool out;
    field_value(p.g, ld3(bconf + 3 * hl[h]), out);
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

cudaError_t launch_select(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const item_out &o,
                          const dock_out &d, int nmax_atoms, cudaStream_t s) {
  (void)nmax_atoms;
  if (b.n_lig == 0) return cudaSuccess;
  const int k = c.k;
  const size_t smem = sizeof(int) * (3 * k + (k & 1) + 2) + sizeof(double) * k + 2 * sizeof(int) * k + 16;
  cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_select<<<b.n_lig, kSelThreads, smem, s>>>(b, p, c, o, d);
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

}  // namespace vsd
