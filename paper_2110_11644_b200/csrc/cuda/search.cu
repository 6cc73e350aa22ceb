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

#include "../../../include/vs_crtrig.h"
#include "../../../include/vs_dock.h"
#include "kernels.cuh"

namespace vsd {

namespace {

constexpr int kWarps = 4;
constexpr int kGroup = 16;  // neighbours per group (>= 12)
constexpr double kPi = 3.14159265358979323846;
constexpr double kLatticeStep = 2.0 * kPi / 36;

__device__ __forceinline__ d3 ld3(const double *p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double *p, d3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

// Row `row` of rigid_col (the reference's 3xN apply_rigid, Appendix A item 4).
__device__ __forceinline__ double rigid_row(const double *r, const double *t, d3 v, int col, int row) {
  const double a0 = r[3 * row] * v.x, a1 = r[3 * row + 1] * v.y, a2 = r[3 * row + 2] * v.z;
  const bool packet = (col & 1) == 0 ? row < 2 : row > 0;
  return (packet ? (a0 + a1) + a2 : a0 + (a1 + a2)) + t[row];
}

__device__ __noinline__ void sincos_cr_dev(double a, double *s, double *c) { vs_crtrig::sincos_cr(a, s, c); }

__constant__ double c_lattice_sc_s[72];
__device__ __forceinline__ double c_lattice_sc_dev(int i) { return c_lattice_sc_s[i]; }

enum {
  S_Q = 0,      // current rotation (x, y, z, w)
  S_T = 4,      // current translation
  S_R = 7,      // current rotation matrix
  S_PIV = 16,   // pivot
  S_GEO = 19,   // current geo_score
  S_STEPT = 20,
  S_STEPR = 21,
  S_STEPQ = 22,
  S_ERR = 23,
  S_N = 24
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
  int n_items;
  int Nmax, nmax, mmax;
  int warp_doubles;
  int o_tors, o_Mcur, o_Mvar, o_Rj, o_vb, o_vbest, o_vcur, o_scores, o_cache, o_ang, o_sccur, o_state, o_ints;
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
__device__ __noinline__ bool chain_mats(int t, double st, double ct, int m, const double *base, const uint16_t *ta,
                                        const uint16_t *tb, const uint32_t *tm, const double *Mcur,
                                        const double *sccur, double *out) {
  for (int u = t; u < m; ++u) {
    const int a = ta[u], b = tb[u];
    d3 ea = ld3(base + 3 * a), eb = ld3(base + 3 * b);
    const uint32_t ma = tm[a], mb = tm[b];
    for (int w = 0; w < u; ++w) {
      const double *M = w < t ? Mcur + 12 * w : out + 12 * (w - t);
      if ((ma >> w) & 1u) ea = torsion_apply(M, ea);
      if ((mb >> w) & 1u) eb = torsion_apply(M, eb);
    }
    const double s = u == t ? st : sccur[2 * u];
    const double c = u == t ? ct : sccur[2 * u + 1];
    if (!torsion_setup(ea, eb, s, c, out + 12 * (u - t))) return false;
  }
  return true;
}

// Shared-memory views of one warp plus the current item's ligand tables.
struct WarpState {
  double *tors, *Mcur, *Mvar, *Rj, *vb, *vbest, *vcur, *scores, *cache, *ang, *sccur, *S;
  uint32_t *dm;
  int *cvalid;
  int N, n, m, a0, t0, l, r, k;
  const double *base;
  const uint16_t *hl, *ta, *tb, *ditems;
  const uint32_t *tm;
  const int *dcnt, *doff;
};

// centroid_row over the conformation apply_rigid(tors, T) (or a given
// conformation) computed on the fly: search.cpp:124 / transform.cpp:49-52.
__device__ __noinline__ double pivot_row(const WarpState &w, const double *given, int row) {
  const double *R = w.S + S_R, *T = w.S + S_T;
  auto val = [&](int a) -> double {
    if (given) return given[3 * a + row];
    return rigid_row(R, T, ld3(w.tors + 3 * a), a, row);
  };
  const int N = w.N;
  double p = val(0);
  if (row < 2) {
    const int size4 = (N - 1) & ~3;
    int i = 1;
    for (; i < size4; i += 4) p = p + ((val(i) + val(i + 1)) + (val(i + 2) + val(i + 3)));
    for (; i < N; ++i) p = p + val(i);
  } else {
    for (int i = 1; i < N; ++i) p = p + val(i);
  }
  return p / (double)N;
}

// tors = apply_torsions(base, angles) with the current matrices (warp).
__device__ __noinline__ void rebuild_tors(const WarpState &w, int lane) {
  for (int a = lane; a < w.N; a += 32) {
    d3 x = ld3(w.base + 3 * a);
    const uint32_t mask = w.tm[a];
    for (int u = 0; u < w.m; ++u)
      if ((mask >> u) & 1u) x = torsion_apply(w.Mcur + 12 * u, x);
    st3(w.tors + 3 * a, x);
  }
}

template <int MODE>
__device__ __noinline__ double sample_cold(const search_args &A, const double *pal, d3 p) {
  bool out;
  return field_value_fast<MODE>(A.p.g, A.pg, pal, p, out);
}

// Restart start-up: tables, torsion matrices, torsioned frame, start pose,
// its samples and score, pivot.  Returns false on a degenerate axis.
template <int MODE>
__device__ __noinline__ bool init_restart(const search_args &A, const double *pal, WarpState &w, int lane,
                                          unsigned long long &evals) {
  const bool ls_mode = A.pose_in != nullptr;
  const int m = w.m, n = w.n;
  for (int h = lane; h < n; h += 32) w.dm[h] = A.b.heavy_dmask[w.a0 + h];
  for (int v = lane; v < 2 * m; v += 32) w.cvalid[v] = 0;
  if (A.ang_in) {  // local_search / initial_poses entry points: arbitrary angles
    for (int u = lane; u < m; u += 32) {
      w.ang[u] = A.ang_in[w.t0 + u];
      sincos_cr_dev(w.ang[u], &w.sccur[2 * u], &w.sccur[2 * u + 1]);
    }
  } else {
    for (int u = lane; u < m; u += 32) {
      const int li = A.f.idx[w.t0 + u];
      w.ang[u] = li * kLatticeStep;  // angles_of, search.cpp:40
      w.sccur[2 * u] = c_lattice_sc_dev(2 * li);
      w.sccur[2 * u + 1] = c_lattice_sc_dev(2 * li + 1);
    }
  }
  if (lane == 0) w.S[S_ERR] = 0.0;
  __syncwarp();
  if (lane == 0 && m > 0 && !chain_mats(0, w.sccur[0], w.sccur[1], m, w.base, w.ta, w.tb, w.tm, w.Mcur, w.sccur, w.Mcur))
    w.S[S_ERR] = 1.0;
  __syncwarp();
  if (w.S[S_ERR] != 0.0) return false;
  rebuild_tors(w, lane);  // torsioned frame (search.cpp:115)
  __syncwarp();
  if (!ls_mode && A.ang_in) {  // initial_poses entry: flat centroid of these angles
    if (lane < 3) w.S[S_PIV + lane] = centroid_row(w.tors, w.N, lane);
    __syncwarp();
  }
  if (lane == 0) {  // start pose: initial_poses (search.cpp:95-103) or the given one
    quat q;
    double t[3];
    if (ls_mode) {
      const double *pi = A.pose_in + 8 * w.l;
      q = {pi[0], pi[1], pi[2], pi[3]};
      t[0] = pi[4];
      t[1] = pi[5];
      t[2] = pi[6];
    } else {
      const double *fq = A.c.fibq + 4 * w.r;
      q = {fq[0], fq[1], fq[2], fq[3]};
      const d3 rc = quat_rotate(q, A.ang_in ? ld3(w.S + S_PIV) : ld3(A.f.centroid + 3 * w.l));
      t[0] = A.p.center[0] - rc.x;
      t[1] = A.p.center[1] - rc.y;
      t[2] = A.p.center[2] - rc.z;
    }
    w.S[S_Q] = q.x;
    w.S[S_Q + 1] = q.y;
    w.S[S_Q + 2] = q.z;
    w.S[S_Q + 3] = q.w;
    w.S[S_T] = t[0];
    w.S[S_T + 1] = t[1];
    w.S[S_T + 2] = t[2];
    quat_matrix(q, w.S + S_R);
    w.S[S_STEPT] = A.c.step_t;
    w.S[S_STEPR] = A.c.step_r;
    w.S[S_STEPQ] = A.c.step_q;
  }
  __syncwarp();
  for (int h = lane; h < n; h += 32) {
    const int a = w.hl[h];
    w.vcur[h] = sample_cold<MODE>(A, pal, rigid_col(w.S + S_R, w.S + S_T, ld3(w.tors + 3 * a), a));
  }
  __syncwarp();
  if (lane == 0) {
    if (ls_mode) {
      w.S[S_GEO] = A.pose_in[8 * w.l + 7];
    } else {
      double acc = 0.0;
      for (int h = 0; h < n; ++h) acc += w.vcur[h];
      w.S[S_GEO] = acc;
    }
  }
  if (!ls_mode) evals += (unsigned long long)n;
  if (lane < 3) w.S[S_PIV + lane] = pivot_row(w, ls_mode ? A.conf_in + 3 * (size_t)w.a0 : nullptr, lane);
  __syncwarp();
  return true;
}

// Rigid neighbour transforms (search.cpp:152-167) and, when stale, the
// torsion-neighbour matrices (search.cpp:168-176).  Returns false on a
// degenerate axis.
__device__ __noinline__ bool neighbour_setup(const search_args &A, WarpState &w, int lane, int level, bool mvar_valid) {
  const int m = w.m, J = 12 + 2 * m;
  const double step_t = w.S[S_STEPT], step_q = w.S[S_STEPQ];
  bool ok = true;
  for (int j = lane; j < (mvar_valid ? 12 : J); j += 32) {
    if (j < 12) {
      double *X = w.Rj + 16 * j;
      if (j < 6) {
        const int axis = j >> 1;
        const double sign = (j & 1) ? -1.0 : 1.0;
        for (int q = 0; q < 9; ++q) X[q] = w.S[S_R + q];
        for (int q = 0; q < 3; ++q) X[9 + q] = w.S[S_T + q];
        X[9 + axis] = w.S[S_T + axis] + sign * step_t;
        for (int q = 0; q < 4; ++q) X[12 + q] = w.S[S_Q + q];
      } else {
        const double *sq = A.c.spin + 4 * (6 * level + (j - 6));
        const quat spin{sq[0], sq[1], sq[2], sq[3]};
        const d3 piv = ld3(w.S + S_PIV);
        const d3 spin_t = sub3(piv, quat_rotate(spin, piv));
        const quat cur{w.S[S_Q], w.S[S_Q + 1], w.S[S_Q + 2], w.S[S_Q + 3]};
        const quat qn = quat_normalized(quat_mul(spin, cur));  // compose, transform.cpp:18-19
        const d3 tt = add3(quat_rotate(spin, ld3(w.S + S_T)), spin_t);
        quat_matrix(qn, X);
        X[9] = tt.x;
        X[10] = tt.y;
        X[11] = tt.z;
        X[12] = qn.x;
        X[13] = qn.y;
        X[14] = qn.z;
        X[15] = qn.w;
      }
    } else {
      const int v = j - 12, t = v >> 1;
      const double sign = (v & 1) ? -1.0 : 1.0;
      if (!w.cvalid[v]) {
        sincos_cr_dev(w.ang[t] + sign * step_q, &w.cache[2 * v], &w.cache[2 * v + 1]);
        w.cvalid[v] = 1;
      }
      if (!chain_mats(t, w.cache[2 * v], w.cache[2 * v + 1], m, w.base, w.ta, w.tb, w.tm, w.Mcur, w.sccur,
                      w.Mvar + mvar_off(v, t, m)))
        ok = false;
    }
  }
  return __all_sync(0xffffffffu, ok);
}

// Adopt neighbour bj (search.cpp:178-185) whose per-atom samples are vbest.
__device__ __noinline__ void adopt(WarpState &w, int lane, int bj, double bv) {
  const int m = w.m;
  if (bj < 12) {
    const double *X = w.Rj + 16 * bj;
    if (lane < 9)
      w.S[S_R + lane] = X[lane];
    else if (lane < 12)
      w.S[S_T + lane - 9] = X[lane];
    else if (lane < 16)
      w.S[S_Q + lane - 12] = X[lane];
  } else {
    const int v = bj - 12, t = v >> 1;
    const double sign = (v & 1) ? -1.0 : 1.0;
    const double step_q = w.S[S_STEPQ];
    for (int i = lane; i < 12 * (m - t); i += 32) w.Mcur[12 * t + i] = w.Mvar[mvar_off(v, t, m) + i];
    if (lane == 0) {
      w.ang[t] = w.ang[t] + sign * step_q;
      w.sccur[2 * t] = w.cache[2 * v];
      w.sccur[2 * t + 1] = w.cache[2 * v + 1];
    }
    if (lane < 2) w.cvalid[2 * t + lane] = 0;
    __syncwarp();
    rebuild_tors(w, lane);
  }
  for (int h = lane; h < w.n; h += 32) w.vcur[h] = w.vbest[h];
  if (lane == 0) w.S[S_GEO] = bv;
  __syncwarp();
  if (lane < 3) w.S[S_PIV + lane] = pivot_row(w, nullptr, lane);  // new pivot
}

__device__ __noinline__ void write_outputs(const search_args &A, const WarpState &w, int lane, int item, bool moved,
                                           unsigned long long evals, int n_iter, int n_adopt) {
  const bool ls_mode = A.pose_in != nullptr;
  const int N = w.N, m = w.m;
  const size_t ck = 3 * ((size_t)w.a0 * w.k + (size_t)w.r * N);
  if (ls_mode && !moved) {  // an unmoved pose keeps its input conformation
    for (int i = lane; i < 3 * N; i += 32) A.o.conf[ck + i] = A.conf_in[3 * (size_t)w.a0 + i];
  } else {
    for (int a = lane; a < N; a += 32)
      st3(A.o.conf + ck + 3 * a, rigid_col(w.S + S_R, w.S + S_T, ld3(w.tors + 3 * a), a));
  }
  const size_t tk = (size_t)w.t0 * w.k + (size_t)w.r * m;
  for (int u = lane; u < m; u += 32) A.o.ang[tk + u] = w.ang[u];
  if (lane < 4)
    A.o.T[7 * (size_t)item + lane] = w.S[S_Q + lane];
  else if (lane < 7)
    A.o.T[7 * (size_t)item + lane] = w.S[S_T + lane - 4];
  if (lane == 0) {
    A.o.geo[item] = w.S[S_GEO];
    A.o.evals[item] = evals;
    A.o.status[item] = VS_LIG_OK;
    if (A.o.iters) A.o.iters[item] = n_iter;
    if (A.o.adopts) A.o.adopts[item] = n_adopt;
  }
}

template <int MODE>
__global__ void __launch_bounds__(32 * kWarps, 4) k_search(const search_args *__restrict__ Ap) {
  const search_args &A = *Ap;  // lives in global memory: the cold paths take it by reference
  extern __shared__ double sm[];
  double *pal = sm;  // 16 palette values (CTA-wide)
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < 16) pal[threadIdx.x] = MODE == 0 ? 0.0 : A.p.palette[threadIdx.x];
  __syncthreads();
  double *W = sm + 16 + (size_t)warp * A.warp_doubles;
  WarpState w;
  w.tors = W + A.o_tors;
  w.Mcur = W + A.o_Mcur;
  w.Mvar = W + A.o_Mvar;
  w.Rj = W + A.o_Rj;
  w.vb = W + A.o_vb;
  w.vbest = W + A.o_vbest;
  w.vcur = W + A.o_vcur;
  w.scores = W + A.o_scores;
  w.cache = W + A.o_cache;
  w.ang = W + A.o_ang;
  w.sccur = W + A.o_sccur;
  w.S = W + A.o_state;
  w.dm = reinterpret_cast<uint32_t *>(W + A.o_ints);
  w.cvalid = reinterpret_cast<int *>(w.dm + A.nmax);
  const int k = A.pose_in ? 1 : A.c.k;
  w.k = k;
  const int nmax = A.nmax;
  const grid_view &g = A.p.g;
  const packed_grid &pg = A.pg;

  while (true) {
    int item = 0;
    if (lane == 0) item = atomicAdd(A.work, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= A.n_items) break;
    w.l = item / k;
    w.r = item - w.l * k;
    const lig_meta meta = A.b.meta[w.l];
    if (meta.status != VS_LIG_OK) {
      if (lane == 0) A.o.status[item] = meta.status;
      continue;
    }
    w.N = meta.n_atoms;
    w.n = meta.n_heavy;
    w.m = meta.m;
    w.a0 = A.b.atom_off[w.l];
    w.t0 = A.b.tors_off[w.l];
    w.base = A.b.xyz + 3 * (size_t)w.a0;
    w.hl = A.b.heavy_list + w.a0;
    w.tm = A.b.atom_tmask + w.a0;
    w.ta = A.b.tors_a + w.t0;
    w.tb = A.b.tors_b + w.t0;
    w.dcnt = A.b.d_count + w.t0;
    w.doff = A.b.d_off + w.t0;
    w.ditems = A.b.ditems + A.b.ditem_base[w.l];
    const int n = w.n, m = w.m, J = 12 + 2 * m;
    unsigned long long evals = 0;
    if (!init_restart<MODE>(A, pal, w, lane, evals)) {
      if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
      continue;
    }

    // register copies of the per-item views for the hot loop
    double *const tors = w.tors, *const Mcur = w.Mcur, *const Mvar = w.Mvar, *const Rj = w.Rj, *const vb = w.vb;
    double *const vbest = w.vbest, *const vcur = w.vcur, *const scores = w.scores, *const S = w.S;
    const uint32_t *const dm = w.dm, *const tm = w.tm;
    const uint16_t *const hl = w.hl, *const ditems = w.ditems;
    const int *const dcnt = w.dcnt, *const doff = w.doff;
    const double *const base = w.base;
    // ---- local_search (search.cpp:121-191)
    int level = 0, n_iter = 0, n_adopt = 0;
    bool failed = false, mvar_valid = false, moved = false;
    for (int iter = 0; iter < A.c.max_iter && S[S_STEPT] >= A.c.min_t; ++iter) {
      if (!neighbour_setup(A, w, lane, level, mvar_valid)) {
        failed = true;
        break;
      }
      mvar_valid = true;
      __syncwarp();
      // neighbour groups: rigid first, then torsion neighbours in order
      double bv = S[S_GEO];
      int bj = -1;
      int tg = 0;
      for (int grp = 0; grp == 0 || tg < m; ++grp) {
        int j0, jn, tlo = 0, items;
        if (grp == 0) {
          j0 = 0;
          jn = 12;
          items = 12 * n;
        } else {
          tlo = tg;
          const int thi = min(m, tlo + kGroup / 2);
          tg = thi;
          j0 = 12 + 2 * tlo;
          jn = 2 * (thi - tlo);
          items = 2 * (doff[thi - 1] + dcnt[thi - 1] - doff[tlo]);
        }
        for (int it = lane; it < items; it += 32) {
          d3 p;
          int row, h;
          if (grp == 0) {
            const int j = it / n;
            h = it - j * n;
            const int a = hl[h];
            const double *X = Rj + 16 * j;
            p = rigid_col(X, X + 9, ld3(tors + 3 * a), a);
            row = j;
          } else {
            const int kk = it + 2 * doff[tlo];
            int t = tlo;
            while (kk >= 2 * (doff[t] + dcnt[t])) ++t;
            const int rem = kk - 2 * doff[t];
            const int s = rem >= dcnt[t] ? 1 : 0;
            h = ditems[doff[t] + rem - s * dcnt[t]];
            const int v = 2 * t + s;
            const int a = hl[h];
            d3 x = ld3(base + 3 * a);
            const uint32_t mask = tm[a];
            for (int u = 0; u < m; ++u) {
              if (!((mask >> u) & 1u)) continue;
              x = torsion_apply(u < t ? Mcur + 12 * u : Mvar + mvar_off(v, u, m), x);
            }
            p = rigid_col(S + S_R, S + S_T, x, a);
            row = v - 2 * tlo;
          }
          bool out;
          vb[row * nmax + h] = field_value_fast<MODE>(g, pg, pal, p, out);
        }
        __syncwarp();
        // geo_score of each neighbour in the group (grid.cpp:97-101)
        if (lane < jn) {
          const double *rowp = vb + lane * nmax;
          double acc = 0.0;
          const int t = grp == 0 ? 31 : tlo + (lane >> 1);
          const uint32_t bit = grp == 0 ? 0xffffffffu : (1u << t);
          for (int h = 0; h < n; ++h) acc += (dm[h] & bit) || grp == 0 ? rowp[h] : vcur[h];
          scores[lane] = acc;
        }
        __syncwarp();
        // first strict maximum of the group, then against the running best
        double gv = lane < jn ? scores[lane] : -__longlong_as_double(0x7ff0000000000000LL);
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
          bj = j0 + gj;
          const double *rowp = vb + gj * nmax;
          const uint32_t bit = grp == 0 ? 0xffffffffu : (1u << (tlo + (gj >> 1)));
          for (int h = lane; h < n; h += 32) vbest[h] = (dm[h] & bit) || grp == 0 ? rowp[h] : vcur[h];
        }
        __syncwarp();
      }
      evals += (unsigned long long)n * J;
      ++n_iter;
      if (bj >= 0) {
        ++n_adopt;
        moved = true;
        if (bj >= 12) mvar_valid = false;
        adopt(w, lane, bj, bv);
      } else {
        if (lane == 0) {
          S[S_STEPT] = S[S_STEPT] * 0.5;
          S[S_STEPR] = S[S_STEPR] * 0.5;
          S[S_STEPQ] = S[S_STEPQ] * 0.5;
        }
        for (int v = lane; v < 2 * m; v += 32) w.cvalid[v] = 0;
        mvar_valid = false;
        ++level;
      }
      __syncwarp();
    }
    if (failed) {
      if (lane == 0) A.o.status[item] = VS_LIG_DEGENERATE_AXIS;
      continue;
    }
    write_outputs(A, w, lane, item, moved, evals, n_iter, n_adopt);
    __syncwarp();
  }
}

namespace {

cudaError_t run_search(search_args &A, search_args *dev_args, int num_sms, cudaStream_t s, int *launches) {
  const int Nm = A.Nmax, nm = A.nmax, mm = A.mmax;
  int o = 0;
  auto take = [&](int n) {
    const int at = o;
    o += (n + 1) & ~1;  // keep 16-byte alignment
    return at;
  };
  A.o_tors = take(3 * Nm);
  A.o_Mcur = take(12 * mm);
  A.o_Mvar = take(12 * mm * (mm + 1));
  A.o_Rj = take(16 * 12);
  A.o_vb = take(kGroup * nm);
  A.o_vbest = take(nm);
  A.o_vcur = take(nm);
  A.o_scores = take(kGroup);
  A.o_cache = take(4 * mm);
  A.o_ang = take(mm);
  A.o_sccur = take(2 * mm);
  A.o_state = take(S_N);
  A.o_ints = take((nm + 2 * mm + 3) / 2 + 1);
  A.warp_doubles = o;
  const size_t smem = (size_t)(16 + o * kWarps) * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const void *fn = A.pg.mode == 1 ? (const void *)k_search<1>
                                  : (A.pg.mode == 2 ? (const void *)k_search<2> : (const void *)k_search<0>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kWarps, smem);
  if (per_sm < 1) per_sm = 1;
  int blocks = num_sms * per_sm;
  const int need = (A.n_items + kWarps - 1) / kWarps;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  e = cudaMemcpyAsync(dev_args, &A, sizeof(search_args), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  if (A.pg.mode == 1)
    k_search<1><<<blocks, 32 * kWarps, smem, s>>>(dev_args);
  else if (A.pg.mode == 2)
    k_search<2><<<blocks, 32 * kWarps, smem, s>>>(dev_args);
  else
    k_search<0><<<blocks, 32 * kWarps, smem, s>>>(dev_args);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

void set_lattice_table_search(const double *sc72) { cudaMemcpyToSymbol(c_lattice_sc_s, sc72, sizeof(double) * 72); }

size_t search_args_bytes() { return sizeof(search_args); }

cudaError_t launch_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const flat_out &f,
                          const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                          int num_sms, cudaStream_t s, int *launches, void *args_buf) {
  search_args A{};
  A.b = b;
  A.p = p;
  A.pg = p.packed;
  A.c = c;
  A.f = f;
  A.o = o;
  A.work = work_counter;
  A.n_items = b.n_lig * c.k;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  if (A.n_items == 0) return cudaSuccess;
  return run_search(A, static_cast<search_args *>(args_buf), num_sms, s, launches);
}

cudaError_t launch_initial_poses(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *angles,
                                 const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                                 int num_sms, cudaStream_t s, void *args_buf) {
  search_args A{};
  A.b = b;
  A.p = p;
  A.pg = p.packed;
  A.c = c;
  A.c.max_iter = 0;  // poses only: no local_search iteration
  A.o = o;
  A.ang_in = angles;
  A.work = work_counter;
  A.n_items = b.n_lig * c.k;
  A.Nmax = nmax_atoms > 0 ? nmax_atoms : 1;
  A.nmax = nmax_heavy > 0 ? nmax_heavy : 1;
  A.mmax = mmax > 0 ? mmax : 1;
  if (A.n_items == 0) return cudaSuccess;
  return run_search(A, static_cast<search_args *>(args_buf), num_sms, s, nullptr);
}

cudaError_t launch_local_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *pose_in,
                                const double *ang_in, const double *conf_in, const item_out &o, int *work_counter,
                                int nmax_atoms, int nmax_heavy, int mmax, int num_sms, cudaStream_t s,
                                void *args_buf) {
  search_args A{};
  A.b = b;
  A.p = p;
  A.pg = p.packed;
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
  return run_search(A, static_cast<search_args *>(args_buf), num_sms, s, nullptr);
}

}  // namespace vsd
