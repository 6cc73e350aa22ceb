// cluster_and_select + chem_score + the best pose of one ligand on one warp
// (search.cpp:195-275, chem.cpp:17-46), shared by the stand-alone k_select_warp
// (kernels.cu) and the search kernel's fused epilogue (search.cu, k <= 32):
// the restarts of the ligand are items item0 + r of the item_out arrays, the
// conformation of restart r at confs + 3 r N, its angles at o.ang + tk0 + r m.
#pragma once

#include "../../../include/vs_dock.h"
#include "kernels.cuh"

namespace vsd {

__device__ __forceinline__ d3 sel_ld3(const double *p) { return {p[0], p[1], p[2]}; }

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
    // (an exact d2 >= 20.25 early-out before the sqrt measured 6% slower:
    // the lanes are different poses, so the branch only adds divergence)
    const double d = dsqrt(sqn3(sub3(x, pp)));
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

static __device__ __noinline__ double chem_pose(const pocket_dev &p, const double *conf, const uint16_t *hl, const uint8_t *elem, int n,
                            int &clashes, int &pairs) {
  double total = 0.0;
  clashes = 0;
  pairs = 0;
  for (int h = 0; h < n; ++h) {
    const int a = hl[h];
    chem_atom(p, sel_ld3(conf + 3 * a), chem_class_of(elem[a]), total, clashes, pairs);
  }
  return total;
}

__device__ __forceinline__ int f_sweeps_of(const dock_out &d, int l) { return d.sweeps ? d.sweeps[l] : 0; }

static __device__ __noinline__ void select_ligand_warp(const batch_dev &b, const pocket_dev &p, const search_cfg &c,
                                                   const item_out &o, size_t item0, const double *confs, size_t tk0,
                                                   const dock_out &d, int l, int lane, int *order, int *leaders,
                                                   int *followers) {
  const int k = c.k;
  vs_dock_result *res = reinterpret_cast<vs_dock_result *>(d.results) + l;
  const lig_meta meta = b.meta[l];
  int status = meta.status;
  if (status == VS_LIG_OK) {
    const int st = lane < k ? o.status[item0 + lane] : VS_LIG_OK;
    status = __reduce_max_sync(0xffffffffu, st);
  }
  if (status != VS_LIG_OK) {
    if (lane == 0) {
      vs_dock_result z{};
      z.status = status;
      *res = z;
    }
    return;
  }
  const int N = meta.n_atoms, n = meta.n_heavy, m = meta.m;
  const int a0 = b.atom_off[l], t0 = b.tors_off[l];
  const uint16_t *hl = b.heavy_list + a0;
  const double *geo = o.geo + item0;  // pose r's conformation at confs + 3*r*N
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
      #pragma unroll 1
      for (int h = 0; h < n; ++h) {
        const int a = hl[h];
        sum += sqn3(sub3(sel_ld3(ci + 3 * a), sel_ld3(cl + 3 * a)));
      }
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
  if (d.best_conf)
    for (int i = lane; i < 3 * N; i += 32) d.best_conf[3 * (size_t)a0 + i] = bconf[i];
  if (d.best_ang)
    for (int u = lane; u < m; u += 32) d.best_ang[t0 + u] = o.ang[tk0 + (size_t)bidx * m + u];
  int oob = 0;
  for (int h = lane; h < n; h += 32) {
    bool out;
    field_value(p.g, sel_ld3(bconf + 3 * hl[h]), out);
    oob += out ? 1 : 0;
  }
  oob = __reduce_add_sync(0xffffffffu, oob);
  unsigned long long ev = lane < k ? o.evals[item0 + lane] : 0ull;
  unsigned long long iters = lane < k && o.iters ? (unsigned long long)o.iters[item0 + lane] : 0ull;
  unsigned long long adopts = lane < k && o.adopts ? (unsigned long long)o.adopts[item0 + lane] : 0ull;
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
    const size_t item = item0 + bidx;
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

}  // namespace vsd
