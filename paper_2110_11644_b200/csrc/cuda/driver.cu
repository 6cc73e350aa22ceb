// Host driver of libvsdock.so: implements include/vs_dock.h.
//
// Owns contexts (device + stream + reusable device buffers), device-resident
// pockets (grid + protein + chem culling cells) and the batch pipeline
//   H2D batch -> k_setup -> k_flatten -> k_search -> k_select -> D2H results
// processed in chunks that bound the per-restart scratch.  Input-independent
// trig (Fibonacci restarts, rotation spins: search.cpp:71-82, 97-98, 162-163)
// is computed here once per call with glibc, exactly as the reference does,
// and shipped to the device as tables.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/vs_crtrig.h"
#include "../../../include/vs_codec.h"
#include "../../../include/vs_dock.h"
#include "../../../include/vs_rank.h"
#include "../host/ligand_set.hpp"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;

vs_status fail(vs_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(VS_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <typename T>
  T *as() const {
    return static_cast<T *>(p);
  }
};

constexpr double kPi = 3.14159265358979323846;
std::once_flag g_lattice_once[64];

}  // namespace

struct vs_context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evs[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_flat = nullptr;  // end of flatten (multi-pocket runs reuse evs[2..4] per pocket)
  double stage_ms[4] = {0, 0, 0, 0};  // setup, flatten, search, select
  double last_ms = 0.0;
  int last_launches = 0;
  std::mutex mu;
  // batch inputs
  DevBuf atom_off, bond_off, tors_off, ditem_base, xyz, elem, heavy, bond_a, bond_b, tors_bond, right_off, right_atoms;
  // derived
  DevBuf meta, tmask, heavy_list, dmask, tors_a, tors_b, d_count, d_off, ditems, titems;
  // flatten / search / select
  DevBuf flat_idx, flat_xyz, flat_centroid, flat_sweeps, out_geo, out_T, out_ang, out_conf, out_evals, out_status,
      out_iters, out_adopts, work;
  DevBuf results, best_ang, best_conf, best_idx, sel_scratch, counters, spin, fibq, stepsc, flat_index;
  DevBuf aux0, aux1, aux2, aux3, search_args, lig_index;
  // record decode
  DevBuf dec_bytes, dec_offs, dec_aoff, dec_boff, dec_toff, dec_rsoff, dec_xyz, dec_elem, dec_heavy, dec_order,
      dec_ba, dec_bb, dec_tbond, dec_rslots, dec_rcount, dec_status;
};

struct vs_pocket {
  int device = 0;
  double origin[3] = {0, 0, 0};
  double spacing = 0.5;
  int dims[3] = {0, 0, 0};
  int n_protein = 0;
  DevBuf values, pxyz, pclass, cell_start, cell_rec, packed, palette, screen;
  int packed_mode = 0;
  bool has_screen = false;
  vsd::screen_grid scr{};
  int bricks[2] = {0, 0};
  double cmin[3] = {0, 0, 0};
  double cs = 2.0;
  int cdims[3] = {0, 0, 0};
  bool has_cells = false;

  vsd::pocket_dev dev() const {
    vsd::pocket_dev p{};
    p.g.ox = origin[0];
    p.g.oy = origin[1];
    p.g.oz = origin[2];
    p.g.h = spacing;
    p.g.mx = static_cast<double>(dims[0] - 1);
    p.g.my = static_cast<double>(dims[1] - 1);
    p.g.mz = static_cast<double>(dims[2] - 1);
    p.g.dx = dims[0];
    p.g.dy = dims[1];
    p.g.dz = dims[2];
    p.g.v = values.as<double>();
    const double hs = 0.5 * spacing;  // box_center, pocket.hpp:53-56
    for (int a = 0; a < 3; ++a) p.center[a] = origin[a] + hs * static_cast<double>(dims[a] - 1);
    p.n_protein = n_protein;
    p.pxyz = pxyz.as<double>();
    p.pclass = pclass.as<uint8_t>();
    for (int a = 0; a < 3; ++a) {
      p.cmin[a] = cmin[a];
      p.cdims[a] = cdims[a];
    }
    p.cs = cs;
    p.cell_start = has_cells ? cell_start.as<int>() : nullptr;
    p.cell_rec = has_cells ? reinterpret_cast<const double2 *>(cell_rec.p) : nullptr;
    p.packed.mode = packed_mode;
    p.packed.cx = bricks[0];
    p.packed.cy = bricks[1];
    p.packed.c2 = packed_mode == 1 ? packed.as<uint16_t>() : nullptr;
    p.packed.c4 = packed_mode == 2 ? packed.as<uint32_t>() : nullptr;
    p.packed.inv_h = 1.0 / spacing;  // correctly rounded reciprocal for div_h
    p.palette = palette.as<double>();
    p.scr = scr;
    // The FP32 screen is exact but measured slower than the FP64 search on
    // configs[1]: opt-in with VS_SCREEN=1.
    const char *scr_env = std::getenv("VS_SCREEN");
    p.scr.w = has_screen && scr_env && std::atoi(scr_env) != 0 ? screen.as<uint32_t>() : nullptr;
    return p;
  }
};

namespace {

void ensure_lattice(int device) {
  std::call_once(g_lattice_once[device & 63], [] {
    double sc[72], lo[72];
    constexpr double step = 2.0 * kPi / 36;  // search.cpp:33
    for (int i = 0; i < 36; ++i) {
      vs_crtrig::dd s, c;
      vs_crtrig::sincos_dd(i * step, &s, &c);
      sc[2 * i] = s.hi;
      sc[2 * i + 1] = c.hi;
      lo[2 * i] = s.lo;
      lo[2 * i + 1] = c.lo;
    }
    vsd::set_lattice_table(sc, lo);
  });
}

int chem_class(uint8_t e) { return e == VS_ELEM_C ? 0 : ((e == VS_ELEM_N || e == VS_ELEM_O) ? 1 : 2); }

// Cell edge: the smallest of these whose grid stays within kChemCellsMax
// cells.  Smaller cells list fewer atoms beyond 4.5 A (1 A: 64% of the listed
// atoms are within 4.5 A of a point of the cell, 2 A: 43%); measured select
// per 131k-ligand step: 2 A +12%, 1 A 19.3 ms, 0.75 A 18.4 ms, 0.5 A 17.7 ms
// (records: 32 B per entry, ~60 MB for the 65^3 bench pocket at 0.75 A).
constexpr double kChemCells[] = {0.75, 1.0, 1.5, 2.0, 3.0};
constexpr int64_t kChemCellsMax = int64_t(1) << 21;

// Culling cells for chem_score: every protein atom whose distance to the
// cell's box is below 4.5 A (+1e-6 margin), listed in protein order.
vs_status build_cells(vs_pocket *p, const uint8_t *elem, const double *xyz) {
  const double cutoff = 4.5 + 1e-6;
  // cell edge: smaller cells list fewer atoms beyond 4.5 A per cell (A/B
  // override VSDOCK_CHEM_CELL, development only)
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = p->origin[a] - 5.0;
    hi[a] = p->origin[a] + p->spacing * (p->dims[a] - 1) + 5.0;
    p->cmin[a] = lo[a];
  }
  auto cells_of = [&](double c) {
    int64_t nc = 1;
    for (int a = 0; a < 3; ++a) nc *= static_cast<int64_t>(std::ceil((hi[a] - lo[a]) / c));
    return nc;
  };
  double cs = kChemCells[sizeof(kChemCells) / sizeof(kChemCells[0]) - 1];
  for (const double c : kChemCells)
    if (cells_of(c) <= kChemCellsMax) {
      cs = c;
      break;
    }
  if (const char *e = std::getenv("VSDOCK_CHEM_CELL")) cs = std::atof(e) > 0.25 ? std::atof(e) : cs;  // A/B only
  for (int a = 0; a < 3; ++a) p->cdims[a] = static_cast<int>(std::ceil((hi[a] - lo[a]) / cs));
  p->cs = cs;
  const int64_t ncell = static_cast<int64_t>(p->cdims[0]) * p->cdims[1] * p->cdims[2];
  if (ncell <= 0 || ncell > (1 << 22) || p->n_protein == 0) {
    p->has_cells = false;
    return VS_OK;
  }
  std::vector<std::vector<int>> lists(static_cast<size_t>(ncell));
  const int reach = static_cast<int>(std::ceil(cutoff / cs)) + 1;
  for (int j = 0; j < p->n_protein; ++j) {
    const double x[3] = {xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2]};
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = static_cast<int>(std::floor((x[a] - lo[a]) / cs));
    for (int dz = -reach; dz <= reach; ++dz)
      for (int dy = -reach; dy <= reach; ++dy)
        for (int dx = -reach; dx <= reach; ++dx) {
          const int cc[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
          if (cc[0] < 0 || cc[1] < 0 || cc[2] < 0 || cc[0] >= p->cdims[0] || cc[1] >= p->cdims[1] ||
              cc[2] >= p->cdims[2])
            continue;
          double d2 = 0.0;
          for (int a = 0; a < 3; ++a) {
            const double bl = lo[a] + cc[a] * cs, bh = bl + cs;
            const double q = x[a] < bl ? bl - x[a] : (x[a] > bh ? x[a] - bh : 0.0);
            d2 += q * q;
          }
          if (d2 < cutoff * cutoff)
            lists[static_cast<size_t>(cc[0] + p->cdims[0] * (cc[1] + static_cast<int64_t>(p->cdims[1]) * cc[2]))]
                .push_back(j);
        }
  }
  std::vector<int> start(static_cast<size_t>(ncell) + 1, 0), atoms;
  for (int64_t c = 0; c < ncell; ++c) {
    start[static_cast<size_t>(c)] = static_cast<int>(atoms.size());
    atoms.insert(atoms.end(), lists[static_cast<size_t>(c)].begin(), lists[static_cast<size_t>(c)].end());
  }
  start[static_cast<size_t>(ncell)] = static_cast<int>(atoms.size());
  if (atoms.empty()) atoms.push_back(0);
  // the entries as records (x, y, z, class): chem_atom reads one 32-byte
  // record per protein atom instead of an index and then the atom
  std::vector<double> rec(4 * atoms.size());
  for (size_t q = 0; q < atoms.size(); ++q) {
    const int j = atoms[q];
    for (int a = 0; a < 3; ++a) rec[4 * q + a] = xyz[3 * j + a];
    rec[4 * q + 3] = static_cast<double>(chem_class(elem[j]));
  }
  CUDA_TRY(p->cell_rec.ensure(rec.size() * sizeof(double)));
  CUDA_TRY(cudaMemcpy(p->cell_rec.p, rec.data(), rec.size() * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(p->cell_start.ensure(start.size() * sizeof(int)));
  CUDA_TRY(cudaMemcpy(p->cell_start.p, start.data(), start.size() * sizeof(int), cudaMemcpyHostToDevice));
  p->has_cells = true;
  return VS_OK;
}

// Screen grid of the FP32 search screen (kernels.cuh screen_grid): per cell
// the pair-table offsets of its four x-pairs and the NU flag, plus the
// pocket's error-model constants.  `code` = 2-bit node codes, `pal` <= 4 values.
vs_status build_screen(vs_pocket *p, const std::vector<uint8_t> &code, const std::vector<double> &pal) {
  const int D0 = p->dims[0], D1 = p->dims[1], D2 = p->dims[2];
  vsd::screen_grid &s = p->scr;
  s = vsd::screen_grid{};
  double vmin = 0.0, vmax = 0.0, vabs = 10.0, jump = 0.0;
  bool exact = true;
  for (size_t c = 0; c < pal.size(); ++c) {
    vmin = c == 0 ? pal[c] : std::min(vmin, pal[c]);
    vmax = c == 0 ? pal[c] : std::max(vmax, pal[c]);
    vabs = std::max(vabs, std::fabs(pal[c]));
    jump = std::max(jump, std::fabs(pal[c] + 10.0));
    exact = exact && static_cast<double>(static_cast<float>(pal[c])) == pal[c];
    if (!std::isfinite(pal[c])) return VS_OK;  // no screen: non-finite node values
  }
  for (int i = 0; i < 16; ++i) {
    const double a = pal[std::min<size_t>(i & 3, pal.size() - 1)], b = pal[std::min<size_t>(i >> 2, pal.size() - 1)];
    s.pair[2 * i] = static_cast<float>(a);
    s.pair[2 * i + 1] = static_cast<float>(b - a);
  }
  // error model (search.cu screen_sample): Lipschitz constant of the trilinear
  // field summed over the three axes, in cell units; the FP32 lerp tree's
  // rounding (7 u V) plus the table's (3 u V when a value is not FP32-exact),
  // both padded; a uniform cell's FP32 value is exact iff the palette is.
  const double u = std::ldexp(1.0, -24);
  s.G = static_cast<float>(3.0 * (vmax - vmin) * (1.0 + 1e-6));
  s.J = static_cast<float>(jump * (1.0 + 1e-6));
  s.eval = static_cast<float>(12.0 * u * vabs);
  s.uni = exact ? 0.0f : static_cast<float>(2.0 * u * vabs);
  s.v3 = static_cast<float>(3.0 * vabs * (1.0 + 1e-6));
  s.dx1 = static_cast<float>(D0 - 1);
  s.dy1 = static_cast<float>(D1 - 1);
  s.dz1 = static_cast<float>(D2 - 1);
  s.fdx = static_cast<float>(D0);
  s.fdxy = static_cast<float>(static_cast<double>(D0) * D1);
  const size_t nv = static_cast<size_t>(D0) * D1 * D2;
  std::vector<uint32_t> w(nv, 0u);
  auto at = [&](int x, int y, int z) { return code[static_cast<size_t>(x) + static_cast<size_t>(D0) * (y + static_cast<size_t>(D1) * z)]; };
  for (int iz = 0; iz + 1 < D2; ++iz)
    for (int iy = 0; iy + 1 < D1; ++iy)
      for (int ix = 0; ix + 1 < D0; ++ix) {
        uint32_t word = 0;
        for (int i = 0; i < 4; ++i) {
          const int y = iy + (i & 1), z = iz + (i >> 1);
          word |= static_cast<uint32_t>(8 * (at(ix, y, z) | (at(ix + 1, y, z) << 2))) << (8 * i);
        }
        const uint8_t c0 = at(ix, iy, iz);
        bool nu = false;
        for (int z = std::max(iz - 1, 0); z <= std::min(iz + 2, D2 - 1) && !nu; ++z)
          for (int y = std::max(iy - 1, 0); y <= std::min(iy + 2, D1 - 1) && !nu; ++y)
            for (int x = std::max(ix - 1, 0); x <= std::min(ix + 2, D0 - 1); ++x)
              if (at(x, y, z) != c0) {
                nu = true;
                break;
              }
        if (nu) word |= 0x80000000u;
        w[static_cast<size_t>(ix) + static_cast<size_t>(D0) * (iy + static_cast<size_t>(D1) * iz)] = word;
      }
  if (nv >= (1u << 22)) return VS_OK;  // the FP32 cell index needs M + index < 2^24: no screen
  s.last = static_cast<uint32_t>(nv - 1);
  CUDA_TRY(p->screen.ensure(sizeof(uint32_t) * nv));
  CUDA_TRY(cudaMemcpy(p->screen.p, w.data(), sizeof(uint32_t) * nv, cudaMemcpyHostToDevice));
  p->has_screen = true;
  return VS_OK;
}

// Cell-packed palette grid for the search sampler (dmath.cuh): when the node
// values take at most 4 (16) distinct doubles, each cell's 8 corner codes fit
// in one 16-bit (32-bit) word.  Values are reproduced exactly via the palette.
vs_status build_packed(vs_pocket *p, const double *values) {
  p->has_screen = false;
  std::vector<double> pal;
  const size_t nv = static_cast<size_t>(p->dims[0]) * p->dims[1] * p->dims[2];
  std::vector<uint8_t> code(nv);
  for (size_t i = 0; i < nv && pal.size() <= 16; ++i) {
    const double v = values[i];
    size_t c = 0;
    uint64_t vb, pb;
    std::memcpy(&vb, &v, 8);
    for (; c < pal.size(); ++c) {
      std::memcpy(&pb, &pal[c], 8);
      if (pb == vb) break;  // bitwise identity keeps -0.0 / NaN payloads exact
    }
    if (c == pal.size()) pal.push_back(v);
    code[i] = static_cast<uint8_t>(c);
  }
  p->packed_mode = pal.size() <= 4 ? 1 : (pal.size() <= 16 ? 2 : 0);
  std::vector<double> pal16(16, 0.0);
  for (size_t c = 0; c < pal.size() && c < 16; ++c) pal16[c] = pal[c];
  CUDA_TRY(p->palette.ensure(sizeof(double) * 16));
  CUDA_TRY(cudaMemcpy(p->palette.p, pal16.data(), sizeof(double) * 16, cudaMemcpyHostToDevice));
  if (p->packed_mode == 0) return VS_OK;
  const int cx = p->dims[0] - 1, cy = p->dims[1] - 1, cz = p->dims[2] - 1;
  const int bx = (cx + 3) / 4, by = (cy + 3) / 4, bz = (cz + 3) / 4;
  p->bricks[0] = bx;
  p->bricks[1] = by;
  const size_t ncell = static_cast<size_t>(bx) * by * bz * 64;  // 4x4x4 bricks (dmath.cuh cell_index)
  const int bits = p->packed_mode == 1 ? 2 : 4;
  std::vector<uint32_t> words(ncell, 0u);
  for (int iz = 0; iz < cz; ++iz)
    for (int iy = 0; iy < cy; ++iy)
      for (int ix = 0; ix < cx; ++ix) {
        uint32_t w = 0;
        for (int c = 0; c < 8; ++c) {
          const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
          const size_t node = static_cast<size_t>(ix + dx) +
                              static_cast<size_t>(p->dims[0]) * (static_cast<size_t>(iy + dy) +
                                                                 static_cast<size_t>(p->dims[1]) * (iz + dz));
          w |= static_cast<uint32_t>(code[node]) << (bits * c);
        }
        const size_t brick = static_cast<size_t>(ix >> 2) + static_cast<size_t>(bx) *
                                 (static_cast<size_t>(iy >> 2) + static_cast<size_t>(by) * (iz >> 2));
        words[(brick << 6) | ((iz & 3) << 4) | ((iy & 3) << 2) | (ix & 3)] = w;
      }
  if (p->packed_mode == 1) {
    {
      const vs_status st = build_screen(p, code, pal);
      if (st != VS_OK) return st;
    }
    std::vector<uint16_t> w16(ncell);
    for (size_t i = 0; i < ncell; ++i) w16[i] = static_cast<uint16_t>(words[i]);
    CUDA_TRY(p->packed.ensure(sizeof(uint16_t) * ncell));
    CUDA_TRY(cudaMemcpy(p->packed.p, w16.data(), sizeof(uint16_t) * ncell, cudaMemcpyHostToDevice));
  } else {
    CUDA_TRY(p->packed.ensure(sizeof(uint32_t) * ncell));
    CUDA_TRY(cudaMemcpy(p->packed.p, words.data(), sizeof(uint32_t) * ncell, cudaMemcpyHostToDevice));
  }
  return VS_OK;
}

vs_status upload_protein(vs_pocket *p, int32_t n, const uint8_t *elem, const double *xyz) {
  p->n_protein = n;
  std::vector<uint8_t> cls(static_cast<size_t>(std::max(n, 1)), 2);
  for (int j = 0; j < n; ++j) cls[static_cast<size_t>(j)] = static_cast<uint8_t>(chem_class(elem[j]));
  CUDA_TRY(p->pxyz.ensure(sizeof(double) * 3 * std::max(n, 1)));
  CUDA_TRY(p->pclass.ensure(std::max(n, 1)));
  if (n > 0) {
    CUDA_TRY(cudaMemcpy(p->pxyz.p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(p->pclass.p, cls.data(), static_cast<size_t>(n), cudaMemcpyHostToDevice));
  }
  return build_cells(p, elem, xyz);
}

// One chunk of a ligand batch staged on the device.
struct Staged {
  vsd::batch_dev b{};
  int n = 0;
  int Nmax = 0, nmax = 0, mmax = 0;
  int atoms = 0, torsions = 0;
  std::vector<int> atom_off, bond_off, tors_off, right_off, ditem_base;
  std::vector<int> lN, ln, lm;  // per ligand: atoms, heavy atoms, torsions
};

template <typename T>
vs_status h2d(DevBuf &buf, const T *src, size_t count, cudaStream_t s) {
  CUDA_TRY(buf.ensure(sizeof(T) * std::max<size_t>(count, 1)));
  if (count) CUDA_TRY(cudaMemcpyAsync(buf.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  return VS_OK;
}

// Stage ligands [l0, l1) of `in` (offsets rebased to 0).
vs_status stage(vs_context *ctx, const vs_ligand_batch *in, int l0, int l1, Staged &st) {
  const int n = l1 - l0;
  st.n = n;
  const int A0 = in->atom_offset[l0], A1 = in->atom_offset[l1];
  const int B0 = in->bond_offset[l0], B1 = in->bond_offset[l1];
  const int T0 = in->torsion_offset[l0], T1 = in->torsion_offset[l1];
  const int R0 = in->right_offset[T0], R1 = in->right_offset[T1];
  st.atoms = A1 - A0;
  st.torsions = T1 - T0;
  st.atom_off.resize(n + 1);
  st.bond_off.resize(n + 1);
  st.tors_off.resize(n + 1);
  st.ditem_base.resize(n + 1);
  st.right_off.resize(T1 - T0 + 1);
  st.Nmax = st.nmax = st.mmax = 0;
  st.lN.assign(n, 0);
  st.ln.assign(n, 0);
  st.lm.assign(n, 0);
  int dbase = 0;
  for (int i = 0; i <= n; ++i) {
    st.atom_off[i] = in->atom_offset[l0 + i] - A0;
    st.bond_off[i] = in->bond_offset[l0 + i] - B0;
    st.tors_off[i] = in->torsion_offset[l0 + i] - T0;
    st.ditem_base[i] = dbase;
    if (i < n) {
      const int N = in->atom_offset[l0 + i + 1] - in->atom_offset[l0 + i];
      const int m = in->torsion_offset[l0 + i + 1] - in->torsion_offset[l0 + i];
      int h = 0;
      for (int a = in->atom_offset[l0 + i]; a < in->atom_offset[l0 + i + 1]; ++a) h += in->is_heavy[a] ? 1 : 0;
      st.lN[i] = N;
      st.ln[i] = h;
      st.lm[i] = m;
      if (N <= VS_MAX_ATOMS && m <= VS_MAX_TORSIONS && h <= VS_MAX_HEAVY) {
        st.Nmax = std::max(st.Nmax, N);
        st.mmax = std::max(st.mmax, m);
        st.nmax = std::max(st.nmax, h);
      }
      dbase += std::min(m, VS_MAX_TORSIONS) * std::min(N, VS_MAX_ATOMS);
    }
  }
  for (int t = 0; t <= T1 - T0; ++t) st.right_off[t] = in->right_offset[T0 + t] - R0;
  cudaStream_t s = ctx->stream;
  vs_status rc;
  if ((rc = h2d(ctx->atom_off, st.atom_off.data(), n + 1, s))) return rc;
  if ((rc = h2d(ctx->bond_off, st.bond_off.data(), n + 1, s))) return rc;
  if ((rc = h2d(ctx->tors_off, st.tors_off.data(), n + 1, s))) return rc;
  if ((rc = h2d(ctx->ditem_base, st.ditem_base.data(), n + 1, s))) return rc;
  if ((rc = h2d(ctx->right_off, st.right_off.data(), T1 - T0 + 1, s))) return rc;
  if ((rc = h2d(ctx->xyz, in->xyz + 3 * static_cast<size_t>(A0), 3 * static_cast<size_t>(A1 - A0), s))) return rc;
  if ((rc = h2d(ctx->elem, in->element + A0, A1 - A0, s))) return rc;
  if ((rc = h2d(ctx->heavy, in->is_heavy + A0, A1 - A0, s))) return rc;
  if ((rc = h2d(ctx->bond_a, in->bond_a + B0, B1 - B0, s))) return rc;
  if ((rc = h2d(ctx->bond_b, in->bond_b + B0, B1 - B0, s))) return rc;
  if ((rc = h2d(ctx->tors_bond, in->torsion_bond + T0, T1 - T0, s))) return rc;
  if ((rc = h2d(ctx->right_atoms, in->right_atoms + R0, R1 - R0, s))) return rc;
  const size_t na = std::max(st.atoms, 1), nt = std::max(st.torsions, 1);
  CUDA_TRY(ctx->meta.ensure(sizeof(vsd::lig_meta) * std::max(n, 1)));
  CUDA_TRY(ctx->tmask.ensure(4 * na));
  CUDA_TRY(ctx->heavy_list.ensure(2 * na));
  CUDA_TRY(ctx->dmask.ensure(4 * na));
  CUDA_TRY(ctx->tors_a.ensure(2 * nt));
  CUDA_TRY(ctx->tors_b.ensure(2 * nt));
  CUDA_TRY(ctx->d_count.ensure(4 * nt));
  CUDA_TRY(ctx->d_off.ensure(4 * nt));
  CUDA_TRY(ctx->ditems.ensure(2 * static_cast<size_t>(std::max(dbase, 1))));
  CUDA_TRY(ctx->titems.ensure(8 * static_cast<size_t>(std::max(dbase, 1))));
  vsd::batch_dev &b = st.b;
  b.n_lig = n;
  b.atom_off = ctx->atom_off.as<int>();
  b.bond_off = ctx->bond_off.as<int>();
  b.tors_off = ctx->tors_off.as<int>();
  b.ditem_base = ctx->ditem_base.as<int>();
  b.xyz = ctx->xyz.as<double>();
  b.elem = ctx->elem.as<uint8_t>();
  b.heavy = ctx->heavy.as<uint8_t>();
  b.bond_a = ctx->bond_a.as<uint16_t>();
  b.bond_b = ctx->bond_b.as<uint16_t>();
  b.tors_bond = ctx->tors_bond.as<uint16_t>();
  b.right_off = ctx->right_off.as<int>();
  b.right_atoms = ctx->right_atoms.as<uint16_t>();
  b.meta = ctx->meta.as<vsd::lig_meta>();
  b.atom_tmask = ctx->tmask.as<uint32_t>();
  b.heavy_list = ctx->heavy_list.as<uint16_t>();
  b.heavy_dmask = ctx->dmask.as<uint32_t>();
  b.tors_a = ctx->tors_a.as<uint16_t>();
  b.tors_b = ctx->tors_b.as<uint16_t>();
  b.d_count = ctx->d_count.as<int>();
  b.d_off = ctx->d_off.as<int>();
  b.ditems = ctx->ditems.as<uint16_t>();
  b.titems = ctx->titems.as<uint32_t>();
  return VS_OK;
}

// Host tables of input-independent rotations (glibc trig, as the reference).
// spin: per step level L (step_rotation halved L times, search.cpp:188),
// per neighbour (axis x/y/z, sign +/-), Quaterniond(AngleAxisd(sign*step,
// Unit(axis))) (search.cpp:162-163, Appendix A item 1).
int spin_levels(const vs_scoring_config &c) {
  int levels = 0;
  double st = c.step_translation;
  while (levels < c.max_iterations && st >= c.min_translation && levels < 4096) {
    st *= 0.5;
    ++levels;
  }
  return std::max(levels, 1);
}
void spin_table(const vs_scoring_config &c, int levels, std::vector<double> &out) {
  out.assign(static_cast<size_t>(levels) * 6 * 4, 0.0);
  double step_r = c.step_rotation;
  for (int L = 0; L < levels; ++L) {
    for (int axis = 0; axis < 3; ++axis)
      for (int sgn = 0; sgn < 2; ++sgn) {
        const double sign = sgn ? -1.0 : 1.0;
        const double ha = 0.5 * (sign * step_r);
        const double w = std::cos(ha), s = std::sin(ha);
        const double u[3] = {axis == 0 ? 1.0 : 0.0, axis == 1 ? 1.0 : 0.0, axis == 2 ? 1.0 : 0.0};
        double *q = &out[(static_cast<size_t>(L) * 6 + axis * 2 + sgn) * 4];
        q[0] = s * u[0];
        q[1] = s * u[1];
        q[2] = s * u[2];
        q[3] = w;
      }
    step_r *= 0.5;
  }
}
// fibonacci_axis / fibonacci_rotation_angle / Quaterniond(AngleAxisd)
// (search.cpp:71-82, 97-98).
void fib_table(int k, std::vector<double> &out) {
  constexpr double kGoldenRatio = 1.6180339887498948482;
  constexpr double kGoldenAngle = 2.0 * kPi * (2.0 - kGoldenRatio);
  out.assign(static_cast<size_t>(k) * 4, 0.0);
  for (int i = 0; i < k; ++i) {
    const double z = 1.0 - 2.0 * (i + 0.5) / static_cast<double>(k);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double az = std::fmod(i * kGoldenAngle, 2.0 * kPi);
    const double ax[3] = {r * std::cos(az), r * std::sin(az), z};
    const double angle = 2.0 * kPi * std::fmod(i * kGoldenRatio, 1.0);
    const double ha = 0.5 * angle;
    const double w = std::cos(ha), s = std::sin(ha);
    out[4 * i] = s * ax[0];
    out[4 * i + 1] = s * ax[1];
    out[4 * i + 2] = s * ax[2];
    out[4 * i + 3] = w;
  }
}

vs_status check_cfg(const vs_scoring_config *cfg) {
  if (!cfg) return fail(VS_ERR_INVALID_ARGUMENT, "null scoring config");
  if (cfg->restarts < 1) return fail(VS_ERR_INVALID_ARGUMENT, "restarts must be at least 1");
  if (cfg->rescored < 1) return fail(VS_ERR_INVALID_ARGUMENT, "rescored must be at least 1");
  if (!(cfg->rmsd_threshold > 0.0)) return fail(VS_ERR_INVALID_ARGUMENT, "rmsd threshold must be positive");
  if (cfg->restarts > VS_MAX_RESTARTS) return fail(VS_ERR_LIMIT, "restarts exceed VS_MAX_RESTARTS");
  return VS_OK;
}

// k_flatten's shared memory is 37 copies of a ligand's coordinates, sized by
// the largest ligand of the launch: ligands are launched in atom-count
// buckets so small ligands get more resident CTAs per SM.
vs_status flatten_buckets(vs_context *ctx, const Staged &st, int max_sweeps, const vsd::flat_out &f) {
  static const int kLimits[] = {40, 48, 56, 64, 72, 80, 96, 128, 1 << 30};
  constexpr int kB = sizeof(kLimits) / sizeof(kLimits[0]);
  std::vector<int> order;
  order.reserve(static_cast<size_t>(st.n));
  int start[kB + 1] = {0}, nmax[kB] = {0};
  for (int bi = 0; bi < kB; ++bi) {
    start[bi] = static_cast<int>(order.size());
    const int lo = bi ? kLimits[bi - 1] : 0;
    for (int i = 0; i < st.n; ++i)
      if (st.lN[i] > lo && st.lN[i] <= kLimits[bi]) {
        order.push_back(i);
        nmax[bi] = std::max(nmax[bi], st.lN[i]);
      }
  }
  start[kB] = static_cast<int>(order.size());  // (N == 0 ligands: rejected by k_setup, no flatten)
  vs_status rc;
  if ((rc = h2d(ctx->flat_index, order.data(), order.size(), ctx->stream))) return rc;
  for (int bi = 0; bi < kB; ++bi) {
    const int cnt = start[bi + 1] - start[bi];
    if (cnt == 0) continue;
    CUDA_TRY(vsd::launch_flatten(st.b, max_sweeps, f, std::max(nmax[bi], 1), st.mmax, ctx->stream,
                                 ctx->flat_index.as<int>() + start[bi], cnt));
    ++ctx->last_launches;
  }
  --ctx->last_launches;  // one flatten launch is counted with the fixed stages
  return VS_OK;
}

vs_status upload_tables(vs_context *ctx, const vs_scoring_config &c, int k, vsd::search_cfg &sc) {
  std::vector<double> spin, fib, stepsc;
  const int levels = spin_levels(c);
  spin_table(c, levels, spin);
  // double-double sin/cos of the torsion step at each level (the search's
  // incremental neighbour trig, vs_crtrig.h sincos_shift)
  stepsc.resize(4 * static_cast<size_t>(levels));
  double dq = c.step_torsion;
  for (int L = 0; L < levels; ++L, dq *= 0.5) {
    vs_crtrig::dd s, cc;
    vs_crtrig::sincos_dd(dq, &s, &cc);
    stepsc[4 * L] = s.hi;
    stepsc[4 * L + 1] = s.lo;
    stepsc[4 * L + 2] = cc.hi;
    stepsc[4 * L + 3] = cc.lo;
  }
  fib_table(k, fib);
  vs_status rc;
  if ((rc = h2d(ctx->spin, spin.data(), spin.size(), ctx->stream))) return rc;
  if ((rc = h2d(ctx->fibq, fib.data(), fib.size(), ctx->stream))) return rc;
  if ((rc = h2d(ctx->stepsc, stepsc.data(), stepsc.size(), ctx->stream))) return rc;
  sc.k = k;
  sc.rescored = c.rescored;
  sc.rmsd_threshold = c.rmsd_threshold;
  sc.max_iter = c.max_iterations;
  sc.step_t = c.step_translation;
  sc.step_r = c.step_rotation;
  sc.step_q = c.step_torsion;
  sc.min_t = c.min_translation;
  sc.flatten_sweeps = c.flatten_max_sweeps;
  sc.n_levels = levels;
  sc.spin = ctx->spin.as<double>();
  sc.fibq = ctx->fibq.as<double>();
  sc.stepsc = ctx->stepsc.as<double>();
  // The stream must not outlive the host vectors' copies.
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return VS_OK;
}

// Chunk boundaries so that the per-restart conformation scratch stays under
// `budget` bytes.
std::vector<int> chunks(const vs_ligand_batch *b, int k, size_t budget) {
  std::vector<int> cut{0};
  size_t acc = 0;
  for (int i = 0; i < b->n_ligands; ++i) {
    const size_t N = static_cast<size_t>(b->atom_offset[i + 1] - b->atom_offset[i]);
    const size_t need = N * k * 3 * sizeof(double) + 256 * static_cast<size_t>(k);
    if (acc + need > budget && i > cut.back()) {
      cut.push_back(i);
      acc = 0;
    }
    acc += need;
  }
  cut.push_back(b->n_ligands);
  return cut;
}

vs_status ensure_items(vs_context *ctx, const Staged &st, int k, vsd::item_out &o) {
  const size_t items = static_cast<size_t>(std::max(st.n, 1)) * k;
  CUDA_TRY(ctx->out_geo.ensure(sizeof(double) * items));
  CUDA_TRY(ctx->out_T.ensure(sizeof(double) * 7 * items));
  CUDA_TRY(ctx->out_ang.ensure(sizeof(double) * std::max<size_t>(1, static_cast<size_t>(st.torsions) * k)));
  CUDA_TRY(ctx->out_conf.ensure(sizeof(double) * 3 * std::max<size_t>(1, static_cast<size_t>(st.atoms) * k)));
  CUDA_TRY(ctx->out_evals.ensure(sizeof(unsigned long long) * items));
  CUDA_TRY(ctx->out_status.ensure(sizeof(int) * items));
  CUDA_TRY(ctx->out_iters.ensure(sizeof(int) * items));
  CUDA_TRY(ctx->out_adopts.ensure(sizeof(int) * items));
  CUDA_TRY(ctx->work.ensure(sizeof(int) * 4));
  o.geo = ctx->out_geo.as<double>();
  o.T = ctx->out_T.as<double>();
  o.ang = ctx->out_ang.as<double>();
  o.conf = ctx->out_conf.as<double>();
  o.evals = ctx->out_evals.as<unsigned long long>();
  o.status = ctx->out_status.as<int>();
  o.iters = ctx->out_iters.as<int>();
  o.adopts = ctx->out_adopts.as<int>();
  return VS_OK;
}

vs_status ensure_flat(vs_context *ctx, const Staged &st, vsd::flat_out &f) {
  CUDA_TRY(ctx->flat_idx.ensure(sizeof(int) * std::max(st.torsions, 1)));
  CUDA_TRY(ctx->flat_xyz.ensure(sizeof(double) * 3 * std::max(st.atoms, 1)));
  CUDA_TRY(ctx->flat_centroid.ensure(sizeof(double) * 3 * std::max(st.n, 1)));
  CUDA_TRY(ctx->flat_sweeps.ensure(sizeof(int) * std::max(st.n, 1)));
  f.sweeps = ctx->flat_sweeps.as<int>();
  f.idx = ctx->flat_idx.as<int>();
  f.xyz = ctx->flat_xyz.as<double>();
  f.centroid = ctx->flat_centroid.as<double>();
  return VS_OK;
}

struct CtxLock {
  vs_context *c;
  explicit CtxLock(vs_context *ctx) : c(ctx) {
    c->mu.lock();
    cudaSetDevice(c->device);
  }
  ~CtxLock() { c->mu.unlock(); }
};

}  // namespace

extern "C" {

int vs_abi_version(void) { return VS_ABI_VERSION; }

int vs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char *vs_last_error_message(void) { return g_err.c_str(); }

// Host-side components of the library (host/rank.cpp) report errors through
// the same thread-local message.
vs_status vs_internal_fail(vs_status s, const char *msg) { return fail(s, msg ? msg : ""); }

vs_status vs_host_alloc(size_t bytes, void **out) {
  if (!out) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  CUDA_TRY(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable));
  return VS_OK;
}

void vs_host_free(void *p) {
  if (p) cudaFreeHost(p);
}

void vs_scoring_config_default(vs_scoring_config *c) {
  c->restarts = 256;
  c->rescored = 30;
  c->rmsd_threshold = 3.0;
  c->step_translation = 1.0;
  c->step_rotation = 20.0 * (kPi / 180.0);
  c->step_torsion = 20.0 * (kPi / 180.0);
  c->min_translation = 0.1;
  c->max_iterations = 200;
  c->flatten_max_sweeps = 20;
}

vs_status vs_context_create(int device, vs_context **out) {
  if (!out) return fail(VS_ERR_INVALID_ARGUMENT, "null output");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(VS_ERR_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(VS_ERR_INVALID_ARGUMENT, "device index out of range");
  CUDA_TRY(cudaSetDevice(device));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) return fail(VS_ERR_NO_DEVICE, "libvsdock is built for sm_100a (B200) only");
  auto *ctx = new vs_context;
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return fail(VS_ERR_CUDA, "stream creation failed");
  }
  cudaEventCreate(&ctx->ev0);
  cudaEventCreate(&ctx->ev1);
  for (auto &e : ctx->evs) cudaEventCreate(&e);
  cudaEventCreate(&ctx->ev_flat);
  ensure_lattice(device);
  {
    // eager module load per device, once per process: concurrent first
    // launches from several host threads on a fresh device (the rank's CUDA
    // workers) raced inside CUDA's lazy loading
    static std::mutex mu;
    static bool loaded[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (!loaded[device & 63]) {
      vsd::preload_kernels();
      loaded[device & 63] = true;
    }
  }
  *out = ctx;
  return VS_OK;
}

vs_status vs_context_destroy(vs_context *ctx) {
  if (!ctx) return VS_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  for (auto &e : ctx->evs) cudaEventDestroy(e);
  cudaEventDestroy(ctx->ev_flat);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return VS_OK;
}

vs_status vs_context_last_timing(vs_context *ctx, double *kernel_ms, int32_t *launches) {
  if (!ctx) return fail(VS_ERR_INVALID_ARGUMENT, "null context");
  if (kernel_ms) *kernel_ms = ctx->last_ms;
  if (launches) *launches = ctx->last_launches;
  return VS_OK;
}

vs_status vs_context_stage_timing(vs_context *ctx, double stage_ms[4]) {
  if (!ctx || !stage_ms) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < 4; ++i) stage_ms[i] = ctx->stage_ms[i];
  return VS_OK;
}

vs_status vs_pocket_create(vs_context *ctx, const vs_pocket_desc *d, vs_pocket **out) {
  if (!ctx || !d || !out) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  for (int a = 0; a < 3; ++a)
    if (d->dims[a] < 2) return fail(VS_ERR_INVALID_ARGUMENT, "every pocket dimension must be at least 2");
  if (!(d->spacing > 0.0)) return fail(VS_ERR_INVALID_ARGUMENT, "pocket spacing must be positive");
  CtxLock lock(ctx);
  auto *p = new vs_pocket;
  p->device = ctx->device;
  for (int a = 0; a < 3; ++a) {
    p->origin[a] = d->origin[a];
    p->dims[a] = d->dims[a];
  }
  p->spacing = d->spacing;
  const size_t nv = static_cast<size_t>(d->dims[0]) * d->dims[1] * d->dims[2];
  vs_status rc = VS_OK;
  if (p->values.ensure(sizeof(double) * nv) != cudaSuccess ||
      cudaMemcpy(p->values.p, d->values, sizeof(double) * nv, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(VS_ERR_CUDA, "pocket grid upload failed");
  if (rc == VS_OK) rc = build_packed(p, d->values);
  if (rc == VS_OK) rc = upload_protein(p, d->n_protein, d->protein_element, d->protein_xyz);
  if (rc != VS_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return VS_OK;
}

vs_status vs_pocket_build(vs_context *ctx, int32_t n, const uint8_t *elem, const double *xyz, const double center[3],
                          double radius, double spacing, vs_pocket **out) {
  if (!ctx || !out || !center) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  // Preconditions of build_pocket (grid.cpp:18-25).
  if (radius <= 0.0) return fail(VS_ERR_INVALID_ARGUMENT, "pocket radius must be positive");
  if (spacing < 0.25 || spacing > 1.0) return fail(VS_ERR_INVALID_ARGUMENT, "pocket spacing must lie in [0.25, 1.0]");
  std::vector<double> heavy;
  for (int j = 0; j < n; ++j)
    if (elem[j] != VS_ELEM_H) heavy.insert(heavy.end(), xyz + 3 * j, xyz + 3 * j + 3);
  if (heavy.empty()) return fail(VS_ERR_INVALID_ARGUMENT, "protein has no heavy atoms");
  const int steps = static_cast<int>(std::ceil(2.0 * radius / spacing));
  const int dim = steps + 1;
  if (static_cast<int64_t>(dim) * dim * dim > (int64_t(1) << 27)) return fail(VS_ERR_LIMIT, "pocket grid too large");
  CtxLock lock(ctx);
  auto *p = new vs_pocket;
  p->device = ctx->device;
  p->spacing = spacing;
  for (int a = 0; a < 3; ++a) {
    p->origin[a] = center[a] - radius;  // center - Constant(radius)
    p->dims[a] = dim;
  }
  const size_t nv = static_cast<size_t>(dim) * dim * dim;
  DevBuf hx;
  vs_status rc = VS_OK;
  if (p->values.ensure(sizeof(double) * nv) != cudaSuccess || hx.ensure(sizeof(double) * heavy.size()) != cudaSuccess ||
      cudaMemcpy(hx.p, heavy.data(), sizeof(double) * heavy.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(VS_ERR_CUDA, "pocket build upload failed");
  if (rc == VS_OK) {
    cudaError_t e = vsd::launch_build_pocket(hx.as<double>(), static_cast<int>(heavy.size() / 3), center[0], center[1],
                                             center[2], radius, p->origin[0], p->origin[1], p->origin[2], spacing, dim,
                                             dim, dim, p->values.as<double>(), ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(VS_ERR_CUDA, cudaGetErrorString(e));
  }
  if (rc == VS_OK) {
    std::vector<double> vals(nv);
    if (cudaMemcpy(vals.data(), p->values.p, sizeof(double) * nv, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = fail(VS_ERR_CUDA, "pocket grid download failed");
    else
      rc = build_packed(p, vals.data());
  }
  if (rc == VS_OK) rc = upload_protein(p, n, elem, xyz);
  if (rc != VS_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return VS_OK;
}

vs_status vs_pocket_info(const vs_pocket *p, double origin[3], double *spacing, int32_t dims[3], int32_t *n_protein) {
  if (!p) return fail(VS_ERR_INVALID_ARGUMENT, "null pocket");
  for (int a = 0; a < 3; ++a) {
    if (origin) origin[a] = p->origin[a];
    if (dims) dims[a] = p->dims[a];
  }
  if (spacing) *spacing = p->spacing;
  if (n_protein) *n_protein = p->n_protein;
  return VS_OK;
}

vs_status vs_pocket_download(vs_context *ctx, const vs_pocket *p, double *values) {
  if (!ctx || !p || !values) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  const size_t nv = static_cast<size_t>(p->dims[0]) * p->dims[1] * p->dims[2];
  CUDA_TRY(cudaMemcpy(values, p->values.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
  return VS_OK;
}

vs_status vs_pocket_destroy(vs_pocket *p) {
  if (!p) return VS_OK;
  cudaSetDevice(p->device);
  delete p;
  return VS_OK;
}

vs_status vs_dock_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                        const vs_scoring_config *cfg, vs_dock_result *results, double *best_angles,
                        double *best_conformation) {
  return vs_dock_batch_ex(ctx, pocket, batch, cfg, results, best_angles, best_conformation, nullptr);
}

// The dock path over n_pockets pockets: setup and flatten run once per chunk
// (they depend on the ligands only), then search + select per pocket.
// results / best_angles / best_conformation / counters are arrays of
// n_pockets pointers (entries may be NULL except results).
static vs_status check_pockets(const vs_context *ctx, const vs_pocket *const *pockets, int n_pockets) {
  for (int pi = 0; pi < n_pockets; ++pi)
    if (!pockets[pi]) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
    else if (pockets[pi]->device != ctx->device) return fail(VS_ERR_INVALID_ARGUMENT, "pocket lives on another device");
  return VS_OK;
}

// `pre`: a batch already staged on the device (vs_dock_records); else the
// host batch is staged chunk by chunk.  The caller holds the context lock.
static vs_status dock_impl(vs_context *ctx, const vs_pocket *const *pockets, int n_pockets,
                           const vs_ligand_batch *batch, const vs_scoring_config *cfg, vs_dock_result *const *results_p,
                           double *const *best_angles_p, double *const *best_conf_p, uint64_t *const *counters_p,
                           Staged *pre = nullptr) {
  vs_status rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_pockets(ctx, pockets, n_pockets))) return rc;
  for (int pi = 0; pi < n_pockets; ++pi)
    if (!results_p[pi]) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  const int k = cfg->restarts;
  vsd::search_cfg sc{};
  if ((rc = upload_tables(ctx, *cfg, k, sc))) return rc;
  ctx->last_launches = 0;
  for (double &x : ctx->stage_ms) x = 0.0;
  float total_ms = 0.0f;
  const std::vector<int> cut = pre ? std::vector<int>{0, pre->n} : chunks(batch, k, size_t(32) << 30);
  for (size_t ci = 0; ci + 1 < cut.size(); ++ci) {
    const int l0 = cut[ci], l1 = cut[ci + 1];
    Staged st_local;
    Staged &st = pre ? *pre : st_local;
    if (!pre && (rc = stage(ctx, batch, l0, l1, st))) return rc;
    vsd::flat_out f{};
    vsd::item_out o{};
    if ((rc = ensure_flat(ctx, st, f))) return rc;
    if ((rc = ensure_items(ctx, st, k, o))) return rc;
    o.heavy_conf = 1;
    CUDA_TRY(ctx->results.ensure(sizeof(vs_dock_result) * std::max(st.n, 1)));
    CUDA_TRY(ctx->best_ang.ensure(sizeof(double) * std::max(st.torsions, 1)));
    CUDA_TRY(ctx->best_conf.ensure(sizeof(double) * 3 * std::max(st.atoms, 1)));
    CUDA_TRY(ctx->best_idx.ensure(sizeof(int) * std::max(st.n, 1)));
    CUDA_TRY(ctx->counters.ensure(sizeof(uint64_t) * 9 * std::max(st.n, 1)));
    CUDA_TRY(cudaMemsetAsync(ctx->work.p, 0, sizeof(int), ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->evs[0], ctx->stream));
    CUDA_TRY(vsd::launch_setup(st.b, k, ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->evs[1], ctx->stream));
    // per-ligand sizes for the search buckets come back while flatten runs
    std::vector<vsd::lig_meta> meta(static_cast<size_t>(std::max(st.n, 1)));
    CUDA_TRY(cudaMemcpyAsync(meta.data(), st.b.meta, sizeof(vsd::lig_meta) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    if ((rc = flatten_buckets(ctx, st, cfg->flatten_max_sweeps, f))) return rc;
    CUDA_TRY(cudaEventRecord(ctx->evs[2], ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->ev_flat, ctx->stream));
    CUDA_TRY(ctx->search_args.ensure(vsd::search_scratch_bytes(std::max(st.Nmax, 1), std::max(st.nmax, 1), std::max(st.mmax, 1), ctx->num_sms)));
    CUDA_TRY(cudaEventSynchronize(ctx->ev1));
    float pocket_ms[2] = {0.0f, 0.0f};  // search, select summed over the pockets
    for (int pi = 0; pi < n_pockets; ++pi) {
    const vsd::pocket_dev pd = pockets[pi]->dev();
    vs_dock_result *results = results_p[pi];
    double *best_angles = best_angles_p ? best_angles_p[pi] : nullptr;
    double *best_conformation = best_conf_p ? best_conf_p[pi] : nullptr;
    uint64_t *counters = counters_p ? counters_p[pi] : nullptr;
    vsd::dock_out d{ctx->results.p, ctx->best_ang.as<double>(), ctx->best_conf.as<double>(),
                    counters ? ctx->counters.as<unsigned long long>() : nullptr, f.sweeps,
                    ctx->best_idx.as<int>()};
    if (pi > 0) CUDA_TRY(cudaEventRecord(ctx->evs[2], ctx->stream));
    {
      // Size buckets: ligands grouped by how many 4-warp search CTAs per SM
      // their shared-memory footprint allows, each bucket launched with its
      // own maxima so one large ligand does not shrink everyone's occupancy.
      // bucket = CTAs per SM the ligand's own footprint allows (1..8+), the
      // last bucket holds the ligands k_setup rejected (status only)
      constexpr int kBuckets = 10;
      std::vector<std::vector<int>> buckets(kBuckets);
      const bool screen = pd.scr.w != nullptr && pd.packed.mode == 1;
      for (int i = 0; i < st.n; ++i) {
        const vsd::lig_meta &mt = meta[static_cast<size_t>(i)];
        if (mt.status != VS_LIG_OK) {
          buckets[kBuckets - 1].push_back(i);
          continue;
        }
        const size_t bytes = vsd::search_smem_bytes(mt.n_atoms, mt.n_heavy, mt.m, mt.d_total, screen) + 1024;
        const int ctas = static_cast<int>((228 * 1024) / std::max<size_t>(bytes, 1));
        buckets[std::max(0, std::min(ctas, 8) - 1)].push_back(i);
      }
      std::vector<int> order;
      std::vector<std::pair<int, int>> ranges;
      for (auto &bk : buckets) {
        ranges.push_back({static_cast<int>(order.size()), static_cast<int>(bk.size())});
        order.insert(order.end(), bk.begin(), bk.end());
      }
      if ((rc = h2d(ctx->lig_index, order.data(), order.size(), ctx->stream))) return rc;
      for (size_t bi = 0; bi < buckets.size(); ++bi) {
        if (buckets[bi].empty()) continue;
        int Nm = 1, nm = 1, mm = 1, dm = 1;
        for (int i : buckets[bi]) {
          const vsd::lig_meta &mt = meta[static_cast<size_t>(i)];
          if (mt.status != VS_LIG_OK) continue;
          Nm = std::max(Nm, mt.n_atoms);
          nm = std::max(nm, mt.n_heavy);
          mm = std::max(mm, mt.m);
          dm = std::max(dm, mt.d_total);
        }
        CUDA_TRY(cudaMemsetAsync(ctx->work.p, 0, sizeof(int), ctx->stream));
        CUDA_TRY(vsd::launch_search(st.b, pd, sc, f, o, ctx->work.as<int>(), Nm, nm, mm, ctx->num_sms, ctx->stream,
                                    nullptr, ctx->search_args.p, ctx->lig_index.as<int>() + ranges[bi].first,
                                    ranges[bi].second, dm));
        ++ctx->last_launches;
      }
      --ctx->last_launches;  // counted once below with the fixed launches
    }
    CUDA_TRY(cudaEventRecord(ctx->evs[3], ctx->stream));
    if (const size_t sb = vsd::select_scratch_bytes(st.n, k)) CUDA_TRY(ctx->sel_scratch.ensure(sb));
    CUDA_TRY(vsd::launch_select(st.b, pd, sc, o, d, st.Nmax, ctx->stream, ctx->sel_scratch.as<int>()));
    CUDA_TRY(cudaEventRecord(ctx->evs[4], ctx->stream));
    ctx->last_launches += (pi == 0 ? 4 : 2) + 1;  // + k_best_conf (d.best_conf is always set)
    CUDA_TRY(cudaMemcpyAsync(results + l0, ctx->results.p, sizeof(vs_dock_result) * st.n, cudaMemcpyDeviceToHost,
                             ctx->stream));
    const int T0 = batch ? batch->torsion_offset[l0] : 0, A0 = batch ? batch->atom_offset[l0] : 0;
    if (best_angles && st.torsions)
      CUDA_TRY(cudaMemcpyAsync(best_angles + T0, ctx->best_ang.p, sizeof(double) * st.torsions, cudaMemcpyDeviceToHost,
                               ctx->stream));
    if (best_conformation && st.atoms)
      CUDA_TRY(cudaMemcpyAsync(best_conformation + 3 * static_cast<size_t>(A0), ctx->best_conf.p,
                               sizeof(double) * 3 * st.atoms, cudaMemcpyDeviceToHost, ctx->stream));
    if (counters)
      CUDA_TRY(cudaMemcpyAsync(counters + 9 * static_cast<size_t>(l0), ctx->counters.p, sizeof(uint64_t) * 9 * st.n,
                               cudaMemcpyDeviceToHost, ctx->stream));
    if (n_pockets > 1) {  // per-pocket stage times (the events are reused by the next pocket)
      CUDA_TRY(cudaEventSynchronize(ctx->evs[4]));
      float a = 0.0f, b2 = 0.0f;
      cudaEventElapsedTime(&a, ctx->evs[2], ctx->evs[3]);
      cudaEventElapsedTime(&b2, ctx->evs[3], ctx->evs[4]);
      pocket_ms[0] += a;
      pocket_ms[1] += b2;
    }
    }  // pockets
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    float st_ms[4] = {0, 0, 0, 0};
    cudaEventElapsedTime(&st_ms[0], ctx->evs[0], ctx->evs[1]);
    cudaEventElapsedTime(&st_ms[1], ctx->evs[1], ctx->ev_flat);
    if (n_pockets > 1) {
      st_ms[2] = pocket_ms[0];
      st_ms[3] = pocket_ms[1];
    } else {
      cudaEventElapsedTime(&st_ms[2], ctx->evs[2], ctx->evs[3]);
      cudaEventElapsedTime(&st_ms[3], ctx->evs[3], ctx->evs[4]);
    }
    for (int i = 0; i < 4; ++i) ctx->stage_ms[i] += st_ms[i];
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ctx->evs[0], ctx->evs[4]);
    total_ms += ms;
  }
  ctx->last_ms = total_ms;
  return VS_OK;
}

vs_status vs_dock_batch_ex(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                           const vs_scoring_config *cfg, vs_dock_result *results, double *best_angles,
                           double *best_conformation, uint64_t *counters) {
  if (!ctx || !pocket || !batch || !results) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  return dock_impl(ctx, &pocket, 1, batch, cfg, &results, &best_angles, &best_conformation, &counters);
}

vs_status vs_dock_batch_multi(vs_context *ctx, const vs_pocket *const *pockets, int32_t n_pockets,
                              const vs_ligand_batch *batch, const vs_scoring_config *cfg, vs_dock_result *results) {
  if (!ctx || !pockets || n_pockets < 1 || !batch || !results) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<vs_dock_result *> res(static_cast<size_t>(n_pockets));
  for (int p = 0; p < n_pockets; ++p) res[p] = results + static_cast<size_t>(p) * batch->n_ligands;
  CtxLock lock(ctx);
  return dock_impl(ctx, pockets, n_pockets, batch, cfg, res.data(), nullptr, nullptr, nullptr);
}

vs_status vs_field_values(vs_context *ctx, const vs_pocket *pocket, int64_t n, const double *xyz, double *out) {
  if (!ctx || !pocket || (n > 0 && (!xyz || !out))) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  vs_status rc;
  if ((rc = h2d(ctx->aux0, xyz, 3 * static_cast<size_t>(n), ctx->stream))) return rc;
  CUDA_TRY(ctx->aux1.ensure(sizeof(double) * std::max<int64_t>(n, 1)));
  CUDA_TRY(vsd::launch_field_values(pocket->dev(), n, ctx->aux0.as<double>(), ctx->aux1.as<double>(), ctx->stream));
  if (n) CUDA_TRY(cudaMemcpyAsync(out, ctx->aux1.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return VS_OK;
}

vs_status vs_geo_score_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                             const double *conformation, double *out, uint64_t *evals) {
  if (!ctx || !pocket || !batch || !conformation || !out) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  Staged st;
  vs_status rc;
  if ((rc = stage(ctx, batch, 0, batch->n_ligands, st))) return rc;
  if ((rc = h2d(ctx->aux0, conformation, 3 * static_cast<size_t>(st.atoms), ctx->stream))) return rc;
  CUDA_TRY(ctx->aux1.ensure(sizeof(double) * std::max(st.n, 1)));
  CUDA_TRY(ctx->aux2.ensure(sizeof(unsigned long long) * std::max(st.n, 1)));
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  CUDA_TRY(vsd::launch_geo_score(st.b, pocket->dev(), ctx->aux0.as<double>(), ctx->aux1.as<double>(),
                                 ctx->aux2.as<unsigned long long>(), ctx->stream));
  if (st.n) {
    CUDA_TRY(cudaMemcpyAsync(out, ctx->aux1.p, sizeof(double) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
    if (evals) CUDA_TRY(cudaMemcpyAsync(evals, ctx->aux2.p, sizeof(uint64_t) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return VS_OK;
}

vs_status vs_chem_score_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                              const double *conformation, double *out) {
  if (!ctx || !pocket || !batch || !conformation || !out) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  Staged st;
  vs_status rc;
  if ((rc = stage(ctx, batch, 0, batch->n_ligands, st))) return rc;
  if ((rc = h2d(ctx->aux0, conformation, 3 * static_cast<size_t>(st.atoms), ctx->stream))) return rc;
  CUDA_TRY(ctx->aux1.ensure(sizeof(double) * std::max(st.n, 1)));
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  CUDA_TRY(vsd::launch_chem_score(st.b, pocket->dev(), ctx->aux0.as<double>(), ctx->aux1.as<double>(), ctx->stream));
  if (st.n) CUDA_TRY(cudaMemcpyAsync(out, ctx->aux1.p, sizeof(double) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return VS_OK;
}

vs_status vs_flatten_batch(vs_context *ctx, const vs_ligand_batch *batch, int32_t max_sweeps, double *conformation_out,
                           double *angles_out, int32_t *status_out) {
  if (!ctx || !batch || !conformation_out) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  Staged st;
  vs_status rc;
  if ((rc = stage(ctx, batch, 0, batch->n_ligands, st))) return rc;
  vsd::flat_out f{};
  if ((rc = ensure_flat(ctx, st, f))) return rc;
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  if ((rc = flatten_buckets(ctx, st, max_sweeps, f))) return rc;
  std::vector<int> idx(static_cast<size_t>(std::max(st.torsions, 1)));
  std::vector<vsd::lig_meta> meta(static_cast<size_t>(std::max(st.n, 1)));
  if (st.atoms)
    CUDA_TRY(cudaMemcpyAsync(conformation_out, f.xyz, sizeof(double) * 3 * st.atoms, cudaMemcpyDeviceToHost, ctx->stream));
  if (st.torsions)
    CUDA_TRY(cudaMemcpyAsync(idx.data(), f.idx, sizeof(int) * st.torsions, cudaMemcpyDeviceToHost, ctx->stream));
  if (st.n)
    CUDA_TRY(cudaMemcpyAsync(meta.data(), st.b.meta, sizeof(vsd::lig_meta) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  constexpr double step = 2.0 * kPi / 36;  // angles_of, search.cpp:40
  if (angles_out)
    for (int t = 0; t < st.torsions; ++t) angles_out[t] = idx[static_cast<size_t>(t)] * step;
  if (status_out)
    for (int i = 0; i < st.n; ++i) status_out[i] = meta[static_cast<size_t>(i)].status;
  return VS_OK;
}

vs_status vs_initial_poses(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                           const double *flat_angles, int32_t k, vs_pose *poses_out, double *conformations_out,
                           uint64_t *evals, int32_t *status_out) {
  if (!ctx || !pocket || !batch || !poses_out || !conformations_out || batch->n_ligands != 1)
    return fail(VS_ERR_INVALID_ARGUMENT, "initial_poses takes exactly one ligand");
  if (k < 1) return fail(VS_ERR_INVALID_ARGUMENT, "restart count must be at least 1");  // search.cpp:88
  if (k > VS_MAX_RESTARTS) return fail(VS_ERR_LIMIT, "restarts exceed VS_MAX_RESTARTS");
  CtxLock lock(ctx);
  vs_scoring_config c;
  vs_scoring_config_default(&c);
  c.restarts = k;
  vsd::search_cfg sc{};
  vs_status rc;
  if ((rc = upload_tables(ctx, c, k, sc))) return rc;
  Staged st;
  if ((rc = stage(ctx, batch, 0, 1, st))) return rc;
  std::vector<double> fa(static_cast<size_t>(std::max(st.torsions, 1)), 0.0);
  for (int t = 0; t < st.torsions; ++t) fa[static_cast<size_t>(t)] = flat_angles[t];
  if ((rc = h2d(ctx->aux1, fa.data(), fa.size(), ctx->stream))) return rc;
  vsd::item_out o{};
  if ((rc = ensure_items(ctx, st, k, o))) return rc;
  CUDA_TRY(cudaMemsetAsync(ctx->work.p, 0, sizeof(int), ctx->stream));
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  CUDA_TRY(ctx->search_args.ensure(vsd::search_scratch_bytes(std::max(st.Nmax, 1), std::max(st.nmax, 1), std::max(st.mmax, 1), ctx->num_sms)));
  CUDA_TRY(vsd::launch_initial_poses(st.b, pocket->dev(), sc, ctx->aux1.as<double>(), o, ctx->work.as<int>(), st.Nmax,
                                     st.nmax, st.mmax, ctx->num_sms, ctx->stream, ctx->search_args.p));
  std::vector<double> T(static_cast<size_t>(7) * k), geo(static_cast<size_t>(k));
  std::vector<unsigned long long> ev(static_cast<size_t>(k));
  std::vector<int> stat(static_cast<size_t>(k));
  CUDA_TRY(cudaMemcpyAsync(T.data(), o.T, sizeof(double) * 7 * k, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(geo.data(), o.geo, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(ev.data(), o.evals, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(stat.data(), o.status, sizeof(int) * k, cudaMemcpyDeviceToHost, ctx->stream));
  if (st.atoms)
    CUDA_TRY(cudaMemcpyAsync(conformations_out, o.conf, sizeof(double) * 3 * st.atoms * k, cudaMemcpyDeviceToHost,
                             ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  uint64_t total = 0;
  int status = VS_LIG_OK;
  for (int i = 0; i < k; ++i) {
    for (int q = 0; q < 4; ++q) poses_out[i].rotation[q] = T[7 * i + q];
    for (int q = 0; q < 3; ++q) poses_out[i].translation[q] = T[7 * i + 4 + q];
    poses_out[i].geo_score = geo[static_cast<size_t>(i)];
    total += ev[static_cast<size_t>(i)];
    if (stat[static_cast<size_t>(i)] != VS_LIG_OK) status = stat[static_cast<size_t>(i)];
  }
  if (evals) *evals = total;
  if (status_out) *status_out = status;
  return VS_OK;
}

vs_status vs_cluster_select(vs_context *ctx, const vs_ligand_batch *batch, int32_t n_poses, const double *geo,
                            const double *conformations, double threshold, int32_t top, int32_t *order_out,
                            int32_t *count_out) {
  if (!ctx || !batch || !geo || !conformations || !order_out || !count_out || batch->n_ligands != 1)
    return fail(VS_ERR_INVALID_ARGUMENT, "cluster_select takes exactly one ligand");
  if (n_poses < 1) return fail(VS_ERR_INVALID_ARGUMENT, "cannot cluster an empty pose list");  // search.cpp:198
  if (n_poses > 12 * 1024) return fail(VS_ERR_LIMIT, "too many poses for one cluster_select call");
  CtxLock lock(ctx);
  Staged st;
  vs_status rc;
  if ((rc = stage(ctx, batch, 0, 1, st))) return rc;
  if ((rc = h2d(ctx->aux0, geo, static_cast<size_t>(n_poses), ctx->stream))) return rc;
  if ((rc = h2d(ctx->aux1, conformations, 3 * static_cast<size_t>(st.atoms) * n_poses, ctx->stream))) return rc;
  CUDA_TRY(ctx->aux2.ensure(sizeof(int) * (static_cast<size_t>(n_poses) + 1)));
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  std::vector<vsd::lig_meta> meta(1);
  CUDA_TRY(cudaMemcpyAsync(meta.data(), st.b.meta, sizeof(vsd::lig_meta), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (meta[0].status != VS_LIG_OK && meta[0].status != VS_LIG_NO_HEAVY)
    return fail(VS_ERR_INVALID_ARGUMENT, "ligand rejected by the device checks");
  if (meta[0].n_heavy == 0 && n_poses > 1) return fail(VS_ERR_INVALID_ARGUMENT, "no heavy atoms");
  int *dev_out = ctx->aux2.as<int>();
  CUDA_TRY(vsd::launch_cluster(st.b, n_poses, ctx->aux0.as<double>(), ctx->aux1.as<double>(), threshold, top, dev_out,
                               dev_out + n_poses, ctx->stream));
  std::vector<int> out(static_cast<size_t>(n_poses) + 1);
  CUDA_TRY(cudaMemcpyAsync(out.data(), dev_out, sizeof(int) * (n_poses + 1), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *count_out = out[static_cast<size_t>(n_poses)];
  for (int i = 0; i < *count_out; ++i) order_out[i] = out[static_cast<size_t>(i)];
  return VS_OK;
}

vs_status vs_local_search_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                                const vs_scoring_config *cfg, vs_pose *poses, double *angles, double *conformation,
                                uint64_t *evals, int32_t *status_out) {
  if (!ctx || !pocket || !batch || !cfg || !poses || !conformation)
    return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  vsd::search_cfg sc{};
  vs_status rc;
  if ((rc = upload_tables(ctx, *cfg, 1, sc))) return rc;
  Staged st;
  if ((rc = stage(ctx, batch, 0, batch->n_ligands, st))) return rc;
  std::vector<double> pin(static_cast<size_t>(8) * std::max(st.n, 1));
  for (int i = 0; i < st.n; ++i) {
    for (int q = 0; q < 4; ++q) pin[8 * i + q] = poses[i].rotation[q];
    for (int q = 0; q < 3; ++q) pin[8 * i + 4 + q] = poses[i].translation[q];
    pin[8 * i + 7] = poses[i].geo_score;
  }
  if ((rc = h2d(ctx->aux0, pin.data(), pin.size(), ctx->stream))) return rc;
  if ((rc = h2d(ctx->aux1, angles ? angles : pin.data(), angles ? static_cast<size_t>(st.torsions) : 1, ctx->stream)))
    return rc;
  if ((rc = h2d(ctx->aux2, conformation, 3 * static_cast<size_t>(st.atoms), ctx->stream))) return rc;
  vsd::item_out o{};
  if ((rc = ensure_items(ctx, st, 1, o))) return rc;
  CUDA_TRY(cudaMemsetAsync(ctx->work.p, 0, sizeof(int), ctx->stream));
  CUDA_TRY(vsd::launch_setup(st.b, 1, ctx->stream));
  CUDA_TRY(ctx->search_args.ensure(vsd::search_scratch_bytes(std::max(st.Nmax, 1), std::max(st.nmax, 1), std::max(st.mmax, 1), ctx->num_sms)));
  CUDA_TRY(vsd::launch_local_search(st.b, pocket->dev(), sc, ctx->aux0.as<double>(), ctx->aux1.as<double>(),
                                    ctx->aux2.as<double>(), o, ctx->work.as<int>(), st.Nmax, st.nmax, st.mmax,
                                    ctx->num_sms, ctx->stream, ctx->search_args.p));
  std::vector<double> T(static_cast<size_t>(7) * std::max(st.n, 1)), geo(static_cast<size_t>(std::max(st.n, 1)));
  std::vector<unsigned long long> ev(static_cast<size_t>(std::max(st.n, 1)));
  std::vector<int> stat(static_cast<size_t>(std::max(st.n, 1)));
  if (st.n) {
    CUDA_TRY(cudaMemcpyAsync(T.data(), o.T, sizeof(double) * 7 * st.n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(geo.data(), o.geo, sizeof(double) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ev.data(), o.evals, sizeof(unsigned long long) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(stat.data(), o.status, sizeof(int) * st.n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (angles && st.torsions)
    CUDA_TRY(cudaMemcpyAsync(angles, o.ang, sizeof(double) * st.torsions, cudaMemcpyDeviceToHost, ctx->stream));
  if (st.atoms)
    CUDA_TRY(cudaMemcpyAsync(conformation, o.conf, sizeof(double) * 3 * st.atoms, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < st.n; ++i) {
    if (stat[static_cast<size_t>(i)] == VS_LIG_OK) {
      for (int q = 0; q < 4; ++q) poses[i].rotation[q] = T[7 * i + q];
      for (int q = 0; q < 3; ++q) poses[i].translation[q] = T[7 * i + 4 + q];
      poses[i].geo_score = geo[static_cast<size_t>(i)];
    }
    if (evals) evals[i] = ev[static_cast<size_t>(i)];
    if (status_out) status_out[i] = stat[static_cast<size_t>(i)];
  }
  return VS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ codec
namespace {

const char *record_error(int st) {
  switch (st) {
    case VS_REC_BAD_MARKER: return "bad sync marker";
    case VS_REC_TRUNCATED: return "truncated record";
    case VS_REC_LENGTH_MISMATCH: return "record length mismatch";
    case VS_REC_BAD_ELEMENT: return "invalid element code";
    case VS_REC_NONFINITE: return "non-finite coordinate";
    case VS_REC_BAD_BOND: return "invalid bond";
    case VS_REC_BAD_BOND_ORDER: return "invalid bond order";
    case VS_REC_BAD_TORSION_INDEX: return "invalid torsion bond index";
    case VS_REC_NOT_BRIDGE: return "invalid torsion: torsion bond is not a bridge";
    case VS_REC_DISCONNECTED: return "record graph is disconnected";
    case VS_REC_TOO_LARGE: return "record too large for the GPU decoder (> 4096 atoms)";
    default: return "";
  }
}

uint32_t rd16h(const uint8_t *p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8); }

// Host side of the record decode: per record, the framing checks of
// decode_record (marker, truncation, payload length) and the counts.
void frame_host(const uint8_t *bytes, int64_t size, const int64_t *offsets, size_t N, std::vector<int32_t> &st,
                std::vector<int32_t> &na, std::vector<int32_t> &nb, std::vector<int32_t> &nt,
                std::vector<std::string> *names) {
  st.assign(N, VS_REC_OK);
  na.assign(N, 0);
  nb.assign(N, 0);
  nt.assign(N, 0);
  if (names) names->assign(N, std::string());
  for (size_t r = 0; r < N; ++r) {
    const int64_t at = offsets[r];
    if (at < 0 || at + 2 > size || bytes[at] != 0xD0 || bytes[at + 1] != 0xC5) {
      st[r] = VS_REC_BAD_MARKER;
      continue;
    }
    if (at + 6 > size) {
      st[r] = VS_REC_TRUNCATED;
      continue;
    }
    const uint64_t len = rd16h(bytes + at + 2) | (static_cast<uint64_t>(rd16h(bytes + at + 4)) << 16);
    const int64_t end = at + 6 + static_cast<int64_t>(len);
    if (end > size || at + 8 > size) {
      st[r] = VS_REC_TRUNCATED;
      continue;
    }
    const uint32_t name_len = rd16h(bytes + at + 6);
    if (at + 8 + static_cast<int64_t>(name_len) + 6 > size) {
      st[r] = VS_REC_TRUNCATED;
      continue;
    }
    const uint8_t *q = bytes + at + 8 + name_len;
    const uint32_t a = rd16h(q), b = rd16h(q + 2), t = rd16h(q + 4);
    const uint64_t payload = 2ull + name_len + 6 + 14ull * a + 5ull * b + 2ull * t;
    if (payload != len) {
      st[r] = VS_REC_LENGTH_MISMATCH;
      continue;
    }
    if (names) (*names)[r].assign(reinterpret_cast<const char *>(bytes + at + 8), name_len);
    na[r] = static_cast<int32_t>(a);
    nb[r] = static_cast<int32_t>(b);
    nt[r] = static_cast<int32_t>(t);
  }
}

}  // namespace

// decode_record (binary_codec.cpp:165-222) of n records on the GPU: the host
// reads only the framing (marker, length, name, counts) to size the outputs;
// payloads, validation and torsion partitions run in k_decode (codec.cu).
extern "C" vs_status vs_decode_records(vs_context *ctx, const uint8_t *bytes, int64_t size, const int64_t *offsets,
                                       int32_t n, vs_ligand_set **out) {
  if (!ctx || !out || n < 0 || (n > 0 && (!bytes || !offsets))) return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  CtxLock lock(ctx);
  auto *set = new vs_ligand_set;
  const size_t N = static_cast<size_t>(n);
  std::vector<int32_t> st, na, nb, nt;
  frame_host(bytes, size, offsets, N, st, na, nb, nt, &set->names);
  std::vector<int32_t> aoff(N + 1, 0), boff(N + 1, 0), toff(N + 1, 0);
  for (size_t r = 0; r < N; ++r) {
    aoff[r + 1] = aoff[r] + na[r];
    boff[r + 1] = boff[r] + nb[r];
    toff[r + 1] = toff[r] + nt[r];
  }
  std::vector<int64_t> rsoff(static_cast<size_t>(toff[N]) + 1, 0);
  for (size_t r = 0; r < N; ++r)
    for (int k = 0; k < nt[r]; ++k) rsoff[toff[r] + k + 1] = rsoff[toff[r] + k] + na[r];
  const size_t atoms = aoff[N], bonds = boff[N], tors = toff[N], slots = rsoff.back();
  vs_status rc;
  cudaStream_t s = ctx->stream;
  if ((rc = h2d(ctx->dec_bytes, bytes, static_cast<size_t>(std::max<int64_t>(size, 0)), s))) return rc;
  if ((rc = h2d(ctx->dec_offs, offsets, N, s))) return rc;
  if ((rc = h2d(ctx->dec_aoff, aoff.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->dec_boff, boff.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->dec_toff, toff.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->dec_rsoff, rsoff.data(), rsoff.size(), s))) return rc;
  if ((rc = h2d(ctx->dec_status, st.data(), N, s))) return rc;
  CUDA_TRY(ctx->dec_xyz.ensure(sizeof(double) * 3 * std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->dec_elem.ensure(std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->dec_heavy.ensure(std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->dec_order.ensure(std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->dec_ba.ensure(sizeof(uint16_t) * std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->dec_bb.ensure(sizeof(uint16_t) * std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->dec_tbond.ensure(sizeof(uint16_t) * std::max<size_t>(tors, 1)));
  CUDA_TRY(ctx->dec_rslots.ensure(sizeof(uint16_t) * std::max<size_t>(slots, 1)));
  CUDA_TRY(ctx->dec_rcount.ensure(sizeof(int) * std::max<size_t>(tors, 1)));
  CUDA_TRY(vsd::launch_decode(ctx->dec_bytes.as<uint8_t>(), ctx->dec_offs.as<int64_t>(), n, ctx->dec_aoff.as<int>(),
                              ctx->dec_boff.as<int>(), ctx->dec_toff.as<int>(), ctx->dec_rsoff.as<int64_t>(),
                              ctx->dec_xyz.as<double>(), ctx->dec_elem.as<uint8_t>(), ctx->dec_heavy.as<uint8_t>(),
                              ctx->dec_order.as<uint8_t>(), ctx->dec_ba.as<uint16_t>(), ctx->dec_bb.as<uint16_t>(),
                              ctx->dec_tbond.as<uint16_t>(), ctx->dec_rslots.as<uint16_t>(), ctx->dec_rcount.as<int>(),
                              ctx->dec_status.as<int>(), s));
  std::vector<double> xyz(3 * atoms);
  std::vector<uint8_t> elem(atoms), heavy(atoms), order(bonds);
  std::vector<uint16_t> ba(bonds), bb(bonds), tb(tors), rsl(slots);
  std::vector<int> rcount(tors);
  auto d2h = [&](void *dst, const DevBuf &src, size_t bytes_) -> cudaError_t {
    return bytes_ ? cudaMemcpyAsync(dst, src.p, bytes_, cudaMemcpyDeviceToHost, s) : cudaSuccess;
  };
  CUDA_TRY(d2h(xyz.data(), ctx->dec_xyz, sizeof(double) * 3 * atoms));
  CUDA_TRY(d2h(elem.data(), ctx->dec_elem, atoms));
  CUDA_TRY(d2h(heavy.data(), ctx->dec_heavy, atoms));
  CUDA_TRY(d2h(order.data(), ctx->dec_order, bonds));
  CUDA_TRY(d2h(ba.data(), ctx->dec_ba, sizeof(uint16_t) * bonds));
  CUDA_TRY(d2h(bb.data(), ctx->dec_bb, sizeof(uint16_t) * bonds));
  CUDA_TRY(d2h(tb.data(), ctx->dec_tbond, sizeof(uint16_t) * tors));
  CUDA_TRY(d2h(rsl.data(), ctx->dec_rslots, sizeof(uint16_t) * slots));
  CUDA_TRY(d2h(rcount.data(), ctx->dec_rcount, sizeof(int) * tors));
  CUDA_TRY(d2h(st.data(), ctx->dec_status, sizeof(int32_t) * N));
  CUDA_TRY(cudaStreamSynchronize(s));
  // the set: failed records become empty entries with the reference's message
  bool all_ok = true;
  for (size_t r = 0; r < N && all_ok; ++r) all_ok = st[r] == VS_REC_OK;
  if (all_ok) {  // the device arrays already are the set's layout
    set->status.assign(N, 0);
    set->errors.assign(N, std::string());
    set->atom_off = std::move(aoff);
    set->bond_off = std::move(boff);
    set->tors_off = std::move(toff);
    set->xyz = std::move(xyz);
    set->elem = std::move(elem);
    set->heavy = std::move(heavy);
    set->border = std::move(order);
    set->ba = std::move(ba);
    set->bb = std::move(bb);
    set->tbond = std::move(tb);
    set->right_off.assign(tors + 1, 0);
    for (size_t k = 0; k < tors; ++k) set->right_off[k + 1] = set->right_off[k] + rcount[k];
    set->ratoms.resize(static_cast<size_t>(set->right_off[tors]));
    for (size_t k = 0; k < tors; ++k)
      std::memcpy(set->ratoms.data() + set->right_off[k], rsl.data() + rsoff[k], sizeof(uint16_t) * rcount[k]);
    *out = set;
    return VS_OK;
  }
  set->status.assign(N, 0);
  set->errors.assign(N, std::string());
  set->atom_off.push_back(0);
  set->bond_off.push_back(0);
  set->tors_off.push_back(0);
  set->right_off.push_back(0);
  for (size_t r = 0; r < N; ++r) {
    set->status[r] = st[r];
    if (st[r] == VS_REC_OK) {
      for (int a = aoff[r]; a < aoff[r + 1]; ++a) {
        for (int c = 0; c < 3; ++c) set->xyz.push_back(xyz[3 * static_cast<size_t>(a) + c]);
        set->elem.push_back(elem[a]);
        set->heavy.push_back(heavy[a]);
      }
      for (int k = boff[r]; k < boff[r + 1]; ++k) {
        set->ba.push_back(ba[k]);
        set->bb.push_back(bb[k]);
        set->border.push_back(order[k]);
      }
      for (int k = toff[r]; k < toff[r + 1]; ++k) {
        set->tbond.push_back(tb[k]);
        set->ratoms.insert(set->ratoms.end(), rsl.begin() + rsoff[k], rsl.begin() + rsoff[k] + rcount[k]);
        set->right_off.push_back(static_cast<int32_t>(set->ratoms.size()));
      }
    } else {
      set->errors[r] = record_error(st[r]);
    }
    set->atom_off.push_back(static_cast<int32_t>(set->elem.size()));
    set->bond_off.push_back(static_cast<int32_t>(set->ba.size()));
    set->tors_off.push_back(static_cast<int32_t>(set->tbond.size()));
  }
  *out = set;
  return VS_OK;
}

// The pipeline's decode -> dock without a host round trip of the decoded
// batch: records are framed on the host, decoded by k_decode straight into
// the dock path's device input arrays, and docked against every pocket.
extern "C" vs_status vs_dock_records(vs_context *ctx, const vs_pocket *const *pockets, int32_t n_pockets,
                                     const uint8_t *bytes, int64_t size, const int64_t *offsets, int32_t n,
                                     const vs_scoring_config *cfg, vs_dock_result *results, int32_t *record_status) {
  if (!ctx || !pockets || n_pockets < 1 || n < 0 || !results || (n > 0 && (!bytes || !offsets)))
    return fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  vs_status rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_pockets(ctx, pockets, n_pockets))) return rc;
  CtxLock lock(ctx);
  const size_t N = static_cast<size_t>(n);
  std::vector<int32_t> st, na, nb, nt;
  frame_host(bytes, size, offsets, N, st, na, nb, nt, nullptr);
  Staged sg;
  sg.n = n;
  sg.atom_off.assign(N + 1, 0);
  sg.bond_off.assign(N + 1, 0);
  sg.tors_off.assign(N + 1, 0);
  for (size_t r = 0; r < N; ++r) {
    sg.atom_off[r + 1] = sg.atom_off[r] + na[r];
    sg.bond_off[r + 1] = sg.bond_off[r] + nb[r];
    sg.tors_off[r + 1] = sg.tors_off[r] + nt[r];
  }
  sg.atoms = sg.atom_off[N];
  sg.torsions = sg.tors_off[N];
  const size_t atoms = sg.atoms, bonds = sg.bond_off[N], tors = sg.torsions;
  std::vector<int64_t> rsoff(tors + 1, 0);
  for (size_t r = 0; r < N; ++r)
    for (int q = 0; q < nt[r]; ++q) rsoff[sg.tors_off[r] + q + 1] = rsoff[sg.tors_off[r] + q] + na[r];
  cudaStream_t s = ctx->stream;
  if ((rc = h2d(ctx->dec_bytes, bytes, static_cast<size_t>(std::max<int64_t>(size, 0)), s))) return rc;
  if ((rc = h2d(ctx->dec_offs, offsets, N, s))) return rc;
  if ((rc = h2d(ctx->atom_off, sg.atom_off.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->bond_off, sg.bond_off.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->tors_off, sg.tors_off.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->dec_rsoff, rsoff.data(), rsoff.size(), s))) return rc;
  if ((rc = h2d(ctx->dec_status, st.data(), N, s))) return rc;
  CUDA_TRY(ctx->xyz.ensure(sizeof(double) * 3 * std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->elem.ensure(std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->heavy.ensure(std::max<size_t>(atoms, 1)));
  CUDA_TRY(ctx->dec_order.ensure(std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->bond_a.ensure(sizeof(uint16_t) * std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->bond_b.ensure(sizeof(uint16_t) * std::max<size_t>(bonds, 1)));
  CUDA_TRY(ctx->tors_bond.ensure(sizeof(uint16_t) * std::max<size_t>(tors, 1)));
  CUDA_TRY(ctx->dec_rslots.ensure(sizeof(uint16_t) * std::max<int64_t>(rsoff.back(), 1)));
  CUDA_TRY(ctx->dec_rcount.ensure(sizeof(int) * std::max<size_t>(tors, 1)));
  CUDA_TRY(ctx->aux3.ensure(sizeof(int) * std::max<size_t>(N, 1)));  // heavy atoms per record
  CUDA_TRY(vsd::launch_decode(ctx->dec_bytes.as<uint8_t>(), ctx->dec_offs.as<int64_t>(), n, ctx->atom_off.as<int>(),
                              ctx->bond_off.as<int>(), ctx->tors_off.as<int>(), ctx->dec_rsoff.as<int64_t>(),
                              ctx->xyz.as<double>(), ctx->elem.as<uint8_t>(), ctx->heavy.as<uint8_t>(),
                              ctx->dec_order.as<uint8_t>(), ctx->bond_a.as<uint16_t>(), ctx->bond_b.as<uint16_t>(),
                              ctx->tors_bond.as<uint16_t>(), ctx->dec_rslots.as<uint16_t>(), ctx->dec_rcount.as<int>(),
                              ctx->dec_status.as<int>(), s, ctx->aux3.as<int>()));
  std::vector<int> rcount(tors), nh(N);
  if (tors) CUDA_TRY(cudaMemcpyAsync(rcount.data(), ctx->dec_rcount.p, sizeof(int) * tors, cudaMemcpyDeviceToHost, s));
  if (N) {
    CUDA_TRY(cudaMemcpyAsync(nh.data(), ctx->aux3.p, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(st.data(), ctx->dec_status.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  // the staging metadata of stage(), from the counts; failed records are
  // rejected by k_setup (pre_status) and own no right sets
  sg.ditem_base.assign(N + 1, 0);
  sg.right_off.assign(tors + 1, 0);
  sg.lN.assign(N, 0);
  sg.ln.assign(N, 0);
  sg.lm.assign(N, 0);
  sg.Nmax = sg.nmax = sg.mmax = 0;
  int dbase = 0;
  for (size_t r = 0; r < N; ++r) {
    sg.ditem_base[r] = dbase;
    const int Na = na[r], m = nt[r], h = st[r] == VS_REC_OK ? nh[r] : 0;
    sg.lN[r] = Na;
    sg.ln[r] = h;
    sg.lm[r] = m;
    if (st[r] == VS_REC_OK && Na <= VS_MAX_ATOMS && m <= VS_MAX_TORSIONS && h <= VS_MAX_HEAVY) {
      sg.Nmax = std::max(sg.Nmax, Na);
      sg.mmax = std::max(sg.mmax, m);
      sg.nmax = std::max(sg.nmax, h);
    }
    dbase += std::min(m, VS_MAX_TORSIONS) * std::min(Na, VS_MAX_ATOMS);
    for (int q = 0; q < m; ++q) {
      const size_t t = static_cast<size_t>(sg.tors_off[r]) + q;
      sg.right_off[t + 1] = sg.right_off[t] + (st[r] == VS_REC_OK ? rcount[t] : 0);
      if (st[r] != VS_REC_OK) rcount[t] = 0;
    }
  }
  sg.ditem_base[N] = dbase;
  if ((rc = h2d(ctx->ditem_base, sg.ditem_base.data(), N + 1, s))) return rc;
  if ((rc = h2d(ctx->right_off, sg.right_off.data(), tors + 1, s))) return rc;
  if ((rc = h2d(ctx->dec_rcount, rcount.data(), tors, s))) return rc;
  std::vector<int32_t> pre(N);
  for (size_t r = 0; r < N; ++r) pre[r] = st[r] != VS_REC_OK;
  if ((rc = h2d(ctx->aux2, pre.data(), N, s))) return rc;
  CUDA_TRY(ctx->right_atoms.ensure(sizeof(uint16_t) * std::max<int>(sg.right_off[tors], 1)));
  CUDA_TRY(vsd::launch_compact_right(ctx->dec_rslots.as<uint16_t>(), ctx->dec_rsoff.as<int64_t>(),
                                     ctx->dec_rcount.as<int>(), ctx->right_off.as<int>(), static_cast<int>(tors),
                                     ctx->right_atoms.as<uint16_t>(), s));
  const size_t ta = std::max<size_t>(atoms, 1), tt = std::max<size_t>(tors, 1);
  CUDA_TRY(ctx->meta.ensure(sizeof(vsd::lig_meta) * std::max<size_t>(N, 1)));
  CUDA_TRY(ctx->tmask.ensure(4 * ta));
  CUDA_TRY(ctx->heavy_list.ensure(2 * ta));
  CUDA_TRY(ctx->dmask.ensure(4 * ta));
  CUDA_TRY(ctx->tors_a.ensure(2 * tt));
  CUDA_TRY(ctx->tors_b.ensure(2 * tt));
  CUDA_TRY(ctx->d_count.ensure(4 * tt));
  CUDA_TRY(ctx->d_off.ensure(4 * tt));
  CUDA_TRY(ctx->ditems.ensure(2 * static_cast<size_t>(std::max(dbase, 1))));
  CUDA_TRY(ctx->titems.ensure(8 * static_cast<size_t>(std::max(dbase, 1))));
  vsd::batch_dev &b = sg.b;
  b.n_lig = n;
  b.pre_status = ctx->aux2.as<int>();
  b.atom_off = ctx->atom_off.as<int>();
  b.bond_off = ctx->bond_off.as<int>();
  b.tors_off = ctx->tors_off.as<int>();
  b.ditem_base = ctx->ditem_base.as<int>();
  b.xyz = ctx->xyz.as<double>();
  b.elem = ctx->elem.as<uint8_t>();
  b.heavy = ctx->heavy.as<uint8_t>();
  b.bond_a = ctx->bond_a.as<uint16_t>();
  b.bond_b = ctx->bond_b.as<uint16_t>();
  b.tors_bond = ctx->tors_bond.as<uint16_t>();
  b.right_off = ctx->right_off.as<int>();
  b.right_atoms = ctx->right_atoms.as<uint16_t>();
  b.meta = ctx->meta.as<vsd::lig_meta>();
  b.atom_tmask = ctx->tmask.as<uint32_t>();
  b.heavy_list = ctx->heavy_list.as<uint16_t>();
  b.heavy_dmask = ctx->dmask.as<uint32_t>();
  b.tors_a = ctx->tors_a.as<uint16_t>();
  b.tors_b = ctx->tors_b.as<uint16_t>();
  b.d_count = ctx->d_count.as<int>();
  b.d_off = ctx->d_off.as<int>();
  b.ditems = ctx->ditems.as<uint16_t>();
  b.titems = ctx->titems.as<uint32_t>();
  if (record_status)
    for (size_t r = 0; r < N; ++r) record_status[r] = st[r];
  std::vector<vs_dock_result *> res(static_cast<size_t>(n_pockets));
  for (int p = 0; p < n_pockets; ++p) res[p] = results + static_cast<size_t>(p) * N;
  return dock_impl(ctx, pockets, n_pockets, nullptr, cfg, res.data(), nullptr, nullptr, nullptr, &sg);
}
