// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load liboracle.so, and only as the checker.
// ============================================================================
//
// CPU restatement of the reference's dock-and-score hot path
// (/root/reference/proj/src/dockengine/search.cpp, grid.cpp, chem.cpp,
//  src/geometry/transform.cpp, src/molmodel/ligand.cpp).  Plain C++ with
// explicit evaluation order: every floating-point expression whose rounding
// Eigen fixes is written out in the order SURVEY.md Appendix A gives (items
// 1-8 are cited where used).  Build: oracle/Makefile (g++ -O2
// -ffp-contract=off, no -march: SSE2 doubles, no FMA — the reference's
// Release flags).  Pinned against (a) the reference's own known-answer tests,
// ported in tests/test_oracle_kats.py, and (b) the reference sources compiled
// against the Eigen-subset restatement (oracle/_ref, tests/test_oracle_vs_ref.py).
//
// Trig: the reference calls glibc sin/cos (Eigen::AngleAxisd,
// transform.cpp:64).  vso_set_trig_mode(1) swaps the *torsion* sin/cos for
// the correctly rounded routine the GPU uses (include/vs_crtrig.h) so the
// GPU can be checked bit-for-bit; mode 0 (default) is the glibc-faithful
// oracle.  Fibonacci restarts and rotation spins always use glibc (the GPU
// receives those as host-computed tables).
//
// Counters: S, A_rigid, A_tors, R_build, P_flat,
// P_chem, P_rmsd, clash_pairs, oob_samples.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "vs_crtrig.h"
#include "vs_dock.h"

namespace vso {

// ------------------------------------------------------------------ errors
struct LigandError : std::runtime_error {
  int code;
  LigandError(int c, const char *m) : std::runtime_error(m), code(c) {}
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::atomic<int> g_trig_mode{0};

// ------------------------------------------------------------------ math
struct V3 {
  double x, y, z;
  double &operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 vadd(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 vsub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 vscale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 vdiv(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
// Appendix A item 6: 3-element reductions are (a0 + a1) + a2.
inline double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
inline double vnorm(V3 a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(V3 a, V3 b) {  // Appendix A item 3 (generic cross)
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

struct Quat {
  double x, y, z, w;
};
struct M3 {
  double m[3][3];
};
struct RT {
  Quat q{0, 0, 0, 1};
  V3 t{0, 0, 0};
};

// Appendix A item 1: Quaterniond(AngleAxisd(a, u)) with glibc trig.
inline Quat quat_from_angle_axis(double angle, V3 u) {
  const double ha = 0.5 * angle;
  const double c = std::cos(ha);
  const double s = std::sin(ha);
  return {s * u.x, s * u.y, s * u.z, c};
}
// Appendix A item 2.
inline M3 quat_matrix(const Quat &q) {
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  M3 r;
  r.m[0][0] = 1.0 - (tyy + tzz);
  r.m[0][1] = txy - twz;
  r.m[0][2] = txz + twy;
  r.m[1][0] = txy + twz;
  r.m[1][1] = 1.0 - (txx + tzz);
  r.m[1][2] = tyz - twx;
  r.m[2][0] = txz - twy;
  r.m[2][1] = tyz + twx;
  r.m[2][2] = 1.0 - (txx + tyy);
  return r;
}
// Appendix A item 3: q * v.
inline V3 quat_rotate(const Quat &q, V3 v) {
  const V3 qv{q.x, q.y, q.z};
  V3 uv = cross(qv, v);
  uv = vadd(uv, uv);
  return vadd(vadd(v, vscale(q.w, uv)), cross(qv, uv));
}
// Appendix A item 5.
inline Quat quat_mul(const Quat &a, const Quat &b) {
  Quat r;
  r.x = (a.w * b.x + a.y * b.z) - (a.z * b.y - a.x * b.w);
  r.y = (a.w * b.y + a.y * b.w) + (a.z * b.x - a.x * b.z);
  r.z = (a.w * b.z - a.y * b.x) + (a.z * b.w + a.x * b.y);
  r.w = (a.w * b.w - a.y * b.y) - (a.z * b.z + a.x * b.x);
  return r;
}
// Appendix A item 6.
inline Quat quat_normalized(const Quat &q) {
  const double n = std::sqrt((q.x * q.x + q.z * q.z) + (q.y * q.y + q.w * q.w));
  return {q.x / n, q.y / n, q.z / n, q.w / n};
}
// Appendix A item 4, Vector3d result.
inline V3 mat_vec(const M3 &r, V3 v) {
  return {(r.m[0][0] * v.x + r.m[0][1] * v.y) + r.m[0][2] * v.z,
          (r.m[1][0] * v.x + r.m[1][1] * v.y) + r.m[1][2] * v.z,
          r.m[2][0] * v.x + (r.m[2][1] * v.y + r.m[2][2] * v.z)};
}
// Appendix A item 4, column `col` of a 3xN product.
inline V3 mat_col(const M3 &r, V3 v, std::size_t col) {
  V3 o;
  for (int row = 0; row < 3; ++row) {
    const bool packet = (col % 2 == 0) ? (row < 2) : (row > 0);
    o[row] = packet ? (r.m[row][0] * v.x + r.m[row][1] * v.y) + r.m[row][2] * v.z
                    : r.m[row][0] * v.x + (r.m[row][1] * v.y + r.m[row][2] * v.z);
  }
  return o;
}
// Appendix A item 7 with the torsion trig selected by g_trig_mode.
inline M3 angle_axis_matrix(double angle, V3 u) {
  double s, c;
  if (g_trig_mode.load(std::memory_order_relaxed) == 1) {
    vs_crtrig::sincos_cr(angle, &s, &c);
  } else {
    s = std::sin(angle);
    c = std::cos(angle);
  }
  const V3 sa{s * u.x, s * u.y, s * u.z};
  const double omc = 1.0 - c;
  const V3 ca{omc * u.x, omc * u.y, omc * u.z};
  M3 r;
  double tmp = ca.x * u.y;
  r.m[0][1] = tmp - sa.z;
  r.m[1][0] = tmp + sa.z;
  tmp = ca.x * u.z;
  r.m[0][2] = tmp + sa.y;
  r.m[2][0] = tmp - sa.y;
  tmp = ca.y * u.z;
  r.m[1][2] = tmp - sa.x;
  r.m[2][1] = tmp + sa.x;
  r.m[0][0] = ca.x * u.x + c;
  r.m[1][1] = ca.y * u.y + c;
  r.m[2][2] = ca.z * u.z + c;
  return r;
}

// ------------------------------------------------------------------ model
struct Ligand {  // ligand.hpp:28-71
  std::vector<V3> pos;
  std::vector<uint8_t> elem, heavy;
  std::vector<uint16_t> ba, bb;
  std::vector<uint8_t> border;
  std::vector<uint16_t> tors_bond;
  std::vector<std::vector<uint16_t>> right;
  std::size_t n_atoms() const { return pos.size(); }
  std::size_t n_heavy() const {
    std::size_t n = 0;
    for (auto h : heavy) n += h ? 1 : 0;
    return n;
  }
};
using Conf = std::vector<V3>;

struct Pocket {  // pocket.hpp:28-57
  V3 origin;
  double spacing;
  int dims[3];
  const double *values;
  int n_protein;
  const uint8_t *pelem;
  const double *pxyz;
  double at(int ix, int iy, int iz) const {
    return values[static_cast<std::size_t>(ix) +
                  static_cast<std::size_t>(dims[0]) *
                      (static_cast<std::size_t>(iy) +
                       static_cast<std::size_t>(dims[1]) * static_cast<std::size_t>(iz))];
  }
  V3 box_center() const {  // pocket.hpp:53-56
    const double hs = 0.5 * spacing;
    return {origin.x + hs * static_cast<double>(dims[0] - 1),
            origin.y + hs * static_cast<double>(dims[1] - 1),
            origin.z + hs * static_cast<double>(dims[2] - 1)};
  }
};

struct Counters {
  uint64_t S = 0, A_rigid = 0, A_tors = 0, R_build = 0, P_flat = 0, P_chem = 0, P_rmsd = 0;
  int64_t clash_pairs = 0, oob_samples = 0;
};

struct Pose {  // pose.hpp:23-29
  RT T;
  std::vector<double> ang;
  Conf conf;
  double geo = 0.0;
  double chem = 0.0;
};

// ------------------------------------------------------------ geometry
// transform.cpp:30-32: (R * conf).colwise() + t, R from toRotationMatrix.
Conf apply_rigid(const Conf &c, const RT &T) {
  const M3 r = quat_matrix(T.q);
  Conf o(c.size());
  for (std::size_t i = 0; i < c.size(); ++i) {
    const V3 p = mat_col(r, c[i], i);
    o[i] = {p.x + T.t.x, p.y + T.t.y, p.z + T.t.z};
  }
  return o;
}
// transform.cpp:49-52 with Appendix A item 8 (rowwise().mean()).
V3 centroid(const Conf &c) {
  if (c.empty()) throw LigandError(VS_LIG_EMPTY, "empty conformation");
  const std::ptrdiff_t n = static_cast<std::ptrdiff_t>(c.size());
  V3 s{};
  for (int r = 0; r < 2; ++r) {
    double p = c[0][r];
    const std::ptrdiff_t size4 = (n - 1) & ~std::ptrdiff_t(3);
    std::ptrdiff_t i = 1;
    for (; i < size4; i += 4) p = p + ((c[i][r] + c[i + 1][r]) + (c[i + 2][r] + c[i + 3][r]));
    for (; i < n; ++i) p = p + c[i][r];
    s[r] = p;
  }
  double z = c[0].z;
  for (std::ptrdiff_t i = 1; i < n; ++i) z = z + c[i].z;
  s.z = z;
  const double dn = static_cast<double>(n);
  return {s.x / dn, s.y / dn, s.z / dn};
}
// transform.cpp:54-71.
Conf apply_torsion(const Conf &c, const Ligand &lig, std::size_t t, double angle, Counters *k) {
  if (lig.tors_bond[t] >= lig.ba.size())
    throw LigandError(VS_LIG_BAD_TORSION, "torsion bond index out of range");
  const uint16_t a = lig.ba[lig.tors_bond[t]], b = lig.bb[lig.tors_bond[t]];
  if (a >= c.size() || b >= c.size())
    throw LigandError(VS_LIG_BAD_TORSION, "torsion atom index out of range");
  const V3 pivot = c[a];
  const V3 axis = vsub(c[b], pivot);
  const double norm = vnorm(axis);
  if (norm < 1e-9) throw LigandError(VS_LIG_DEGENERATE_AXIS, "degenerate torsion axis");
  const M3 rot = angle_axis_matrix(angle, vdiv(axis, norm));
  Conf o = c;
  for (uint16_t idx : lig.right[t]) {
    if (idx >= c.size()) throw LigandError(VS_LIG_BAD_TORSION, "torsion atom index out of range");
    o[idx] = vadd(mat_vec(rot, vsub(c[idx], pivot)), pivot);
  }
  if (k) {
    k->R_build += 1;
  }
  return o;
}
// transform.cpp:73-81.
Conf apply_torsions(const Conf &base, const Ligand &lig, const std::vector<double> &ang,
                    Counters *k) {
  if (ang.size() != lig.tors_bond.size())
    throw LigandError(VS_LIG_BAD_TORSION, "torsion angle count does not match ligand");
  Conf c = base;
  for (std::size_t i = 0; i < ang.size(); ++i) c = apply_torsion(c, lig, i, ang[i], k);
  return c;
}
// transform.cpp:83-90.
double internal_distance_sum(const Conf &c) {
  double sum = 0.0;
  for (std::size_t i = 0; i < c.size(); ++i)
    for (std::size_t j = i + 1; j < c.size(); ++j) sum += vnorm(vsub(c[i], c[j]));
  return sum;
}
// transform.cpp:99-113.
double heavy_atom_rmsd(const Conf &a, const Conf &b, const Ligand &lig, Counters *k) {
  double sum = 0.0;
  std::size_t heavy = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    if (!lig.heavy[i]) continue;
    sum += sqnorm(vsub(a[i], b[i]));
    ++heavy;
  }
  if (heavy == 0) throw LigandError(VS_LIG_NO_HEAVY, "no heavy atoms");
  if (k) k->P_rmsd += heavy;
  return std::sqrt(sum / static_cast<double>(heavy));
}

// ------------------------------------------------------------ grid
// grid.cpp:59-91.
double field_value(const Pocket &p, V3 pt, bool *outside = nullptr) {
  const V3 local{(pt.x - p.origin.x) / p.spacing, (pt.y - p.origin.y) / p.spacing,
                 (pt.z - p.origin.z) / p.spacing};
  const double mx = static_cast<double>(p.dims[0] - 1);
  const double my = static_cast<double>(p.dims[1] - 1);
  const double mz = static_cast<double>(p.dims[2] - 1);
  if (local.x < 0.0 || local.y < 0.0 || local.z < 0.0 || local.x > mx || local.y > my ||
      local.z > mz) {
    if (outside) *outside = true;
    return -10.0;  // kClashValue, grid.hpp:23
  }
  if (outside) *outside = false;
  int ix = std::min(static_cast<int>(local.x), p.dims[0] - 2);
  int iy = std::min(static_cast<int>(local.y), p.dims[1] - 2);
  int iz = std::min(static_cast<int>(local.z), p.dims[2] - 2);
  ix = std::max(ix, 0);
  iy = std::max(iy, 0);
  iz = std::max(iz, 0);
  const double fx = local.x - ix, fy = local.y - iy, fz = local.z - iz;
  double acc = 0.0;
  for (int cz = 0; cz < 2; ++cz)
    for (int cy = 0; cy < 2; ++cy)
      for (int cx = 0; cx < 2; ++cx) {
        const double w = ((cx ? fx : 1.0 - fx) * (cy ? fy : 1.0 - fy)) * (cz ? fz : 1.0 - fz);
        acc += w * p.at(ix + cx, iy + cy, iz + cz);
      }
  return acc;
}
// grid.cpp:93-104.
double geo_score(const Pocket &p, const Ligand &lig, const Conf &c, Counters *k) {
  double total = 0.0;
  uint64_t heavy = 0;
  for (std::size_t i = 0; i < lig.n_atoms(); ++i) {
    if (!lig.heavy[i]) continue;
    total += field_value(p, c[i]);
    ++heavy;
  }
  if (k) k->S += heavy;
  return total;
}

// ------------------------------------------------------------ chem
// chem.cpp:12-46.
inline int chem_class(uint8_t e) {  // elements.hpp:32-42: 0 hydrophobic, 1 polar, 2 other
  if (e == VS_ELEM_C) return 0;
  if (e == VS_ELEM_N || e == VS_ELEM_O) return 1;
  return 2;
}
inline double pair_weight(int a, int b) {  // chem.cpp:24-29
  if (a == 2 || b == 2) return 0.05;
  if (a == 0 && b == 0) return 0.4;
  if (a == 1 && b == 1) return 1.0;
  return 0.1;
}
double chem_score(const Pocket &p, const Ligand &lig, const Conf &c, Counters *k,
                  int64_t *clash_pairs) {
  double total = 0.0;
  for (std::size_t i = 0; i < lig.n_atoms(); ++i) {
    if (!lig.heavy[i]) continue;
    const int ci = chem_class(lig.elem[i]);
    const V3 x = c[i];
    for (int j = 0; j < p.n_protein; ++j) {
      const V3 pp{p.pxyz[3 * j], p.pxyz[3 * j + 1], p.pxyz[3 * j + 2]};
      const double d = vnorm(vsub(x, pp));
      if (d >= 4.5) continue;
      const double ramp = d <= 3.5 ? 1.0 : (4.5 - d) / (4.5 - 3.5);
      total += pair_weight(ci, chem_class(p.pelem[j])) * ramp;
      if (d < 2.0) {
        total -= 5.0;
        if (clash_pairs) ++*clash_pairs;
      }
      if (k) k->P_chem += 1;
    }
  }
  return total;
}

// ------------------------------------------------------------ search
constexpr double kPi = 3.14159265358979323846;
constexpr double kGoldenRatio = 1.6180339887498948482;

// search.cpp:27-69.
std::pair<Conf, std::vector<double>> flatten(const Ligand &lig, const Conf &base, int max_sweeps,
                                             Counters *k) {
  const std::size_t m = lig.tors_bond.size();
  if (m == 0) return {base, {}};
  constexpr int kSteps = 36;
  constexpr double kStep = 2.0 * kPi / kSteps;
  std::vector<int> index(m, 0);
  auto angles_of = [&](const std::vector<int> &idx) {
    std::vector<double> a(m);
    for (std::size_t i = 0; i < m; ++i) a[i] = idx[i] * kStep;
    return a;
  };
  std::size_t right_total = 0;
  for (auto &r : lig.right) right_total += r.size();
  const uint64_t pairs = lig.n_atoms() * (lig.n_atoms() - 1) / 2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    bool changed = false;
    for (std::size_t t = 0; t < m; ++t) {
      std::vector<int> cand = index;
      int best_off = 0;
      double best = -std::numeric_limits<double>::infinity();
      for (int off = 0; off < kSteps; ++off) {
        cand[t] = (index[t] + off) % kSteps;
        const double spread = internal_distance_sum(apply_torsions(base, lig, angles_of(cand), k));
        if (k) {
          k->P_flat += pairs;
          k->A_tors += right_total;
        }
        if (spread > best) {
          best = spread;
          best_off = off;
        }
      }
      if (best_off != 0) {
        index[t] = (index[t] + best_off) % kSteps;
        changed = true;
      }
    }
    if (!changed) break;
  }
  const std::vector<double> a = angles_of(index);
  return {apply_torsions(base, lig, a, k), a};
}

// search.cpp:71-82.
V3 fibonacci_axis(int i, int k) {
  constexpr double kGoldenAngle = 2.0 * kPi * (2.0 - kGoldenRatio);
  const double z = 1.0 - 2.0 * (i + 0.5) / static_cast<double>(k);
  const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
  const double az = std::fmod(i * kGoldenAngle, 2.0 * kPi);
  return {r * std::cos(az), r * std::sin(az), z};
}
double fibonacci_rotation_angle(int i) { return 2.0 * kPi * std::fmod(i * kGoldenRatio, 1.0); }

// search.cpp:84-107.
std::vector<Pose> initial_poses(const Pocket &p, const Ligand &lig, const Conf &base,
                                const std::vector<double> &flat_ang, int k, Counters *cn) {
  if (k < 1) throw ConfigError("restart count must be at least 1");
  const Conf flat = apply_torsions(base, lig, flat_ang, cn);
  const V3 fc = centroid(flat);
  const V3 center = p.box_center();
  std::vector<Pose> poses;
  poses.reserve(static_cast<std::size_t>(k));
  for (int i = 0; i < k; ++i) {
    Pose pose;
    pose.T.q = quat_from_angle_axis(fibonacci_rotation_angle(i), fibonacci_axis(i, k));
    pose.T.t = vsub(center, quat_rotate(pose.T.q, fc));
    pose.ang = flat_ang;
    pose.conf = apply_rigid(flat, pose.T);
    if (cn) cn->A_rigid += lig.n_atoms();
    pose.geo = geo_score(p, lig, pose.conf, cn);
    poses.push_back(std::move(pose));
  }
  return poses;
}

// transform.cpp:16-21.
RT compose(const RT &b, const RT &a) {
  RT o;
  o.q = quat_normalized(quat_mul(b.q, a.q));
  o.t = vadd(quat_rotate(b.q, a.t), b.t);
  return o;
}

#ifdef VSO_TRACE
// Development analysis only: per neighbour the score, the current score and,
// over its moved heavy-atom samples, the sum of the cells' L1 gradient bounds
// (local units), their count and the smallest distance to a node-box face.
FILE *g_trace = nullptr;
void trace_neighbour(const Pocket &p, const Ligand &lig, const Conf &c, const Conf &cur, double score, double cs) {
  if (!g_trace) return;
  double gsum = 0.0, gmax = 0.0, minface = 1e9;
  int nm = 0;
  for (std::size_t i = 0; i < lig.n_atoms(); ++i) {
    if (!lig.heavy[i]) continue;
    if (std::memcmp(&c[i], &cur[i], sizeof(V3)) == 0) continue;
    ++nm;
    double l[3];
    int ix[3];
    for (int a = 0; a < 3; ++a) {
      l[a] = (c[i][a] - p.origin[a]) / p.spacing;
      minface = std::min(minface, std::min(std::fabs(l[a]), std::fabs(l[a] - (p.dims[a] - 1))));
      ix[a] = std::max(0, std::min((int)std::floor(l[a]), p.dims[a] - 2));
    }
    bool out = false;
    for (int a = 0; a < 3; ++a) out |= l[a] < 0 || l[a] > p.dims[a] - 1;
    if (out) continue;
    double v[8];
    for (int q = 0; q < 8; ++q) v[q] = p.at(ix[0] + (q & 1), ix[1] + ((q >> 1) & 1), ix[2] + (q >> 2));
    double g = 0.0;
    for (int a = 0; a < 3; ++a) {
      double mx = 0.0;
      for (int q = 0; q < 8; ++q)
        if (!((q >> a) & 1)) mx = std::max(mx, std::fabs(v[q | (1 << a)] - v[q]));
      g += mx;
    }
    gsum += g;
    gmax += g > 0 ? 1.0 : 0.0;  // non-uniform moved samples
  }
  const double rec[6] = {score, cs, gsum, (double)nm, minface, gmax};
  std::fwrite(rec, sizeof rec, 1, g_trace);
}
#endif

// search.cpp:109-193.
Pose local_search(const Pocket &p, const Ligand &lig, Pose pose, const vs_scoring_config &cfg,
                  Counters *cn) {
  const Conf base = lig.pos;
  const std::size_t m = pose.ang.size();
  const std::size_t nh = lig.n_heavy();
  Conf torsioned = apply_torsions(base, lig, pose.ang, cn);
  double step_t = cfg.step_translation, step_r = cfg.step_rotation, step_q = cfg.step_torsion;
  for (int iter = 0; iter < cfg.max_iterations && step_t >= cfg.min_translation; ++iter) {
#ifdef VSO_TRACE
    if (g_trace) {
      const double rec[6] = {-1e300, (double)(12 + 2 * m), step_t, 0, 0, 0};
      std::fwrite(rec, sizeof rec, 1, g_trace);
    }
#endif
    const V3 pivot = centroid(pose.conf);
    double best_score = pose.geo;
    bool improved = false;
    RT best_T;
    std::vector<double> best_ang;
    Conf best_tors, best_conf;
    auto consider = [&](const RT &T, const std::vector<double> *ang, const Conf &frame) {
      const Conf conf = apply_rigid(frame, T);
      const double score = geo_score(p, lig, conf, cn);
#ifdef VSO_TRACE
      trace_neighbour(p, lig, conf, pose.conf, score, pose.geo);
#endif
      if (score > best_score) {
        best_score = score;
        improved = true;
        best_T = T;
        if (ang) {
          best_ang = *ang;
          best_tors = frame;
        } else {
          best_ang.clear();
        }
        best_conf = conf;
      }
    };
    for (int axis = 0; axis < 3; ++axis)
      for (const double sign : {1.0, -1.0}) {
        RT t = pose.T;
        t.t[axis] += sign * step_t;
        if (cn) cn->A_rigid += nh;
        consider(t, nullptr, torsioned);
      }
    for (int axis = 0; axis < 3; ++axis)
      for (const double sign : {1.0, -1.0}) {
        V3 unit{0.0, 0.0, 0.0};
        unit[axis] = 1.0;
        RT spin;
        spin.q = quat_from_angle_axis(sign * step_r, unit);
        spin.t = vsub(pivot, quat_rotate(spin.q, pivot));
        if (cn) cn->A_rigid += nh;
        consider(compose(spin, pose.T), nullptr, torsioned);
      }
    std::vector<double> ang = pose.ang;
    for (std::size_t t = 0; t < m; ++t) {
      for (const double sign : {1.0, -1.0}) {
        ang[t] = pose.ang[t] + sign * step_q;
        if (cn) {
          cn->A_rigid += nh;
          for (std::size_t u = 0; u < m; ++u)
            for (uint16_t idx : lig.right[u]) cn->A_tors += lig.heavy[idx] ? 1 : 0;
        }
        consider(pose.T, &ang, apply_torsions(base, lig, ang, cn));
      }
      ang[t] = pose.ang[t];
    }
    if (improved) {
      if (cn) cn->A_rigid += lig.n_atoms();  // adopted pose materialised in full
      pose.T = best_T;
      if (!best_ang.empty()) {
        pose.ang = std::move(best_ang);
        torsioned = std::move(best_tors);
      }
      pose.conf = std::move(best_conf);
      pose.geo = best_score;
    } else {
      step_t *= 0.5;
      step_r *= 0.5;
      step_q *= 0.5;
    }
  }
  return pose;
}

// search.cpp:195-236.  Returns indices into `poses` in output order.
std::vector<std::size_t> cluster_and_select(const std::vector<Pose> &poses, const Ligand &lig,
                                            double threshold, std::size_t top, Counters *cn) {
  if (poses.empty()) throw ConfigError("cannot cluster an empty pose list");
  std::vector<std::size_t> visit(poses.size());
  std::iota(visit.begin(), visit.end(), 0);
  std::stable_sort(visit.begin(), visit.end(),
                   [&](std::size_t a, std::size_t b) { return poses[a].geo > poses[b].geo; });
  std::vector<std::size_t> leaders, followers;
  for (std::size_t idx : visit) {
    bool joined = false;
    for (std::size_t l : leaders)
      if (heavy_atom_rmsd(poses[idx].conf, poses[l].conf, lig, cn) <= threshold) {
        joined = true;
        break;
      }
    (joined ? followers : leaders).push_back(idx);
  }
  std::vector<std::size_t> out;
  for (std::size_t i : leaders) {
    if (out.size() == top) break;
    out.push_back(i);
  }
  for (std::size_t i : followers) {
    if (out.size() == top) break;
    out.push_back(i);
  }
  return out;
}

struct DockOut {
  double best_score = 0;
  Pose best;
  uint64_t poses_evaluated = 0;
  std::size_t n_survivors = 0;
  Counters cn;
};

// search.cpp:238-276.
DockOut dock_and_score(const Pocket &p, const Ligand &lig, const vs_scoring_config &cfg) {
  DockOut out;
  Counters &cn = out.cn;
  const Conf base = lig.pos;
  auto flat = flatten(lig, base, cfg.flatten_max_sweeps, &cn);
  std::vector<Pose> poses = initial_poses(p, lig, base, flat.second, cfg.restarts, &cn);
  for (Pose &pose : poses) pose = local_search(p, lig, std::move(pose), cfg, &cn);
  const std::vector<std::size_t> surv = cluster_and_select(
      poses, lig, cfg.rmsd_threshold, static_cast<std::size_t>(cfg.rescored), &cn);
  std::size_t best = 0;
  double best_chem = -std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < surv.size(); ++i) {
    Pose &s = poses[surv[i]];
    s.chem = chem_score(p, lig, s.conf, &cn, nullptr);
    if (s.chem > best_chem) {
      best_chem = s.chem;
      best = i;
    }
  }
  out.best_score = best_chem;
  out.best = poses[surv[best]];
  out.poses_evaluated = poses.size();
  out.n_survivors = surv.size();
  // Integer parity diagnostics of the best pose (Appendix B).
  int64_t clash = 0;
  chem_score(p, lig, out.best.conf, nullptr, &clash);
  cn.clash_pairs = clash;
  for (std::size_t i = 0; i < lig.n_atoms(); ++i) {
    if (!lig.heavy[i]) continue;
    bool outside = false;
    field_value(p, out.best.conf[i], &outside);
    cn.oob_samples += outside ? 1 : 0;
  }
  return out;
}

// search.cpp:278-353 (test oracle only).
Pose exhaustive_dock(const Pocket &p, const Ligand &lig) {
  if (lig.n_atoms() > 5) throw ConfigError("exhaustive dock handles at most 5 atoms");
  if (!lig.tors_bond.empty()) throw ConfigError("exhaustive dock requires a rigid ligand");
  for (int a = 0; a < 3; ++a)
    if ((p.dims[a] - 1) * p.spacing > 16.0 + 1e-9)
      throw ConfigError("exhaustive dock pocket side exceeds 16 A");
  constexpr int kOri = 512;
  constexpr double kLat = 0.25;
  const Conf base = lig.pos;
  const V3 bc = centroid(base);
  std::vector<Quat> rots;
  std::vector<Conf> rotated;
  Conf centered;
  for (std::size_t i = 0; i < lig.n_atoms(); ++i)
    if (lig.heavy[i]) centered.push_back(vsub(base[i], bc));
  for (int o = 0; o < kOri; ++o) {
    const Quat q = quat_from_angle_axis(fibonacci_rotation_angle(o), fibonacci_axis(o, kOri));
    rots.push_back(q);
    const M3 r = quat_matrix(q);
    Conf c(centered.size());
    for (std::size_t i = 0; i < centered.size(); ++i) c[i] = mat_col(r, centered[i], i);
    rotated.push_back(c);
  }
  int cnt[3];
  for (int a = 0; a < 3; ++a)
    cnt[a] = static_cast<int>(std::floor((p.dims[a] - 1) * p.spacing / kLat + 1e-9)) + 1;
  double best = -std::numeric_limits<double>::infinity();
  V3 best_pt = p.origin;
  int best_o = 0;
  for (int iz = 0; iz < cnt[2]; ++iz)
    for (int iy = 0; iy < cnt[1]; ++iy)
      for (int ix = 0; ix < cnt[0]; ++ix) {
        const V3 pt{p.origin.x + kLat * ix, p.origin.y + kLat * iy, p.origin.z + kLat * iz};
        for (int o = 0; o < kOri; ++o) {
          double s = 0.0;
          for (const V3 &v : rotated[o]) s += field_value(p, vadd(v, pt));
          if (s > best) {
            best = s;
            best_pt = pt;
            best_o = o;
          }
        }
      }
  Pose pose;
  pose.T.q = rots[static_cast<std::size_t>(best_o)];
  pose.T.t = vsub(best_pt, quat_rotate(pose.T.q, bc));
  pose.conf = apply_rigid(base, pose.T);
  pose.geo = geo_score(p, lig, pose.conf, nullptr);
  return pose;
}

// ------------------------------------------------------------ torsions
// ligand.cpp:15-139: adjacency, bridge bonds (iterative Tarjan), heavy
// degree, BFS partition, detect_torsions.
struct Graph {
  std::size_t n;
  std::vector<uint16_t> a, b;
  std::vector<uint8_t> order, heavy;
  std::vector<std::vector<std::pair<uint16_t, uint16_t>>> adj() const {
    std::vector<std::vector<std::pair<uint16_t, uint16_t>>> g(n);
    for (std::size_t i = 0; i < a.size(); ++i) {
      g[a[i]].emplace_back(b[i], static_cast<uint16_t>(i));
      g[b[i]].emplace_back(a[i], static_cast<uint16_t>(i));
    }
    return g;
  }
};
std::vector<uint8_t> reach(const std::vector<std::vector<std::pair<uint16_t, uint16_t>>> &g,
                           uint16_t start, int skip) {
  std::vector<uint8_t> seen(g.size(), 0);
  std::vector<uint16_t> stack{start};
  seen[start] = 1;
  while (!stack.empty()) {
    const uint16_t at = stack.back();
    stack.pop_back();
    for (auto [nx, bond] : g[at]) {
      if (static_cast<int>(bond) == skip || seen[nx]) continue;
      seen[nx] = 1;
      stack.push_back(nx);
    }
  }
  return seen;
}
std::vector<uint8_t> bridges(const Graph &gr) {
  const auto g = gr.adj();
  std::vector<uint8_t> br(gr.a.size(), 0);
  std::vector<int> disc(gr.n, -1), low(gr.n, 0);
  int timer = 0;
  struct F {
    uint16_t at;
    int in_bond;
    std::size_t next;
  };
  for (std::size_t root = 0; root < gr.n; ++root) {
    if (disc[root] != -1) continue;
    std::vector<F> st{{static_cast<uint16_t>(root), -1, 0}};
    disc[root] = low[root] = timer++;
    while (!st.empty()) {
      F &f = st.back();
      if (f.next < g[f.at].size()) {
        auto [nx, bond] = g[f.at][f.next++];
        if (static_cast<int>(bond) == f.in_bond) continue;
        if (disc[nx] == -1) {
          disc[nx] = low[nx] = timer++;
          st.push_back({nx, static_cast<int>(bond), 0});
        } else {
          low[f.at] = std::min(low[f.at], disc[nx]);
        }
      } else {
        const F done = f;
        st.pop_back();
        if (!st.empty()) {
          F &par = st.back();
          low[par.at] = std::min(low[par.at], low[done.at]);
          if (low[done.at] > disc[par.at]) br[static_cast<std::size_t>(done.in_bond)] = 1;
        }
      }
    }
  }
  return br;
}
int heavy_degree(const Graph &g, uint16_t atom) {
  int d = 0;
  for (std::size_t i = 0; i < g.a.size(); ++i) {
    if (g.a[i] == atom && g.heavy[g.b[i]]) ++d;
    if (g.b[i] == atom && g.heavy[g.a[i]]) ++d;
  }
  return d;
}

// ------------------------------------------------------------ batch views
Ligand ligand_from_batch(const vs_ligand_batch *b, int i) {
  Ligand l;
  const int a0 = b->atom_offset[i], a1 = b->atom_offset[i + 1];
  for (int a = a0; a < a1; ++a) {
    l.pos.push_back({b->xyz[3 * a], b->xyz[3 * a + 1], b->xyz[3 * a + 2]});
    l.elem.push_back(b->element[a]);
    l.heavy.push_back(b->is_heavy[a] ? 1 : 0);
  }
  const int b0 = b->bond_offset[i], b1 = b->bond_offset[i + 1];
  for (int k = b0; k < b1; ++k) {
    l.ba.push_back(b->bond_a[k]);
    l.bb.push_back(b->bond_b[k]);
    l.border.push_back(b->bond_order ? b->bond_order[k] : 1);
  }
  const int t0 = b->torsion_offset[i], t1 = b->torsion_offset[i + 1];
  for (int t = t0; t < t1; ++t) {
    l.tors_bond.push_back(b->torsion_bond[t]);
    l.right.emplace_back(b->right_atoms + b->right_offset[t], b->right_atoms + b->right_offset[t + 1]);
  }
  return l;
}
Pocket pocket_from_desc(const vs_pocket_desc *d) {
  Pocket p;
  p.origin = {d->origin[0], d->origin[1], d->origin[2]};
  p.spacing = d->spacing;
  for (int a = 0; a < 3; ++a) p.dims[a] = d->dims[a];
  p.values = d->values;
  p.n_protein = d->n_protein;
  p.pelem = d->protein_element;
  p.pxyz = d->protein_xyz;
  return p;
}
Conf conf_of(const double *xyz, int a0, int a1) {
  Conf c;
  for (int a = a0; a < a1; ++a) c.push_back({xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]});
  return c;
}

template <typename F>
void parallel_for(int n, int nthreads, F &&f) {
  if (nthreads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&] {
      for (int i = next++; i < n; i = next++) f(i);
    });
  for (auto &th : pool) th.join();
}

}  // namespace vso

using namespace vso;

// ============================================================== C API
extern "C" {

int vso_set_trig_mode(int mode) {
  g_trig_mode.store(mode);
  return 0;
}

void vso_config_default(vs_scoring_config *c) {
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

// dock_and_score over a batch on `nthreads` host threads (the reference's
// docker workers, pipeline.cpp:346-363).  counters (may be NULL): 9 per
// ligand in Appendix B order S, A_rigid, A_tors, R_build, P_flat, P_chem,
// P_rmsd, clash_pairs, oob_samples.
#ifdef VSO_TRACE
void vso_trace_open(const char *path) { vso::g_trace = std::fopen(path, "wb"); }
void vso_trace_close() {
  if (vso::g_trace) std::fclose(vso::g_trace);
  vso::g_trace = nullptr;
}
#endif
int vso_dock_batch(const vs_pocket_desc *pd, const vs_ligand_batch *b, const vs_scoring_config *cfg,
                   int nthreads, vs_dock_result *res, double *best_angles, double *best_conf,
                   uint64_t *counters) {
  if (cfg->restarts < 1 || cfg->rescored < 1 || !(cfg->rmsd_threshold > 0.0))
    return VS_ERR_INVALID_ARGUMENT;  // search.cpp:240-243
  const Pocket p = pocket_from_desc(pd);
  parallel_for(b->n_ligands, nthreads, [&](int i) {
    vs_dock_result &r = res[i];
    std::memset(&r, 0, sizeof(r));
    try {
      const Ligand lig = ligand_from_batch(b, i);
      DockOut o = dock_and_score(p, lig, *cfg);
      r.status = std::isfinite(o.best_score) ? VS_LIG_OK : VS_LIG_NONFINITE;
      r.best_score = o.best_score;
      r.best_geo_score = o.best.geo;
      r.rotation[0] = o.best.T.q.x;
      r.rotation[1] = o.best.T.q.y;
      r.rotation[2] = o.best.T.q.z;
      r.rotation[3] = o.best.T.q.w;
      for (int a = 0; a < 3; ++a) r.translation[a] = o.best.T.t[a];
      r.poses_evaluated = o.poses_evaluated;
      r.scoring_evals = o.cn.S;
      r.n_survivors = static_cast<int32_t>(o.n_survivors);
      r.clash_pairs = static_cast<int32_t>(o.cn.clash_pairs);
      r.oob_samples = static_cast<int32_t>(o.cn.oob_samples);
      if (best_angles)
        for (std::size_t t = 0; t < o.best.ang.size(); ++t)
          best_angles[b->torsion_offset[i] + t] = o.best.ang[t];
      if (best_conf)
        for (std::size_t a = 0; a < o.best.conf.size(); ++a) {
          const int g = b->atom_offset[i] + static_cast<int>(a);
          best_conf[3 * g] = o.best.conf[a].x;
          best_conf[3 * g + 1] = o.best.conf[a].y;
          best_conf[3 * g + 2] = o.best.conf[a].z;
        }
      if (counters) {
        uint64_t *c = counters + 9 * i;
        c[0] = o.cn.S;
        c[1] = o.cn.A_rigid;
        c[2] = o.cn.A_tors;
        c[3] = o.cn.R_build;
        c[4] = o.cn.P_flat;
        c[5] = o.cn.P_chem;
        c[6] = o.cn.P_rmsd;
        c[7] = static_cast<uint64_t>(o.cn.clash_pairs);
        c[8] = static_cast<uint64_t>(o.cn.oob_samples);
      }
    } catch (const LigandError &e) {
      r.status = e.code;
    } catch (const std::exception &) {
      r.status = VS_LIG_EMPTY;
    }
  });
  return VS_OK;
}

int vso_field_values(const vs_pocket_desc *pd, int64_t n, const double *xyz, double *out) {
  const Pocket p = pocket_from_desc(pd);
  for (int64_t i = 0; i < n; ++i) out[i] = field_value(p, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
  return VS_OK;
}

int vso_geo_score(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *conf,
                  double *out, uint64_t *evals) {
  const Pocket p = pocket_from_desc(pd);
  for (int i = 0; i < b->n_ligands; ++i) {
    const Ligand lig = ligand_from_batch(b, i);
    Counters k;
    out[i] = geo_score(p, lig, conf_of(conf, b->atom_offset[i], b->atom_offset[i + 1]), &k);
    if (evals) evals[i] = k.S;
  }
  return VS_OK;
}

int vso_chem_score(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *conf,
                   double *out) {
  const Pocket p = pocket_from_desc(pd);
  for (int i = 0; i < b->n_ligands; ++i) {
    const Ligand lig = ligand_from_batch(b, i);
    out[i] = chem_score(p, lig, conf_of(conf, b->atom_offset[i], b->atom_offset[i + 1]), nullptr,
                        nullptr);
  }
  return VS_OK;
}

int vso_flatten(const vs_ligand_batch *b, int max_sweeps, double *conf_out, double *angles_out,
                int32_t *status, int nthreads) {
  parallel_for(b->n_ligands, nthreads, [&](int i) {
    try {
      const Ligand lig = ligand_from_batch(b, i);
      auto f = flatten(lig, lig.pos, max_sweeps, nullptr);
      for (std::size_t a = 0; a < f.first.size(); ++a) {
        const int g = b->atom_offset[i] + static_cast<int>(a);
        conf_out[3 * g] = f.first[a].x;
        conf_out[3 * g + 1] = f.first[a].y;
        conf_out[3 * g + 2] = f.first[a].z;
      }
      for (std::size_t t = 0; t < f.second.size(); ++t) angles_out[b->torsion_offset[i] + t] = f.second[t];
      if (status) status[i] = VS_LIG_OK;
    } catch (const LigandError &e) {
      if (status) status[i] = e.code;
    }
  });
  return VS_OK;
}

double vso_internal_distance_sum(int n, const double *xyz) { return internal_distance_sum(conf_of(xyz, 0, n)); }

int vso_local_search(const vs_pocket_desc *pd, const vs_ligand_batch *b, const vs_scoring_config *cfg,
                     vs_pose *poses, double *angles, double *conf, uint64_t *evals, int32_t *status) {
  const Pocket p = pocket_from_desc(pd);
  for (int i = 0; i < b->n_ligands; ++i) {
    try {
      const Ligand lig = ligand_from_batch(b, i);
      const int a0 = b->atom_offset[i], a1 = b->atom_offset[i + 1];
      const int t0 = b->torsion_offset[i], t1 = b->torsion_offset[i + 1];
      Pose in;
      in.T.q = {poses[i].rotation[0], poses[i].rotation[1], poses[i].rotation[2], poses[i].rotation[3]};
      in.T.t = {poses[i].translation[0], poses[i].translation[1], poses[i].translation[2]};
      in.geo = poses[i].geo_score;
      in.ang.assign(angles + t0, angles + t1);
      in.conf = conf_of(conf, a0, a1);
      Counters k;
      Pose o = local_search(p, lig, in, *cfg, &k);
      poses[i].rotation[0] = o.T.q.x;
      poses[i].rotation[1] = o.T.q.y;
      poses[i].rotation[2] = o.T.q.z;
      poses[i].rotation[3] = o.T.q.w;
      for (int a = 0; a < 3; ++a) poses[i].translation[a] = o.T.t[a];
      poses[i].geo_score = o.geo;
      for (int t = t0; t < t1; ++t) angles[t] = o.ang[static_cast<std::size_t>(t - t0)];
      for (int a = a0; a < a1; ++a) {
        conf[3 * a] = o.conf[static_cast<std::size_t>(a - a0)].x;
        conf[3 * a + 1] = o.conf[static_cast<std::size_t>(a - a0)].y;
        conf[3 * a + 2] = o.conf[static_cast<std::size_t>(a - a0)].z;
      }
      if (evals) evals[i] = k.S;
      if (status) status[i] = VS_LIG_OK;
    } catch (const LigandError &e) {
      if (status) status[i] = e.code;
    }
  }
  return VS_OK;
}

// initial_poses for ligand 0 of the batch; out: k poses, confs: k*3N.
int vso_initial_poses(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *flat_angles,
                      int k, vs_pose *out, double *confs, uint64_t *evals) {
  try {
    const Pocket p = pocket_from_desc(pd);
    const Ligand lig = ligand_from_batch(b, 0);
    std::vector<double> fa(flat_angles, flat_angles + lig.tors_bond.size());
    Counters cn;
    auto poses = initial_poses(p, lig, lig.pos, fa, k, &cn);
    for (int i = 0; i < k; ++i) {
      out[i].rotation[0] = poses[i].T.q.x;
      out[i].rotation[1] = poses[i].T.q.y;
      out[i].rotation[2] = poses[i].T.q.z;
      out[i].rotation[3] = poses[i].T.q.w;
      for (int a = 0; a < 3; ++a) out[i].translation[a] = poses[i].T.t[a];
      out[i].geo_score = poses[i].geo;
      for (std::size_t a = 0; a < lig.n_atoms(); ++a) {
        confs[(i * lig.n_atoms() + a) * 3] = poses[i].conf[a].x;
        confs[(i * lig.n_atoms() + a) * 3 + 1] = poses[i].conf[a].y;
        confs[(i * lig.n_atoms() + a) * 3 + 2] = poses[i].conf[a].z;
      }
    }
    if (evals) *evals = cn.S;
    return VS_OK;
  } catch (const ConfigError &) {
    return VS_ERR_INVALID_ARGUMENT;
  } catch (const LigandError &e) {
    return 100 + e.code;
  }
}

// cluster_and_select for ligand 0 over n poses (geo scores + confs n*3N);
// order_out receives up to `top` pose indices; returns the count (or <0).
int vso_cluster_select(const vs_ligand_batch *b, int n, const double *geo, const double *confs,
                       double threshold, int top, int32_t *order_out) {
  try {
    const Ligand lig = ligand_from_batch(b, 0);
    std::vector<Pose> poses(static_cast<std::size_t>(n));
    const int na = static_cast<int>(lig.n_atoms());
    for (int i = 0; i < n; ++i) {
      poses[i].geo = geo[i];
      poses[i].conf = conf_of(confs + static_cast<std::size_t>(i) * na * 3, 0, na);
    }
    auto ord = cluster_and_select(poses, lig, threshold, static_cast<std::size_t>(top), nullptr);
    for (std::size_t i = 0; i < ord.size(); ++i) order_out[i] = static_cast<int32_t>(ord[i]);
    return static_cast<int>(ord.size());
  } catch (...) {
    return -1;
  }
}

int vso_exhaustive_dock(const vs_pocket_desc *pd, const vs_ligand_batch *b, vs_pose *out,
                        double *conf_out) {
  try {
    const Pocket p = pocket_from_desc(pd);
    const Ligand lig = ligand_from_batch(b, 0);
    Pose o = exhaustive_dock(p, lig);
    out->rotation[0] = o.T.q.x;
    out->rotation[1] = o.T.q.y;
    out->rotation[2] = o.T.q.z;
    out->rotation[3] = o.T.q.w;
    for (int a = 0; a < 3; ++a) out->translation[a] = o.T.t[a];
    out->geo_score = o.geo;
    for (std::size_t a = 0; a < o.conf.size(); ++a) {
      conf_out[3 * a] = o.conf[a].x;
      conf_out[3 * a + 1] = o.conf[a].y;
      conf_out[3 * a + 2] = o.conf[a].z;
    }
    return VS_OK;
  } catch (...) {
    return VS_ERR_INVALID_ARGUMENT;
  }
}

int vso_fibonacci(int k, double *axes, double *angles) {
  for (int i = 0; i < k; ++i) {
    const V3 a = fibonacci_axis(i, k);
    axes[3 * i] = a.x;
    axes[3 * i + 1] = a.y;
    axes[3 * i + 2] = a.z;
    angles[i] = fibonacci_rotation_angle(i);
  }
  return VS_OK;
}

// detect_torsions (ligand.cpp:126-139) for ligand i of a batch whose
// torsion arrays are ignored: writes the rotatable bond indices to
// bonds_out (capacity n_bonds) and, per torsion, a right-set membership
// byte mask (n_atoms each) to right_mask_out.  Returns the torsion count.
int vso_detect_torsions(const vs_ligand_batch *b, int i, uint16_t *bonds_out, uint8_t *right_mask_out) {
  Graph g;
  const int a0 = b->atom_offset[i], a1 = b->atom_offset[i + 1];
  g.n = static_cast<std::size_t>(a1 - a0);
  for (int a = a0; a < a1; ++a) g.heavy.push_back(b->is_heavy[a] ? 1 : 0);
  for (int k = b->bond_offset[i]; k < b->bond_offset[i + 1]; ++k) {
    g.a.push_back(b->bond_a[k]);
    g.b.push_back(b->bond_b[k]);
    g.order.push_back(b->bond_order[k]);
  }
  const auto br = bridges(g);
  const auto adj = g.adj();
  int m = 0;
  for (std::size_t k = 0; k < g.a.size(); ++k) {
    if (g.order[k] != 1 || !br[k]) continue;
    if (!g.heavy[g.a[k]] || !g.heavy[g.b[k]]) continue;
    if (heavy_degree(g, g.a[k]) < 2 || heavy_degree(g, g.b[k]) < 2) continue;
    const auto left = reach(adj, g.a[k], static_cast<int>(k));  // ligand.cpp:110-124
    bonds_out[m] = static_cast<uint16_t>(k);
    for (std::size_t a = 0; a < g.n; ++a) right_mask_out[m * g.n + a] = left[a] ? 0 : 1;
    ++m;
  }
  return m;
}

// The correctly rounded routine the GPU uses (include/vs_crtrig.h), host build.
void vso_sincos_cr(double x, double *s, double *c) { vs_crtrig::sincos_cr(x, s, c); }
// The search's incremental torsion trig (vs_crtrig::sincos_shift, what the
// GPU uses for neighbour angles) along random move chains: starts at lattice
// angles idx * 2pi/36, applies n_moves moves of +-step * 2^-L (L < levels),
// compares each result's hi parts with sincos_cr of the new angle.  Returns
// the number of mismatching sin or cos values out of 2 * chains * n_moves.
uint64_t vso_sincos_shift_check(int chains, int n_moves, double step, int levels, uint64_t seed) {
  uint64_t bad = 0, st = seed * 0x9e3779b97f4a7c15ull + 1;
  auto next = [&st]() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
  };
  const double lattice = 2.0 * 3.14159265358979323846 / 36;
  for (int ch = 0; ch < chains; ++ch) {
    double a = static_cast<double>(next() % 36) * lattice;
    vs_crtrig::dd sa, ca;
    vs_crtrig::sincos_dd(a, &sa, &ca);
    for (int k = 0; k < n_moves; ++k) {
      const int L = static_cast<int>(next() % static_cast<uint64_t>(levels));
      double d = step;
      for (int i = 0; i < L; ++i) d *= 0.5;
      vs_crtrig::dd sd, cd;
      vs_crtrig::sincos_dd(d, &sd, &cd);
      if (next() & 1) {
        d = -d;
        sd = vs_crtrig::dd_neg(sd);
      }
      double an;
      vs_crtrig::dd sn, cn;
      if (!vs_crtrig::sincos_shift(a, sa, ca, d, sd, cd, &an, &sn, &cn)) vs_crtrig::sincos_dd(an, &sn, &cn);
      double es, ec;
      vs_crtrig::sincos_cr(an, &es, &ec);
      bad += (sn.hi != es) + (cn.hi != ec);
      a = an;
      sa = sn;
      ca = cn;
    }
  }
  return bad;
}

void vso_sincos_glibc(double x, double *s, double *c) {
  *s = std::sin(x);
  *c = std::cos(x);
}

// Canonical pose materialisation (pose.hpp:20-22): per ligand,
// apply_rigid(apply_torsions(base, angles), T).  poses: vs_pose per ligand.
int vso_materialize(const vs_ligand_batch *b, const double *angles, const vs_pose *poses, double *conf_out,
                    int32_t *status) {
  for (int i = 0; i < b->n_ligands; ++i) {
    try {
      const Ligand lig = ligand_from_batch(b, i);
      std::vector<double> a(angles + b->torsion_offset[i], angles + b->torsion_offset[i + 1]);
      RT T;
      T.q = {poses[i].rotation[0], poses[i].rotation[1], poses[i].rotation[2], poses[i].rotation[3]};
      T.t = {poses[i].translation[0], poses[i].translation[1], poses[i].translation[2]};
      const Conf c = apply_rigid(apply_torsions(lig.pos, lig, a, nullptr), T);
      for (std::size_t k = 0; k < c.size(); ++k) {
        const int g = b->atom_offset[i] + static_cast<int>(k);
        conf_out[3 * g] = c[k].x;
        conf_out[3 * g + 1] = c[k].y;
        conf_out[3 * g + 2] = c[k].z;
      }
      if (status) status[i] = VS_LIG_OK;
    } catch (const LigandError &e) {
      if (status) status[i] = e.code;
    }
  }
  return VS_OK;
}

}  // extern "C"
