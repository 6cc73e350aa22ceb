// libvscreen_b200.so: the reference's C++ dock-path API (proj/include/vscreen,
// re-declared in include/vscreen/) implemented over the B200 C ABI.
//
// GPU-backed (libvsdock.so): dock_and_score, dock_and_score_batch, flatten,
// initial_poses, local_search, cluster_and_select, geo_score,
// pocket_field_value, build_pocket, chem_score.  Host value-type helpers
// (the reference's callers use them to post-process a DockResult):
// compose/inverse/apply_rigid/apply_torsion(s)/centroid/rmsd, the ligand
// graph queries, fibonacci_axis/angle, exhaustive_dock (a test helper,
// search.cpp:278-353).  Host helpers follow SURVEY.md Appendix A arithmetic
// through Eigen (here the Eigen-subset in third_party/; with a real Eigen
// they follow that Eigen).
//
// Pockets are uploaded once per distinct Pocket object and cached (the
// reference treats Pocket as immutable and shared).
#include <algorithm>
#include <cmath>
#include <charconv>
#include <chrono>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <mutex>
#include <numbers>
#include <numeric>
#include <optional>
#include <string>
#include <tuple>
#include <vector>

#include "vs_dock.h"
#include "vs_prep.h"
#include "vs_rank.h"
#include "vscreen/dockengine/chem.hpp"
#include "vscreen/dockengine/grid.hpp"
#include "vscreen/dockengine/search.hpp"
#include "vscreen/error.hpp"
#include "vscreen/pipeline/pipeline.hpp"

namespace vscreen {
namespace {

std::string last_error() { return std::string(vs_last_error_message()); }

void check(vs_status s, const char *what) {
  if (s == VS_OK) return;
  if (s == VS_ERR_INVALID_ARGUMENT) throw InvalidArgument(std::string(what) + ": " + last_error());
  throw DeviceError(std::string(what) + ": " + last_error());
}

// One vs_context per device, created on first use.  The calling thread's
// device is vscreen::b200::use_device() (thread-local), else $VS_DEVICE, else 0,
// so W reference-style docker threads can spread over the GPUs of a box.
constexpr int kMaxDevices = 64;
thread_local int tl_device = -1;

int current_device() {
  if (tl_device >= 0) return tl_device;
  const char *env = std::getenv("VS_DEVICE");
  return env ? std::atoi(env) : 0;
}

vs_context *context() {
  static std::mutex mu;
  static vs_context *ctx[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) throw DeviceError("vscreen::b200: device index out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!ctx[dev]) check(vs_context_create(dev, &ctx[dev]), "vs_context_create");
  return ctx[dev];
}

// SoA packing of ligands (vs_ligand_batch) with optional coordinate override.
struct Packed {
  std::vector<int32_t> ao{0}, bo{0}, to{0}, ro{0};
  std::vector<double> xyz;
  std::vector<uint8_t> el, hv, bord;
  std::vector<uint16_t> ba, bb, tb, ra;
  vs_ligand_batch view{};
  void add(const Ligand &l, const Conformation *conf = nullptr) {
    for (std::size_t i = 0; i < l.atoms.size(); ++i) {
      const Eigen::Vector3d p = conf ? Eigen::Vector3d(conf->col(static_cast<Eigen::Index>(i))) : l.atoms[i].position;
      xyz.insert(xyz.end(), {p.x(), p.y(), p.z()});
      el.push_back(static_cast<uint8_t>(l.atoms[i].element));
      hv.push_back(l.atoms[i].is_heavy ? 1 : 0);
    }
    for (const Bond &b : l.bonds) {
      ba.push_back(b.a);
      bb.push_back(b.b);
      bord.push_back(static_cast<uint8_t>(b.order));
    }
    for (const TorsionalBond &t : l.torsions) {
      tb.push_back(t.bond_index);
      ra.insert(ra.end(), t.right_set.begin(), t.right_set.end());
      ro.push_back(static_cast<int32_t>(ra.size()));
    }
    ao.push_back(static_cast<int32_t>(el.size()));
    bo.push_back(static_cast<int32_t>(ba.size()));
    to.push_back(static_cast<int32_t>(tb.size()));
  }
  const vs_ligand_batch *finish() {
    auto nn = [](auto &v) { if (v.empty()) v.resize(1); };
    nn(xyz), nn(el), nn(hv), nn(bord), nn(ba), nn(bb), nn(tb), nn(ra);
    view.n_ligands = static_cast<int32_t>(ao.size() - 1);
    view.atom_offset = ao.data();
    view.xyz = xyz.data();
    view.element = el.data();
    view.is_heavy = hv.data();
    view.bond_offset = bo.data();
    view.bond_a = ba.data();
    view.bond_b = bb.data();
    view.bond_order = bord.data();
    view.torsion_offset = to.data();
    view.torsion_bond = tb.data();
    view.right_offset = ro.data();
    view.right_atoms = ra.data();
    return &view;
  }
};

vs_scoring_config to_c(const ScoringConfig &c) {
  return {c.restarts, c.rescored, c.rmsd_threshold, c.step_translation, c.step_rotation, c.step_torsion,
          c.min_translation, c.max_iterations, c.flatten_max_sweeps};
}

// Device pockets, cached by CONTENT: the key is a 64-bit FNV-1a hash of the
// grid values, origin, spacing, dims and protein atoms, and a hit is
// confirmed against a stored copy of all of them, so a Pocket mutated in
// place or a new Pocket at a recycled address is never served the old device
// grid (the reference's own tests rebuild pockets per SUBCASE,
// test_dockengine.cpp:215-240).  One entry set per device.
struct PocketKey {
  int device = 0;
  std::vector<double> meta;  // origin (3), spacing, dims (3)
  std::vector<double> values;
  std::vector<uint8_t> el;
  std::vector<double> xyz;
  bool operator==(const PocketKey &o) const {
    return device == o.device && meta == o.meta && el == o.el && values.size() == o.values.size() &&
           xyz.size() == o.xyz.size() &&
           std::memcmp(values.data(), o.values.data(), values.size() * sizeof(double)) == 0 &&
           std::memcmp(xyz.data(), o.xyz.data(), xyz.size() * sizeof(double)) == 0;
  }
};

uint64_t fnv1a(uint64_t h, const void *p, std::size_t n) {
  const auto *b = static_cast<const unsigned char *>(p);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

struct PocketCache {
  std::mutex mu;
  std::multimap<uint64_t, std::pair<PocketKey, vs_pocket *>> map;
  vs_pocket *get(const Pocket &p) {
    PocketKey k;
    k.device = current_device();
    k.meta = {p.origin[0], p.origin[1], p.origin[2], p.spacing, double(p.dims[0]), double(p.dims[1]),
              double(p.dims[2])};
    k.values = p.values;
    for (const ProteinAtom &a : p.protein_atoms) {
      k.el.push_back(static_cast<uint8_t>(a.element));
      k.xyz.insert(k.xyz.end(), {a.position.x(), a.position.y(), a.position.z()});
    }
    uint64_t h = 1469598103934665603ull;
    h = fnv1a(h, &k.device, sizeof k.device);
    h = fnv1a(h, k.meta.data(), k.meta.size() * sizeof(double));
    h = fnv1a(h, k.values.data(), k.values.size() * sizeof(double));
    h = fnv1a(h, k.el.data(), k.el.size());
    h = fnv1a(h, k.xyz.data(), k.xyz.size() * sizeof(double));
    vs_context *ctx = context();
    std::lock_guard<std::mutex> lock(mu);
    for (auto [it, end] = map.equal_range(h); it != end; ++it)
      if (it->second.first == k) return it->second.second;
    vs_pocket_desc d{};
    for (int a = 0; a < 3; ++a) {
      d.origin[a] = p.origin[a];
      d.dims[a] = p.dims[a];
    }
    d.spacing = p.spacing;
    d.values = p.values.data();
    d.n_protein = static_cast<int32_t>(k.el.size());
    d.protein_element = k.el.empty() ? nullptr : k.el.data();
    d.protein_xyz = k.xyz.empty() ? nullptr : k.xyz.data();
    vs_pocket *hd = nullptr;
    check(vs_pocket_create(ctx, &d, &hd), "vs_pocket_create");
    if (map.size() >= 64) {  // bounded: drop everything (pockets are cheap to re-upload)
      for (auto &kv : map) vs_pocket_destroy(kv.second.second);
      map.clear();
    }
    map.emplace(h, std::make_pair(std::move(k), hd));
    return hd;
  }
};
PocketCache &pockets() {
  static PocketCache c;
  return c;
}

const char *status_text(int st) {
  switch (st) {
    case VS_LIG_EMPTY: return "empty conformation";
    case VS_LIG_DEGENERATE_AXIS: return "degenerate torsion axis";
    case VS_LIG_BAD_TORSION: return "torsion index out of range";
    case VS_LIG_NO_HEAVY: return "no heavy atoms";
    case VS_LIG_TOO_LARGE: return "ligand exceeds the B200 kernel limits";
    default: return "ligand error";
  }
}

Conformation conf_from(const double *xyz, int n) {
  Conformation c(3, n);
  for (int i = 0; i < n; ++i) c.col(i) = Eigen::Vector3d(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  return c;
}

constexpr double kPi = std::numbers::pi;

}  // namespace

// ------------------------------------------------------------ ligand graph
std::vector<std::vector<std::pair<std::uint16_t, std::uint16_t>>> adjacency(const Ligand &ligand) {
  std::vector<std::vector<std::pair<std::uint16_t, std::uint16_t>>> adj(ligand.atoms.size());
  for (std::size_t i = 0; i < ligand.bonds.size(); ++i) {
    adj[ligand.bonds[i].a].emplace_back(ligand.bonds[i].b, static_cast<std::uint16_t>(i));
    adj[ligand.bonds[i].b].emplace_back(ligand.bonds[i].a, static_cast<std::uint16_t>(i));
  }
  return adj;
}

static std::vector<bool> reach(const Ligand &l, std::uint16_t start, int skip) {
  const auto adj = adjacency(l);
  std::vector<bool> seen(adj.size(), false);
  std::vector<std::uint16_t> st{start};
  seen[start] = true;
  while (!st.empty()) {
    const auto at = st.back();
    st.pop_back();
    for (auto [nx, b] : adj[at])
      if (static_cast<int>(b) != skip && !seen[nx]) {
        seen[nx] = true;
        st.push_back(nx);
      }
  }
  return seen;
}

bool is_connected(const Ligand &ligand) {
  if (ligand.atoms.empty()) return false;
  const auto s = reach(ligand, 0, -1);
  return std::all_of(s.begin(), s.end(), [](bool v) { return v; });
}

std::vector<bool> bridge_bonds(const Ligand &ligand) {
  Packed pk;
  pk.add(ligand);
  std::vector<uint8_t> out(std::max<std::size_t>(ligand.bonds.size(), 1));
  if (vs_bridge_bonds(pk.finish(), 0, out.data()) < 0) throw InvalidArgument("bond index out of range");
  return std::vector<bool>(out.begin(), out.begin() + static_cast<std::ptrdiff_t>(ligand.bonds.size()));
}

int heavy_degree(const Ligand &ligand, std::uint16_t atom) {
  int d = 0;
  for (const Bond &b : ligand.bonds) {
    if (b.a == atom && ligand.atoms[b.b].is_heavy) ++d;
    if (b.b == atom && ligand.atoms[b.a].is_heavy) ++d;
  }
  return d;
}

TorsionalBond torsion_partition(const Ligand &ligand, std::uint16_t bond_index) {
  if (bond_index >= ligand.bonds.size()) throw InvalidArgument("torsion bond index out of range");
  const Bond &bond = ligand.bonds[bond_index];
  const auto left = reach(ligand, bond.a, bond_index);
  if (left[bond.b]) throw InvalidArgument("torsion bond is not a bridge");
  TorsionalBond t;
  t.bond_index = bond_index;
  for (std::uint16_t i = 0; i < ligand.atoms.size(); ++i) (left[i] ? t.left_set : t.right_set).push_back(i);
  return t;
}

Ligand detect_torsions(Ligand ligand) {
  Packed pk;
  ligand.torsions.clear();
  pk.add(ligand);
  const std::size_t nb = std::max<std::size_t>(ligand.bonds.size(), 1), na = std::max<std::size_t>(ligand.atoms.size(), 1);
  std::vector<uint16_t> bonds(nb);
  std::vector<uint8_t> masks(nb * na);
  const int m = vs_detect_torsions(pk.finish(), 0, bonds.data(), masks.data());
  if (m < 0) throw InvalidArgument("bond index out of range");
  for (int t = 0; t < m; ++t) ligand.torsions.push_back(torsion_partition(ligand, bonds[static_cast<std::size_t>(t)]));
  return ligand;
}

// ------------------------------------------------------------ geometry (host helpers)
RigidTransform identity_transform() { return RigidTransform{}; }

RigidTransform compose(const RigidTransform &b, const RigidTransform &a) {
  RigidTransform o;
  o.rotation = (b.rotation * a.rotation).normalized();
  o.translation = b.rotation * a.translation + b.translation;
  return o;
}

RigidTransform inverse(const RigidTransform &t) {
  RigidTransform o;
  o.rotation = t.rotation.conjugate();
  o.translation = -(o.rotation * t.translation);
  return o;
}

Conformation apply_rigid(const Conformation &conf, const RigidTransform &t) {
  const Conformation rotated = t.rotation.toRotationMatrix() * conf;
  return rotated.colwise() + t.translation;
}

Conformation conformation_of(const Ligand &ligand) {
  Conformation c(3, static_cast<Eigen::Index>(ligand.atoms.size()));
  for (std::size_t i = 0; i < ligand.atoms.size(); ++i) c.col(static_cast<Eigen::Index>(i)) = ligand.atoms[i].position;
  return c;
}

Ligand with_conformation(Ligand ligand, const Conformation &conf) {
  if (conf.cols() != static_cast<Eigen::Index>(ligand.atoms.size()))
    throw InvalidArgument("conformation length does not match atom count");
  for (std::size_t i = 0; i < ligand.atoms.size(); ++i) ligand.atoms[i].position = conf.col(static_cast<Eigen::Index>(i));
  return ligand;
}

Eigen::Vector3d centroid(const Conformation &conf) {
  if (conf.cols() == 0) throw InvalidArgument("empty conformation");
  return conf.rowwise().mean();
}

Conformation apply_torsion(const Conformation &conf, const Ligand &ligand, const TorsionalBond &torsion, double angle) {
  if (torsion.bond_index >= ligand.bonds.size()) throw InvalidArgument("torsion bond index out of range");
  const Bond &bond = ligand.bonds[torsion.bond_index];
  const Eigen::Vector3d pivot = conf.col(bond.a);
  const Eigen::Vector3d axis = Eigen::Vector3d(conf.col(bond.b)) - pivot;
  const double len = axis.norm();
  if (len < 1e-9) throw InvalidArgument("degenerate torsion axis");
  const Eigen::AngleAxisd rot(angle, axis / len);
  Conformation out = conf;
  for (const std::uint16_t idx : torsion.right_set) {
    if (idx >= conf.cols()) throw InvalidArgument("torsion atom index out of range");
    out.col(idx) = rot * (Eigen::Vector3d(conf.col(idx)) - pivot) + pivot;
  }
  return out;
}

Conformation apply_torsions(const Conformation &base, const Ligand &ligand, const std::vector<double> &angles) {
  if (angles.size() != ligand.torsions.size()) throw InvalidArgument("torsion angle count does not match ligand");
  Conformation c = base;
  for (std::size_t i = 0; i < angles.size(); ++i) c = apply_torsion(c, ligand, ligand.torsions[i], angles[i]);
  return c;
}

double internal_distance_sum(const Conformation &conf) {
  double s = 0.0;
  for (Eigen::Index i = 0; i < conf.cols(); ++i)
    for (Eigen::Index j = i + 1; j < conf.cols(); ++j)
      s += (Eigen::Vector3d(conf.col(i)) - Eigen::Vector3d(conf.col(j))).norm();
  return s;
}

double rmsd(const Conformation &a, const Conformation &b) {
  if (a.cols() != b.cols()) throw InvalidArgument("conformation length mismatch");
  if (a.cols() == 0) throw InvalidArgument("empty conformation");
  double s = 0.0;
  for (Eigen::Index i = 0; i < a.cols(); ++i) s += (Eigen::Vector3d(a.col(i)) - Eigen::Vector3d(b.col(i))).squaredNorm();
  return std::sqrt(s / static_cast<double>(a.cols()));
}

double heavy_atom_rmsd(const Conformation &a, const Conformation &b, const Ligand &ligand) {
  if (a.cols() != b.cols() || a.cols() != static_cast<Eigen::Index>(ligand.atoms.size()))
    throw InvalidArgument("conformation length mismatch");
  double s = 0.0;
  std::size_t heavy = 0;
  for (Eigen::Index i = 0; i < a.cols(); ++i) {
    if (!ligand.atoms[static_cast<std::size_t>(i)].is_heavy) continue;
    s += (Eigen::Vector3d(a.col(i)) - Eigen::Vector3d(b.col(i))).squaredNorm();
    ++heavy;
  }
  if (heavy == 0) throw InvalidArgument("no heavy atoms");
  return std::sqrt(s / static_cast<double>(heavy));
}

// ------------------------------------------------------------ grid / chem (GPU)
Pocket build_pocket(const std::vector<ProteinAtom> &protein, const std::string &id, const Eigen::Vector3d &center,
                    double radius, double spacing) {
  std::vector<uint8_t> el;
  std::vector<double> xyz;
  for (const ProteinAtom &a : protein) {
    el.push_back(static_cast<uint8_t>(a.element));
    xyz.insert(xyz.end(), {a.position.x(), a.position.y(), a.position.z()});
  }
  const double c[3] = {center.x(), center.y(), center.z()};
  vs_pocket *h = nullptr;
  check(vs_pocket_build(context(), static_cast<int32_t>(el.size()), el.empty() ? nullptr : el.data(),
                        xyz.empty() ? nullptr : xyz.data(), c, radius, spacing, &h),
        "build_pocket");
  Pocket p;
  p.id = id;
  double org[3], sp;
  int32_t dims[3], np;
  vs_pocket_info(h, org, &sp, dims, &np);
  p.origin = Eigen::Vector3d(org[0], org[1], org[2]);
  p.spacing = sp;
  p.dims = {dims[0], dims[1], dims[2]};
  p.values.resize(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
  const vs_status st = vs_pocket_download(context(), h, p.values.data());
  vs_pocket_destroy(h);
  check(st, "build_pocket download");
  p.protein_atoms = protein;
  return p;
}

double pocket_field_value(const Pocket &pocket, const Eigen::Vector3d &point) {
  const double xyz[3] = {point.x(), point.y(), point.z()};
  double out = 0.0;
  check(vs_field_values(context(), pockets().get(pocket), 1, xyz, &out), "pocket_field_value");
  return out;
}

double geo_score(const Pocket &pocket, const Ligand &ligand, const Conformation &conf, EvalCounter *counter) {
  Packed pk;
  pk.add(ligand, &conf);
  double out = 0.0;
  uint64_t ev = 0;
  check(vs_geo_score_batch(context(), pockets().get(pocket), pk.finish(), pk.xyz.data(), &out, &ev), "geo_score");
  if (counter) counter->scoring_evals += ev;
  return out;
}

double chem_pair_weight(ChemClass a, ChemClass b) {
  if (a == ChemClass::Other || b == ChemClass::Other) return 0.05;
  if (a == ChemClass::Hydrophobic && b == ChemClass::Hydrophobic) return 0.4;
  if (a == ChemClass::Polar && b == ChemClass::Polar) return 1.0;
  return 0.1;
}

double chem_score(const Pocket &pocket, const Ligand &ligand, const Conformation &conf) {
  Packed pk;
  pk.add(ligand, &conf);
  double out = 0.0;
  check(vs_chem_score_batch(context(), pockets().get(pocket), pk.finish(), pk.xyz.data(), &out), "chem_score");
  return out;
}

// ------------------------------------------------------------ search (GPU)
FlattenResult flatten(const Ligand &ligand, const Conformation &base, int max_sweeps) {
  Packed pk;
  pk.add(ligand, &base);
  const int n = static_cast<int>(ligand.atoms.size()), m = static_cast<int>(ligand.torsions.size());
  std::vector<double> conf(static_cast<std::size_t>(std::max(3 * n, 3))), ang(static_cast<std::size_t>(std::max(m, 1)));
  int32_t st = 0;
  check(vs_flatten_batch(context(), pk.finish(), max_sweeps, conf.data(), ang.data(), &st), "flatten");
  if (st != VS_LIG_OK) throw InvalidArgument(status_text(st));
  return {conf_from(conf.data(), n), std::vector<double>(ang.begin(), ang.begin() + m)};
}

Eigen::Vector3d fibonacci_axis(int i, int k) {
  constexpr double kGoldenRatio = 1.6180339887498948482;
  constexpr double kGoldenAngle = 2.0 * kPi * (2.0 - kGoldenRatio);
  const double z = 1.0 - 2.0 * (i + 0.5) / static_cast<double>(k);
  const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
  const double az = std::fmod(i * kGoldenAngle, 2.0 * kPi);
  return {r * std::cos(az), r * std::sin(az), z};
}

double fibonacci_rotation_angle(int i) {
  constexpr double kGoldenRatio = 1.6180339887498948482;
  return 2.0 * kPi * std::fmod(i * kGoldenRatio, 1.0);
}

std::vector<Pose> initial_poses(const Pocket &pocket, const Ligand &ligand, const Conformation &base,
                                const std::vector<double> &flat_angles, int k, EvalCounter *counter) {
  if (k < 1) throw InvalidArgument("restart count must be at least 1");
  Packed pk;
  pk.add(ligand, &base);
  const int n = static_cast<int>(ligand.atoms.size());
  std::vector<vs_pose> poses(static_cast<std::size_t>(k));
  std::vector<double> conf(static_cast<std::size_t>(std::max(3 * n * k, 3)));
  uint64_t ev = 0;
  int32_t st = 0;
  check(vs_initial_poses(context(), pockets().get(pocket), pk.finish(), flat_angles.data(), k, poses.data(),
                         conf.data(), &ev, &st),
        "initial_poses");
  if (st != VS_LIG_OK) throw InvalidArgument(status_text(st));
  if (counter) counter->scoring_evals += ev;
  std::vector<Pose> out(static_cast<std::size_t>(k));
  for (int i = 0; i < k; ++i) {
    Pose &p = out[static_cast<std::size_t>(i)];
    p.transform.rotation = Eigen::Quaterniond(poses[i].rotation[3], poses[i].rotation[0], poses[i].rotation[1],
                                              poses[i].rotation[2]);
    p.transform.translation = Eigen::Vector3d(poses[i].translation[0], poses[i].translation[1], poses[i].translation[2]);
    p.torsion_angles = flat_angles;
    p.conformation = conf_from(conf.data() + static_cast<std::size_t>(3 * n * i), n);
    p.geo_score = poses[i].geo_score;
  }
  return out;
}

Pose local_search(const Pocket &pocket, const Ligand &ligand, Pose pose, const ScoringConfig &config,
                  EvalCounter *counter) {
  Packed pk;
  pk.add(ligand);
  const vs_scoring_config cfg = to_c(config);
  vs_pose p{};
  p.rotation[0] = pose.transform.rotation.x();
  p.rotation[1] = pose.transform.rotation.y();
  p.rotation[2] = pose.transform.rotation.z();
  p.rotation[3] = pose.transform.rotation.w();
  for (int a = 0; a < 3; ++a) p.translation[a] = pose.transform.translation[a];
  p.geo_score = pose.geo_score;
  std::vector<double> ang = pose.torsion_angles;
  if (ang.empty()) ang.push_back(0.0);
  const int n = static_cast<int>(ligand.atoms.size());
  std::vector<double> conf(static_cast<std::size_t>(std::max(3 * n, 3)));
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) conf[static_cast<std::size_t>(3 * i + c)] = pose.conformation(c, i);
  uint64_t ev = 0;
  int32_t st = 0;
  check(vs_local_search_batch(context(), pockets().get(pocket), pk.finish(), &cfg, &p, ang.data(), conf.data(), &ev,
                              &st),
        "local_search");
  if (st != VS_LIG_OK) throw InvalidArgument(status_text(st));
  if (counter) counter->scoring_evals += ev;
  pose.transform.rotation = Eigen::Quaterniond(p.rotation[3], p.rotation[0], p.rotation[1], p.rotation[2]);
  pose.transform.translation = Eigen::Vector3d(p.translation[0], p.translation[1], p.translation[2]);
  pose.geo_score = p.geo_score;
  for (std::size_t t = 0; t < pose.torsion_angles.size(); ++t) pose.torsion_angles[t] = ang[t];
  pose.conformation = conf_from(conf.data(), n);
  return pose;
}

std::vector<Pose> cluster_and_select(const std::vector<Pose> &poses, const Ligand &ligand, double threshold,
                                     std::size_t top) {
  if (poses.empty()) throw InvalidArgument("cannot cluster an empty pose list");
  Packed pk;
  pk.add(ligand);
  const int n = static_cast<int>(ligand.atoms.size());
  std::vector<double> geo, confs;
  for (const Pose &p : poses) {
    if (p.conformation.cols() != n) throw InvalidArgument("conformation length mismatch");
    geo.push_back(p.geo_score);
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) confs.push_back(p.conformation(c, i));
  }
  if (confs.empty()) confs.push_back(0.0);
  std::vector<int32_t> order(poses.size());
  int32_t count = 0;
  check(vs_cluster_select(context(), pk.finish(), static_cast<int32_t>(poses.size()), geo.data(), confs.data(),
                          threshold, static_cast<int32_t>(std::min<std::size_t>(top, poses.size())), order.data(),
                          &count),
        "cluster_and_select");
  std::vector<Pose> out;
  for (int i = 0; i < count; ++i) out.push_back(poses[static_cast<std::size_t>(order[static_cast<std::size_t>(i)])]);
  return out;
}

std::vector<DockResult> dock_and_score_batch(const Pocket &pocket, std::span<const Ligand> ligands,
                                             const ScoringConfig &config, std::vector<std::string> *errors) {
  Packed pk;
  for (const Ligand &l : ligands) pk.add(l);
  const vs_scoring_config cfg = to_c(config);
  std::vector<vs_dock_result> res(std::max<std::size_t>(ligands.size(), 1));
  std::vector<double> ang(std::max<std::size_t>(pk.tb.size(), 1)), conf(std::max<std::size_t>(pk.xyz.size(), 3));
  const vs_ligand_batch *view = pk.finish();
  check(vs_dock_batch(context(), pockets().get(pocket), view, &cfg, res.data(), ang.data(), conf.data()),
        "dock_and_score");
  std::vector<DockResult> out(ligands.size());
  if (errors) errors->assign(ligands.size(), std::string());
  for (std::size_t i = 0; i < ligands.size(); ++i) {
    DockResult &d = out[i];
    d.smiles = ligands[i].name;
    const vs_dock_result &r = res[i];
    if (r.status != VS_LIG_OK && r.status != VS_LIG_NONFINITE) {
      d.best_score = std::numeric_limits<double>::quiet_NaN();
      if (errors) (*errors)[i] = status_text(r.status);
      continue;
    }
    d.best_score = r.best_score;
    d.poses_evaluated = r.poses_evaluated;
    d.scoring_evals = r.scoring_evals;
    Pose &p = d.best_pose;
    p.transform.rotation = Eigen::Quaterniond(r.rotation[3], r.rotation[0], r.rotation[1], r.rotation[2]);
    p.transform.translation = Eigen::Vector3d(r.translation[0], r.translation[1], r.translation[2]);
    p.torsion_angles.assign(ang.begin() + view->torsion_offset[i], ang.begin() + view->torsion_offset[i + 1]);
    const int a0 = view->atom_offset[i], n = view->atom_offset[i + 1] - a0;
    p.conformation = conf_from(conf.data() + 3 * static_cast<std::size_t>(a0), n);
    p.geo_score = r.best_geo_score;
    p.chem_score = r.best_score;
  }
  return out;
}

DockResult dock_and_score(const Pocket &pocket, const Ligand &ligand, const ScoringConfig &config) {
  if (config.restarts < 1) throw InvalidArgument("restarts must be at least 1");
  if (config.rescored < 1) throw InvalidArgument("rescored must be at least 1");
  if (!(config.rmsd_threshold > 0.0)) throw InvalidArgument("rmsd threshold must be positive");
  std::vector<std::string> err;
  auto out = dock_and_score_batch(pocket, std::span<const Ligand>(&ligand, 1), config, &err);
  if (!err[0].empty()) throw InvalidArgument(err[0]);
  return out[0];
}

// Test helper of the reference (search.cpp:278-353): brute force on the host.
Pose exhaustive_dock(const Pocket &pocket, const Ligand &ligand) {
  if (ligand.atoms.size() > 5) throw InvalidArgument("exhaustive dock handles at most 5 atoms");
  if (!ligand.torsions.empty()) throw InvalidArgument("exhaustive dock requires a rigid ligand");
  for (int axis = 0; axis < 3; ++axis)
    if ((pocket.dims[axis] - 1) * pocket.spacing > 16.0 + 1e-9)
      throw InvalidArgument("exhaustive dock pocket side exceeds 16 A");
  const Conformation base = conformation_of(ligand);
  const Eigen::Vector3d c = centroid(base);
  std::vector<Eigen::Vector3d> heavy;
  for (std::size_t i = 0; i < ligand.atoms.size(); ++i)
    if (ligand.atoms[i].is_heavy) heavy.push_back(Eigen::Vector3d(base.col(static_cast<Eigen::Index>(i))) - c);
  Conformation centered(3, static_cast<Eigen::Index>(heavy.size()));
  for (std::size_t i = 0; i < heavy.size(); ++i) centered.col(static_cast<Eigen::Index>(i)) = heavy[i];
  constexpr int kOri = 512;
  std::vector<Eigen::Quaterniond> rots;
  std::vector<Conformation> rotated;
  for (int o = 0; o < kOri; ++o) {
    rots.emplace_back(Eigen::AngleAxisd(fibonacci_rotation_angle(o), fibonacci_axis(o, kOri)));
    rotated.push_back(rots.back().toRotationMatrix() * centered);
  }
  int cnt[3];
  for (int a = 0; a < 3; ++a) cnt[a] = static_cast<int>(std::floor((pocket.dims[a] - 1) * pocket.spacing / 0.25 + 1e-9)) + 1;
  // node-value sampling through the GPU, one batched call per lattice plane
  double best = -std::numeric_limits<double>::infinity();
  Eigen::Vector3d best_pt = pocket.origin;
  int best_o = 0;
  for (int iz = 0; iz < cnt[2]; ++iz) {
    std::vector<double> pts;
    for (int iy = 0; iy < cnt[1]; ++iy)
      for (int ix = 0; ix < cnt[0]; ++ix) {
        const Eigen::Vector3d pt = pocket.origin + 0.25 * Eigen::Vector3d(ix, iy, iz);
        for (int o = 0; o < kOri; ++o)
          for (Eigen::Index a = 0; a < centered.cols(); ++a) {
            const Eigen::Vector3d q = Eigen::Vector3d(rotated[o].col(a)) + pt;
            pts.insert(pts.end(), {q.x(), q.y(), q.z()});
          }
      }
    std::vector<double> vals(pts.size() / 3 + 1);
    check(vs_field_values(context(), pockets().get(pocket), static_cast<int64_t>(pts.size() / 3), pts.data(),
                          vals.data()),
          "exhaustive_dock");
    std::size_t at = 0;
    for (int iy = 0; iy < cnt[1]; ++iy)
      for (int ix = 0; ix < cnt[0]; ++ix) {
        const Eigen::Vector3d pt = pocket.origin + 0.25 * Eigen::Vector3d(ix, iy, iz);
        for (int o = 0; o < kOri; ++o) {
          double s = 0.0;
          for (Eigen::Index a = 0; a < centered.cols(); ++a) s += vals[at++];
          if (s > best) {
            best = s;
            best_pt = pt;
            best_o = o;
          }
        }
      }
  }
  Pose pose;
  pose.transform.rotation = rots[static_cast<std::size_t>(best_o)];
  pose.transform.translation = best_pt - pose.transform.rotation * c;
  pose.conformation = apply_rigid(base, pose.transform);
  pose.geo_score = geo_score(pocket, ligand, pose.conformation);
  return pose;
}

}  // namespace vscreen

// ------------------------------------------------------------ pipeline
namespace vscreen {

// io.hpp: sources and sinks
std::size_t MemorySource::read_at(std::uint64_t offset, std::span<std::uint8_t> out) {
  if (offset >= bytes_.size()) return 0;
  const std::size_t n = std::min<std::size_t>(out.size(), bytes_.size() - static_cast<std::size_t>(offset));
  std::memcpy(out.data(), bytes_.data() + offset, n);
  return n;
}

FileSource::FileSource(const std::string &path) : in_(path, std::ios::binary), path_(path) {
  if (!in_) throw IoError("cannot open input '" + path + "'");
  in_.seekg(0, std::ios::end);
  size_ = static_cast<std::uint64_t>(in_.tellg());
}

std::size_t FileSource::read_at(std::uint64_t offset, std::span<std::uint8_t> out) {
  if (offset >= size_) return 0;
  in_.clear();
  in_.seekg(static_cast<std::streamoff>(offset));
  in_.read(reinterpret_cast<char *>(out.data()), static_cast<std::streamsize>(out.size()));
  if (in_.bad()) throw IoError("read failed on '" + path_ + "'");
  return static_cast<std::size_t>(in_.gcount());
}

FileSink::FileSink(const std::string &path) : out_(path, std::ios::binary | std::ios::trunc), path_(path) {
  if (!out_) throw IoError("cannot open output '" + path + "'");
}

void FileSink::write(std::string_view bytes) {
  out_.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!out_) throw IoError("write failed on '" + path_ + "'");
}

void FileSink::finish() {
  out_.flush();
  if (!out_) throw IoError("cannot finish output '" + path_ + "'");
}

std::vector<RankPlan> plan_slabs(std::uint64_t file_size, int n_ranks) {
  if (n_ranks < 1) throw InvalidArgument("rank count must be at least 1");
  std::vector<RankPlan> plans(static_cast<std::size_t>(n_ranks));
  for (int i = 0; i < n_ranks; ++i) {
    RankPlan &p = plans[static_cast<std::size_t>(i)];
    p.rank = i;
    p.n_ranks = n_ranks;
    p.slab_start = file_size * static_cast<std::uint64_t>(i) / static_cast<std::uint64_t>(n_ranks);
    p.slab_stop = file_size * static_cast<std::uint64_t>(i + 1) / static_cast<std::uint64_t>(n_ranks);
  }
  return plans;
}

std::string format_row(const OutputRow &row) {
  if (!std::isfinite(row.score)) throw InvalidArgument("output row score must be finite");
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, row.score, std::chars_format::fixed, 4);
  if (r.ec != std::errc()) throw InvalidArgument("output row score does not format");
  std::string line = row.smiles;
  line += '\t';
  line.append(buf, r.ptr);
  line += '\n';
  return line;
}

namespace {
// RankStats fields in the .stats file's order: (key, integer member or
// seconds member)
struct StatField {
  const char *key;
  std::uint64_t RankStats::*u64;
  double RankStats::*sec;
  int RankStats::*i32;
  std::size_t RankStats::*sz;
};
const StatField kStatFields[] = {
    {"ligands_docked", &RankStats::ligands_docked, nullptr, nullptr, nullptr},
    {"records_skipped", &RankStats::records_skipped, nullptr, nullptr, nullptr},
    {"dock_errors", &RankStats::dock_errors, nullptr, nullptr, nullptr},
    {"rows_written", &RankStats::rows_written, nullptr, nullptr, nullptr},
    {"chunks_read", &RankStats::chunks_read, nullptr, nullptr, nullptr},
    {"bytes_read", &RankStats::bytes_read, nullptr, nullptr, nullptr},
    {"write_calls", &RankStats::write_calls, nullptr, nullptr, nullptr},
    {"bytes_written", &RankStats::bytes_written, nullptr, nullptr, nullptr},
    {"workers", nullptr, nullptr, &RankStats::workers, nullptr},
    {"wall_seconds", nullptr, &RankStats::wall_seconds, nullptr, nullptr},
    {"reader_busy_seconds", nullptr, &RankStats::reader_busy_seconds, nullptr, nullptr},
    {"splitter_busy_seconds", nullptr, &RankStats::splitter_busy_seconds, nullptr, nullptr},
    {"docker_busy_seconds", nullptr, &RankStats::docker_busy_seconds, nullptr, nullptr},
    {"writer_busy_seconds", nullptr, &RankStats::writer_busy_seconds, nullptr, nullptr},
    {"chunk_queue_high_water", nullptr, nullptr, nullptr, &RankStats::chunk_queue_high_water},
    {"item_queue_high_water", nullptr, nullptr, nullptr, &RankStats::item_queue_high_water},
    {"row_queue_high_water", nullptr, nullptr, nullptr, &RankStats::row_queue_high_water},
};
}  // namespace

std::string format_rank_stats(const RankStats &st) {
  std::string out;
  for (const StatField &f : kStatFields) {
    out += f.key;
    out += '=';
    if (f.sec) {
      char buf[64];
      const auto r = std::to_chars(buf, buf + sizeof buf, st.*f.sec, std::chars_format::fixed, 6);
      out += r.ec == std::errc() ? std::string(buf, r.ptr) : std::string("0.000000");
    } else if (f.u64) {
      out += std::to_string(st.*f.u64);
    } else if (f.i32) {
      out += std::to_string(st.*f.i32);
    } else {
      out += std::to_string(st.*f.sz);
    }
    out += '\n';
  }
  return out;
}

RankStats parse_rank_stats(std::string_view text) {
  RankStats st;
  std::size_t at = 0;
  while (at < text.size()) {
    std::size_t eol = text.find('\n', at);
    if (eol == std::string_view::npos) eol = text.size();
    const std::string_view line = text.substr(at, eol - at);
    const std::size_t line_at = at;
    at = eol + 1;
    if (line.empty()) continue;
    const std::size_t eq = line.find('=');
    if (eq == std::string_view::npos) throw ParseError("stats line missing '='", line_at);
    const std::string_view key = line.substr(0, eq), value = line.substr(eq + 1);
    const StatField *f = nullptr;
    for (const StatField &c : kStatFields)
      if (key == c.key) f = &c;
    if (!f) throw ParseError("unknown stats key '" + std::string(key) + "'", line_at);
    const char *b = value.data(), *e = value.data() + value.size();
    if (f->sec) {
      double v = 0.0;
      const auto r = std::from_chars(b, e, v);
      if (r.ec != std::errc() || r.ptr != e) throw ParseError("bad stats value '" + std::string(value) + "'", line_at);
      st.*f->sec = v;
    } else {
      std::uint64_t v = 0;
      const auto r = std::from_chars(b, e, v);
      if (r.ec != std::errc() || r.ptr != e) throw ParseError("bad stats count '" + std::string(value) + "'", line_at);
      if (f->u64) st.*f->u64 = v;
      else if (f->i32) st.*f->i32 = static_cast<int>(v);
      else st.*f->sz = static_cast<std::size_t>(v);
    }
  }
  return st;
}

namespace {
struct RankIo {
  ByteSource *src;
  Sink *sink;
  std::string error;
};
int64_t rank_read(void *u, uint64_t off, uint8_t *out, int64_t n) {
  auto *io = static_cast<RankIo *>(u);
  try {
    return static_cast<int64_t>(io->src->read_at(off, std::span<std::uint8_t>(out, static_cast<std::size_t>(n))));
  } catch (const std::exception &e) {
    io->error = e.what();
    return -1;
  }
}
int32_t rank_write(void *u, const char *b, int64_t n) {
  auto *io = static_cast<RankIo *>(u);
  try {
    io->sink->write(std::string_view(b, static_cast<std::size_t>(n)));
    return 0;
  } catch (const std::exception &e) {
    io->error = e.what();
    return 1;
  }
}
}  // namespace

DockerStats docker_worker(BoundedQueue<WorkItem> &in, BoundedQueue<OutputRow> &out, const Pocket &pocket,
                          const ScoringConfig &scoring, double synthetic_slowdown) {
  if (synthetic_slowdown < 1.0) throw InvalidArgument("synthetic slowdown must be at least 1");
  constexpr std::size_t kBatch = 65536;
  DockerStats st;
  std::vector<Ligand> batch;
  std::vector<std::string> errors;
  while (std::optional<WorkItem> first = in.pop()) {
    const auto t0 = std::chrono::steady_clock::now();
    batch.clear();
    batch.push_back(std::move(first->ligand));
    while (batch.size() < kBatch) {
      std::optional<WorkItem> next = in.try_pop();
      if (!next) break;
      batch.push_back(std::move(next->ligand));
    }
    errors.clear();
    const std::vector<DockResult> res = dock_and_score_batch(pocket, batch, scoring, &errors);
    st.busy_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t i = 0; i < batch.size(); ++i) {
      if (!errors[i].empty() || !std::isfinite(res[i].best_score)) {
        ++st.dock_errors;
        continue;
      }
      if (!out.push(OutputRow{res[i].smiles, res[i].best_score})) return st;  // writer gone
      ++st.rows;
    }
  }
  return st;
}

RankStats run_rank(const RankPlan &plan, ByteSource &source, Sink &sink, const Pocket &pocket,
                   const PipelineConfig &config) {
  int total = 0;
  for (const WorkerClass &wc : config.workers) {
    if (wc.count < 0) throw InvalidArgument("worker count must not be negative");
    if (wc.synthetic_slowdown < 1.0) throw InvalidArgument("synthetic slowdown must be at least 1");
    total += wc.count;
  }
  if (total < 1) throw InvalidArgument("need at least one worker");
  if (config.chunk_bytes == 0) throw InvalidArgument("chunk size must be positive");
  if (plan.slab_start > plan.slab_stop) throw InvalidArgument("slab start past slab stop");
  if (plan.slab_stop > source.size()) throw InvalidArgument("slab exceeds the input size");
  std::vector<uint8_t> el;
  std::vector<double> xyz;
  for (const ProteinAtom &a : pocket.protein_atoms) {
    el.push_back(static_cast<uint8_t>(a.element));
    xyz.insert(xyz.end(), {a.position.x(), a.position.y(), a.position.z()});
  }
  vs_pocket_desc d{};
  for (int a = 0; a < 3; ++a) {
    d.origin[a] = pocket.origin[a];
    d.dims[a] = pocket.dims[a];
  }
  d.spacing = pocket.spacing;
  d.values = pocket.values.data();
  d.n_protein = static_cast<int32_t>(el.size());
  d.protein_element = el.empty() ? nullptr : el.data();
  d.protein_xyz = xyz.empty() ? nullptr : xyz.data();
  vs_rank_config rc;
  vs_rank_config_default(&rc);
  int32_t dev = 0;
  if (tl_device >= 0) {  // the calling thread pinned a GPU (b200::use_device)
    dev = tl_device;
    rc.n_devices = 1;
    rc.devices = &dev;
  }
  rc.workers_per_device = total;
  rc.chunk_bytes = static_cast<int64_t>(config.chunk_bytes);
  rc.writer_buffer_bytes = static_cast<int64_t>(std::max<std::size_t>(config.writer_buffer_bytes, 1));
  const vs_scoring_config cfg = to_c(config.scoring);
  RankIo io{&source, &sink, {}};
  vs_rank_stats st{};
  const vs_status rs = vs_run_rank(source.size(), rank_read, &io, plan.slab_start, plan.slab_stop, &d, &cfg, &rc,
                                   rank_write, &io, &st);
  if (!io.error.empty()) throw IoError(io.error);
  if (rs == VS_ERR_INVALID_ARGUMENT) {
    const std::string msg = last_error();
    if (msg.rfind("corrupt record stream", 0) == 0) throw CodecError(msg);
    throw InvalidArgument(msg);
  }
  check(rs, "run_rank");
  sink.finish();
  RankStats out;
  out.ligands_docked = st.ligands_docked;
  out.records_skipped = st.records_skipped;
  out.dock_errors = st.dock_errors;
  out.rows_written = st.rows_written;
  out.chunks_read = st.chunks_read;
  out.bytes_read = st.bytes_read;
  out.write_calls = st.write_calls;
  out.bytes_written = st.bytes_written;
  out.workers = st.workers;
  out.wall_seconds = st.wall_seconds;
  out.reader_busy_seconds = st.reader_busy_seconds;
  out.splitter_busy_seconds = st.splitter_busy_seconds;
  out.docker_busy_seconds = st.docker_busy_seconds;
  out.writer_busy_seconds = st.writer_busy_seconds;
  return out;
}

RankStats run_rank(const RankPlan &plan, const Pocket &pocket, const PipelineConfig &config) {
  FileSource source(plan.input_path);
  FileSink sink(plan.output_path);
  return run_rank(plan, source, sink, pocket, config);
}

void merge_outputs(const std::vector<std::string> &paths, const std::string &merged_path) {
  std::ofstream out(merged_path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open merged output '" + merged_path + "'");
  for (const std::string &path : paths) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("missing rank output '" + path + "'");
    out << in.rdbuf();
    if (in.bad() || !out) throw IoError("merge failed while copying '" + path + "'");
  }
  out.flush();
  if (!out) throw IoError("cannot finish merged output '" + merged_path + "'");
}

}  // namespace vscreen

// ------------------------------------------------------------ b200 extras
#include "vscreen/b200/prepare.hpp"

namespace vscreen::b200 {

static std::vector<Ligand> prep_many(const std::vector<std::string> &smiles, int mode) {
  std::vector<const char *> ptrs;
  for (const auto &s : smiles) ptrs.push_back(s.c_str());
  vs_ligand_set *set = nullptr;
  if (vs_prep_smiles_batch(static_cast<int32_t>(ptrs.size()), ptrs.data(), mode, 8, &set) != VS_OK)
    throw InvalidArgument("vs_prep_smiles_batch failed");
  vs_ligand_batch v{};
  const int32_t *st = nullptr;
  vs_ligand_set_view(set, &v, &st);
  std::vector<Ligand> out;
  std::string err;
  for (std::size_t i = 0; i < smiles.size(); ++i) {
    if (st[i] != 0) {
      err = vs_ligand_set_error(set, static_cast<int32_t>(i));
      break;
    }
    Ligand l;
    l.name = smiles[i];
    for (int a = v.atom_offset[i]; a < v.atom_offset[i + 1]; ++a) {
      Atom at;
      at.element = static_cast<Element>(v.element[a]);
      at.is_heavy = v.is_heavy[a] != 0;
      at.position = Eigen::Vector3d(v.xyz[3 * a], v.xyz[3 * a + 1], v.xyz[3 * a + 2]);
      l.atoms.push_back(at);
    }
    for (int k = v.bond_offset[i]; k < v.bond_offset[i + 1]; ++k)
      l.bonds.push_back({v.bond_a[k], v.bond_b[k], static_cast<BondOrder>(v.bond_order[k])});
    for (int t = v.torsion_offset[i]; t < v.torsion_offset[i + 1]; ++t)
      l.torsions.push_back(torsion_partition(l, v.torsion_bond[t]));
    out.push_back(std::move(l));
  }
  vs_ligand_set_free(set);
  if (!err.empty()) throw ParseError(err);
  return out;
}

Ligand prepare_smiles(const std::string &smiles, int mode) { return prep_many({smiles}, mode)[0]; }

void use_device(int device) {
  if (device < 0 || device >= kMaxDevices) throw InvalidArgument("use_device: device index out of range");
  tl_device = device;
}

int device_count() { return vs_device_count(); }

std::vector<Ligand> prepare_ligands(const std::vector<std::string> &smiles, bool quantize) {
  std::vector<Ligand> ligs = prep_many(smiles, 1);
  for (Ligand &l : ligs) {
    FlattenResult f = flatten(l, conformation_of(l), 20);
    l = with_conformation(std::move(l), f.conformation);
    if (quantize)
      for (Atom &a : l.atoms)
        for (int k = 0; k < 3; ++k) {
          volatile float narrowed = static_cast<float>(a.position[k]);
          a.position[k] = static_cast<double>(narrowed);
        }
  }
  return ligs;
}

}  // namespace vscreen::b200
