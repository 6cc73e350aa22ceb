// ============================================================================
// ORACLE/_REF WRAPPER — TEST INFRASTRUCTURE ONLY.
// ============================================================================
// C entry points over the reference's OWN sources, compiled unchanged from
// /root/reference/proj/src (see oracle/build_ref.sh) against the Eigen-subset
// restatement in third_party/eigen_subset.  The output library lives in
// oracle/_ref/ (git-ignored, shipped to the GPU box by gpurun).  Entry points
// mirror liboracle.so's vso_* so tests can compare the two line by line.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "vs_dock.h"
#include "vscreen/dockengine/chem.hpp"
#include "vscreen/dockengine/grid.hpp"
#include "vscreen/dockengine/pocket_io.hpp"
#include "vscreen/dockengine/search.hpp"
#include "vscreen/error.hpp"
#include "vscreen/geometry/embed.hpp"
#include "vscreen/geometry/hydrogens.hpp"
#include "vscreen/geometry/transform.hpp"
#include "vscreen/molmodel/binary_codec.hpp"
#include "vscreen/molmodel/smiles.hpp"
#include "vscreen/pipeline/pipeline.hpp"
#include "vscreen/workflow/workflow.hpp"

using namespace vscreen;

namespace {

Ligand ligand_from_batch(const vs_ligand_batch *b, int i) {
  Ligand l;
  const int a0 = b->atom_offset[i], a1 = b->atom_offset[i + 1];
  for (int a = a0; a < a1; ++a) {
    Atom at;
    at.element = static_cast<Element>(b->element[a]);
    at.position = Eigen::Vector3d(b->xyz[3 * a], b->xyz[3 * a + 1], b->xyz[3 * a + 2]);
    at.is_heavy = b->is_heavy[a] != 0;
    l.atoms.push_back(at);
  }
  for (int k = b->bond_offset[i]; k < b->bond_offset[i + 1]; ++k)
    l.bonds.push_back({b->bond_a[k], b->bond_b[k],
                       static_cast<BondOrder>(b->bond_order ? b->bond_order[k] : 1)});
  const std::size_t n = l.atoms.size();
  for (int t = b->torsion_offset[i]; t < b->torsion_offset[i + 1]; ++t) {
    TorsionalBond tb;
    tb.bond_index = b->torsion_bond[t];
    std::vector<uint8_t> in_right(n, 0);
    for (int r = b->right_offset[t]; r < b->right_offset[t + 1]; ++r) {
      tb.right_set.push_back(b->right_atoms[r]);
      if (b->right_atoms[r] < n) in_right[b->right_atoms[r]] = 1;
    }
    for (std::size_t a = 0; a < n; ++a)
      if (!in_right[a]) tb.left_set.push_back(static_cast<uint16_t>(a));
    l.torsions.push_back(std::move(tb));
  }
  return l;
}

Pocket pocket_from_desc(const vs_pocket_desc *d) {
  Pocket p;
  p.id = "desc";
  p.origin = Eigen::Vector3d(d->origin[0], d->origin[1], d->origin[2]);
  p.spacing = d->spacing;
  p.dims = {d->dims[0], d->dims[1], d->dims[2]};
  const std::size_t nv = static_cast<std::size_t>(d->dims[0]) * d->dims[1] * d->dims[2];
  p.values.assign(d->values, d->values + nv);
  for (int j = 0; j < d->n_protein; ++j)
    p.protein_atoms.push_back({static_cast<Element>(d->protein_element[j]),
                               Eigen::Vector3d(d->protein_xyz[3 * j], d->protein_xyz[3 * j + 1],
                                               d->protein_xyz[3 * j + 2])});
  return p;
}

Conformation conf_of(const double *xyz, int a0, int a1) {
  Conformation c(3, a1 - a0);
  for (int a = a0; a < a1; ++a)
    c.col(a - a0) = Eigen::Vector3d(xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]);
  return c;
}

void put_conf(const Conformation &c, double *xyz, int a0) {
  for (Eigen::Index a = 0; a < c.cols(); ++a) {
    const Eigen::Vector3d v = c.col(a);
    xyz[3 * (a0 + a)] = v.x();
    xyz[3 * (a0 + a) + 1] = v.y();
    xyz[3 * (a0 + a) + 2] = v.z();
  }
}

void put_pose(const Pose &p, vs_pose *o) {
  o->rotation[0] = p.transform.rotation.x();
  o->rotation[1] = p.transform.rotation.y();
  o->rotation[2] = p.transform.rotation.z();
  o->rotation[3] = p.transform.rotation.w();
  for (int a = 0; a < 3; ++a) o->translation[a] = p.transform.translation[a];
  o->geo_score = p.geo_score;
}

ScoringConfig to_cfg(const vs_scoring_config *c) {
  ScoringConfig s;
  s.restarts = c->restarts;
  s.rescored = c->rescored;
  s.rmsd_threshold = c->rmsd_threshold;
  s.step_translation = c->step_translation;
  s.step_rotation = c->step_rotation;
  s.step_torsion = c->step_torsion;
  s.min_translation = c->min_translation;
  s.max_iterations = c->max_iterations;
  s.flatten_max_sweeps = c->flatten_max_sweeps;
  return s;
}

int status_of(const std::exception &e) {
  const std::string w = e.what();
  if (w.find("empty conformation") != std::string::npos) return VS_LIG_EMPTY;
  if (w.find("degenerate torsion axis") != std::string::npos) return VS_LIG_DEGENERATE_AXIS;
  if (w.find("no heavy atoms") != std::string::npos) return VS_LIG_NO_HEAVY;
  return VS_LIG_BAD_TORSION;
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

thread_local std::string g_err;

}  // namespace

extern "C" {

const char *vsref_last_error(void) { return g_err.c_str(); }

void vsref_config_default(vs_scoring_config *c) {
  const ScoringConfig s;
  c->restarts = s.restarts;
  c->rescored = s.rescored;
  c->rmsd_threshold = s.rmsd_threshold;
  c->step_translation = s.step_translation;
  c->step_rotation = s.step_rotation;
  c->step_torsion = s.step_torsion;
  c->min_translation = s.min_translation;
  c->max_iterations = s.max_iterations;
  c->flatten_max_sweeps = s.flatten_max_sweeps;
}

// dock_and_score (search.cpp:238-276) per ligand on nthreads workers.
int vsref_dock_batch(const vs_pocket_desc *pd, const vs_ligand_batch *b, const vs_scoring_config *cfg,
                     int nthreads, vs_dock_result *res, double *best_angles, double *best_conf) {
  const Pocket p = pocket_from_desc(pd);
  const ScoringConfig sc = to_cfg(cfg);
  if (sc.restarts < 1 || sc.rescored < 1 || !(sc.rmsd_threshold > 0.0)) return VS_ERR_INVALID_ARGUMENT;
  parallel_for(b->n_ligands, nthreads, [&](int i) {
    vs_dock_result &r = res[i];
    std::memset(&r, 0, sizeof(r));
    try {
      const Ligand lig = ligand_from_batch(b, i);
      const DockResult d = dock_and_score(p, lig, sc);
      r.status = std::isfinite(d.best_score) ? VS_LIG_OK : VS_LIG_NONFINITE;
      r.best_score = d.best_score;
      r.best_geo_score = d.best_pose.geo_score;
      r.rotation[0] = d.best_pose.transform.rotation.x();
      r.rotation[1] = d.best_pose.transform.rotation.y();
      r.rotation[2] = d.best_pose.transform.rotation.z();
      r.rotation[3] = d.best_pose.transform.rotation.w();
      for (int a = 0; a < 3; ++a) r.translation[a] = d.best_pose.transform.translation[a];
      r.poses_evaluated = d.poses_evaluated;
      r.scoring_evals = d.scoring_evals;
      if (best_angles)
        for (std::size_t t = 0; t < d.best_pose.torsion_angles.size(); ++t)
          best_angles[b->torsion_offset[i] + t] = d.best_pose.torsion_angles[t];
      if (best_conf) put_conf(d.best_pose.conformation, best_conf, b->atom_offset[i]);
    } catch (const std::exception &e) {
      r.status = status_of(e);
    }
  });
  return VS_OK;
}

int vsref_field_values(const vs_pocket_desc *pd, int64_t n, const double *xyz, double *out) {
  const Pocket p = pocket_from_desc(pd);
  for (int64_t i = 0; i < n; ++i)
    out[i] = pocket_field_value(p, Eigen::Vector3d(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]));
  return VS_OK;
}

int vsref_geo_score(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *conf,
                    double *out, uint64_t *evals) {
  const Pocket p = pocket_from_desc(pd);
  for (int i = 0; i < b->n_ligands; ++i) {
    EvalCounter c;
    out[i] = geo_score(p, ligand_from_batch(b, i), conf_of(conf, b->atom_offset[i], b->atom_offset[i + 1]), &c);
    if (evals) evals[i] = c.scoring_evals;
  }
  return VS_OK;
}

int vsref_chem_score(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *conf, double *out) {
  const Pocket p = pocket_from_desc(pd);
  for (int i = 0; i < b->n_ligands; ++i)
    out[i] = chem_score(p, ligand_from_batch(b, i), conf_of(conf, b->atom_offset[i], b->atom_offset[i + 1]));
  return VS_OK;
}

int vsref_flatten(const vs_ligand_batch *b, int max_sweeps, double *conf_out, double *angles_out,
                  int32_t *status, int nthreads) {
  parallel_for(b->n_ligands, nthreads, [&](int i) {
    try {
      const Ligand lig = ligand_from_batch(b, i);
      const FlattenResult f = flatten(lig, conformation_of(lig), max_sweeps);
      put_conf(f.conformation, conf_out, b->atom_offset[i]);
      for (std::size_t t = 0; t < f.torsion_angles.size(); ++t) angles_out[b->torsion_offset[i] + t] = f.torsion_angles[t];
      if (status) status[i] = VS_LIG_OK;
    } catch (const std::exception &e) {
      if (status) status[i] = status_of(e);
    }
  });
  return VS_OK;
}

int vsref_local_search(const vs_pocket_desc *pd, const vs_ligand_batch *b, const vs_scoring_config *cfg,
                       vs_pose *poses, double *angles, double *conf, uint64_t *evals, int32_t *status) {
  const Pocket p = pocket_from_desc(pd);
  const ScoringConfig sc = to_cfg(cfg);
  for (int i = 0; i < b->n_ligands; ++i) {
    try {
      const Ligand lig = ligand_from_batch(b, i);
      const int a0 = b->atom_offset[i], a1 = b->atom_offset[i + 1];
      const int t0 = b->torsion_offset[i], t1 = b->torsion_offset[i + 1];
      Pose in;
      in.transform.rotation = Eigen::Quaterniond(poses[i].rotation[3], poses[i].rotation[0],
                                                 poses[i].rotation[1], poses[i].rotation[2]);
      in.transform.translation =
          Eigen::Vector3d(poses[i].translation[0], poses[i].translation[1], poses[i].translation[2]);
      in.geo_score = poses[i].geo_score;
      in.torsion_angles.assign(angles + t0, angles + t1);
      in.conformation = conf_of(conf, a0, a1);
      EvalCounter c;
      const Pose o = local_search(p, lig, in, sc, &c);
      put_pose(o, &poses[i]);
      for (int t = t0; t < t1; ++t) angles[t] = o.torsion_angles[static_cast<std::size_t>(t - t0)];
      put_conf(o.conformation, conf, a0);
      if (evals) evals[i] = c.scoring_evals;
      if (status) status[i] = VS_LIG_OK;
    } catch (const std::exception &e) {
      if (status) status[i] = status_of(e);
    }
  }
  return VS_OK;
}

int vsref_initial_poses(const vs_pocket_desc *pd, const vs_ligand_batch *b, const double *flat_angles,
                        int k, vs_pose *out, double *confs, uint64_t *evals) {
  try {
    const Pocket p = pocket_from_desc(pd);
    const Ligand lig = ligand_from_batch(b, 0);
    std::vector<double> fa(flat_angles, flat_angles + lig.torsions.size());
    EvalCounter c;
    const auto poses = initial_poses(p, lig, conformation_of(lig), fa, k, &c);
    const int na = static_cast<int>(lig.atoms.size());
    for (int i = 0; i < k; ++i) {
      put_pose(poses[i], &out[i]);
      put_conf(poses[i].conformation, confs, i * na);
    }
    if (evals) *evals = c.scoring_evals;
    return VS_OK;
  } catch (const InvalidArgument &e) {
    g_err = e.what();
    return VS_ERR_INVALID_ARGUMENT;
  }
}

int vsref_cluster_select(const vs_ligand_batch *b, int n, const double *geo, const double *confs,
                         double threshold, int top, int32_t *order_out) {
  try {
    const Ligand lig = ligand_from_batch(b, 0);
    const int na = static_cast<int>(lig.atoms.size());
    std::vector<Pose> poses(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      poses[i].geo_score = geo[i];
      poses[i].conformation = conf_of(confs, i * na, (i + 1) * na);
      // Tag each pose through its translation so the output order can be
      // recovered from the returned copies.
      poses[i].transform.translation = Eigen::Vector3d(i, 0, 0);
    }
    const auto out = cluster_and_select(poses, lig, threshold, static_cast<std::size_t>(top));
    for (std::size_t i = 0; i < out.size(); ++i)
      order_out[i] = static_cast<int32_t>(out[i].transform.translation.x());
    return static_cast<int>(out.size());
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

int vsref_exhaustive_dock(const vs_pocket_desc *pd, const vs_ligand_batch *b, vs_pose *out, double *conf_out) {
  try {
    const Pose o = exhaustive_dock(pocket_from_desc(pd), ligand_from_batch(b, 0));
    put_pose(o, out);
    put_conf(o.conformation, conf_out, 0);
    return VS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return VS_ERR_INVALID_ARGUMENT;
  }
}

int vsref_fibonacci(int k, double *axes, double *angles) {
  for (int i = 0; i < k; ++i) {
    const Eigen::Vector3d a = fibonacci_axis(i, k);
    axes[3 * i] = a.x();
    axes[3 * i + 1] = a.y();
    axes[3 * i + 2] = a.z();
    angles[i] = fibonacci_rotation_angle(i);
  }
  return VS_OK;
}

double vsref_internal_distance_sum(int n, const double *xyz) { return internal_distance_sum(conf_of(xyz, 0, n)); }

// ---- ligand preparation (the input side; prep.cpp:37-44, test helpers) ----
// mode 0: prepare_ligand (prep.cpp:37-44): parse, add H, embed, detect
//         torsions, flatten.
// mode 1: test_dockengine.cpp:29-33 prepared(): torsions on the H-added
//         graph, embedded coordinates, no flatten.
// mode 2: detect_torsions(parse_smiles(s)) only (heavy-atom graph, zero
//         coordinates).
// quantize: quantize_to_wire (binary_codec.cpp:254-264) afterwards.
void *vsref_prepare(const char *smiles, int mode, int quantize) {
  try {
    Ligand lig;
    if (mode == 0) {
      lig = add_hydrogens(parse_smiles(smiles));
      const Conformation embedded = embed_3d(lig);
      lig = with_conformation(std::move(lig), embedded);
      lig = detect_torsions(std::move(lig));
      FlattenResult flat = flatten(lig, conformation_of(lig));
      lig = with_conformation(std::move(lig), flat.conformation);
    } else if (mode == 1) {
      lig = detect_torsions(add_hydrogens(parse_smiles(smiles)));
      const Conformation conf = embed_3d(lig);
      lig = with_conformation(std::move(lig), conf);
    } else {
      lig = detect_torsions(parse_smiles(smiles));
    }
    if (quantize) lig = quantize_to_wire(std::move(lig));
    return new Ligand(std::move(lig));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// Decode one .xslb record (binary_codec.cpp:165-222) into a handle.
void *vsref_decode_record(const uint8_t *bytes, int64_t n, int64_t offset, int64_t *next) {
  try {
    auto [lig, end] = decode_record(std::span<const uint8_t>(bytes, static_cast<std::size_t>(n)),
                                    static_cast<std::size_t>(offset));
    if (next) *next = static_cast<int64_t>(end);
    return new Ligand(std::move(lig));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// Encode a handle as one record; returns the byte count (copies when
// out != NULL and cap suffices).
int64_t vsref_encode_record(const void *h, uint8_t *out, int64_t cap) {
  const auto rec = encode_record(*static_cast<const Ligand *>(h));
  if (out && static_cast<int64_t>(rec.size()) <= cap) std::memcpy(out, rec.data(), rec.size());
  return static_cast<int64_t>(rec.size());
}

void vsref_ligand_free(void *h) { delete static_cast<Ligand *>(h); }

// counts[0..3] = atoms, bonds, torsions, total right-set size
void vsref_ligand_counts(const void *h, int32_t *counts) {
  const Ligand &l = *static_cast<const Ligand *>(h);
  counts[0] = static_cast<int32_t>(l.atoms.size());
  counts[1] = static_cast<int32_t>(l.bonds.size());
  counts[2] = static_cast<int32_t>(l.torsions.size());
  int32_t r = 0;
  for (const auto &t : l.torsions) r += static_cast<int32_t>(t.right_set.size());
  counts[3] = r;
}

const char *vsref_ligand_name(const void *h) { return static_cast<const Ligand *>(h)->name.c_str(); }

void vsref_ligand_export(const void *h, double *xyz, uint8_t *elem, uint8_t *heavy, uint16_t *ba,
                         uint16_t *bb, uint8_t *bo, uint16_t *tb, int32_t *roff, uint16_t *ratoms) {
  const Ligand &l = *static_cast<const Ligand *>(h);
  for (std::size_t i = 0; i < l.atoms.size(); ++i) {
    xyz[3 * i] = l.atoms[i].position.x();
    xyz[3 * i + 1] = l.atoms[i].position.y();
    xyz[3 * i + 2] = l.atoms[i].position.z();
    elem[i] = static_cast<uint8_t>(l.atoms[i].element);
    heavy[i] = l.atoms[i].is_heavy ? 1 : 0;
  }
  for (std::size_t i = 0; i < l.bonds.size(); ++i) {
    ba[i] = l.bonds[i].a;
    bb[i] = l.bonds[i].b;
    bo[i] = static_cast<uint8_t>(l.bonds[i].order);
  }
  int32_t off = 0;
  for (std::size_t t = 0; t < l.torsions.size(); ++t) {
    tb[t] = l.torsions[t].bond_index;
    roff[t] = off;
    for (uint16_t a : l.torsions[t].right_set) ratoms[off++] = a;
  }
  roff[l.torsions.size()] = off;
}

// build_pocket (grid.cpp:15-57): writes dims/origin and, when values !=
// NULL, the grid.  Returns VS_OK or VS_ERR_INVALID_ARGUMENT.
int vsref_build_pocket(int32_t n, const uint8_t *elem, const double *xyz, const double center[3],
                       double radius, double spacing, int32_t dims[3], double origin[3], double *values) {
  try {
    std::vector<ProteinAtom> prot;
    for (int j = 0; j < n; ++j)
      prot.push_back({static_cast<Element>(elem[j]), Eigen::Vector3d(xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2])});
    const Pocket p = build_pocket(prot, "built", Eigen::Vector3d(center[0], center[1], center[2]), radius, spacing);
    for (int a = 0; a < 3; ++a) {
      dims[a] = p.dims[a];
      origin[a] = p.origin[a];
    }
    if (values) std::memcpy(values, p.values.data(), p.values.size() * sizeof(double));
    return VS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return VS_ERR_INVALID_ARGUMENT;
  }
}

// run_rank (pipeline.cpp:297-398) over an in-memory .xslb image: the
// reference's reader / splitter / `workers` docker threads / writer.  The
// rank's output text goes to *out (malloc'ed, caller frees with
// vsref_free); counters: ligands_docked, records_skipped, dock_errors,
// rows_written.  Returns VS_OK or VS_ERR_INVALID_ARGUMENT (message in
// vsref_last_error).
int vsref_run_rank(const uint8_t *bytes, int64_t size, uint64_t slab_start, uint64_t slab_stop,
                   const vs_pocket_desc *pd, const vs_scoring_config *cfg, int workers, int64_t chunk_bytes,
                   char **out, int64_t *out_len, uint64_t counters[4]) {
  try {
    const Pocket pocket = pocket_from_desc(pd);
    PipelineConfig pc;
    pc.scoring = to_cfg(cfg);
    pc.workers = {WorkerClass{WorkerKind::Fast, workers, 1.0}};
    pc.chunk_bytes = static_cast<std::size_t>(chunk_bytes);
    MemorySource src(std::vector<std::uint8_t>(bytes, bytes + size));
    StringSink sink;
    RankPlan plan;
    plan.slab_start = slab_start;
    plan.slab_stop = slab_stop;
    const RankStats st = run_rank(plan, src, sink, pocket, pc);
    *out_len = static_cast<int64_t>(sink.data().size());
    *out = static_cast<char *>(std::malloc(sink.data().size() + 1));
    std::memcpy(*out, sink.data().data(), sink.data().size());
    counters[0] = st.ligands_docked;
    counters[1] = st.records_skipped;
    counters[2] = st.dock_errors;
    counters[3] = st.rows_written;
    return VS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return VS_ERR_INVALID_ARGUMENT;
  }
}

// cmd_merge (merge.cpp:81-147) of a campaign directory: writes
// <out_dir>/ranking.tsv; returns the row count, or -1 (message in
// vsref_last_error).
int64_t vsref_cmd_merge(const char *out_dir) {
  try {
    return static_cast<int64_t>(cmd_merge(out_dir).rows);
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

// format_rank_stats (pipeline.cpp:430) of a RankStats with the four counters.
int64_t vsref_format_rank_stats(const uint64_t counters[4], char *out, int64_t cap) {
  RankStats st;
  st.ligands_docked = counters[0];
  st.records_skipped = counters[1];
  st.dock_errors = counters[2];
  st.rows_written = counters[3];
  const std::string t = format_rank_stats(st);
  if (static_cast<int64_t>(t.size()) > cap) return -static_cast<int64_t>(t.size());
  std::memcpy(out, t.data(), t.size());
  return static_cast<int64_t>(t.size());
}

void vsref_free(void *p) { std::free(p); }

}  // extern "C"
