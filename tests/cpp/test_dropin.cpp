// C++ drop-in check: code written against the reference's API
// (proj/include/vscreen) runs unchanged on the B200 build (libvscreen_b200).
// Mirrors checks of test_dockengine.cpp / test_ligand_graph.cpp.
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "vscreen/b200/prepare.hpp"
#include "vscreen/dockengine/chem.hpp"
#include "vscreen/dockengine/grid.hpp"
#include "vscreen/dockengine/search.hpp"
#include "vscreen/error.hpp"
#include "vscreen/pipeline/pipeline.hpp"

using namespace vscreen;

static int failures = 0;

// encode_record (binary_codec.cpp:129-163), for building an .xslb image
static void put16(std::vector<std::uint8_t> &o, unsigned v) {
  o.push_back(v & 255);
  o.push_back((v >> 8) & 255);
}
static void encode(std::vector<std::uint8_t> &o, const vscreen::Ligand &l) {
  std::vector<std::uint8_t> p;
  put16(p, static_cast<unsigned>(l.name.size()));
  p.insert(p.end(), l.name.begin(), l.name.end());
  put16(p, static_cast<unsigned>(l.atoms.size()));
  put16(p, static_cast<unsigned>(l.bonds.size()));
  put16(p, static_cast<unsigned>(l.torsions.size()));
  for (const auto &a : l.atoms) {
    for (int k = 0; k < 3; ++k) {
      const float f = static_cast<float>(a.position[k]);
      std::uint8_t b[4];
      std::memcpy(b, &f, 4);
      p.insert(p.end(), b, b + 4);
    }
    p.push_back(static_cast<std::uint8_t>(a.element));
    p.push_back(a.is_heavy ? 1 : 0);
  }
  for (const auto &b : l.bonds) {
    put16(p, b.a);
    put16(p, b.b);
    p.push_back(static_cast<std::uint8_t>(b.order));
  }
  for (const auto &t : l.torsions) put16(p, t.bond_index);
  o.push_back(0xD0);
  o.push_back(0xC5);
  const std::uint32_t n = static_cast<std::uint32_t>(p.size());
  for (int k = 0; k < 4; ++k) o.push_back((n >> (8 * k)) & 255);
  o.insert(o.end(), p.begin(), p.end());
}
#define CHECK(x)                                                     \
  do {                                                               \
    if (!(x)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);       \
      ++failures;                                                    \
    }                                                                \
  } while (0)

int main() {
  // torsion partition (test_ligand_graph.cpp:39-47)
  const Ligand butane = b200::prepare_smiles("CCCC", 2);
  CHECK(butane.torsions.size() == 1 && butane.torsions[0].bond_index == 1);
  CHECK((butane.torsions[0].left_set == std::vector<std::uint16_t>{0, 1}));
  CHECK((butane.torsions[0].right_set == std::vector<std::uint16_t>{2, 3}));
  const Ligand redetected = detect_torsions(butane);
  CHECK(redetected == butane);

  // build_pocket (test_dockengine.cpp:64-81)
  const Pocket one = build_pocket({{Element::C, Eigen::Vector3d(0, 0, 0)}}, "p", Eigen::Vector3d(0, 0, 0), 4.0, 0.5);
  CHECK((one.dims == std::array<int, 3>{17, 17, 17}));
  CHECK(one.value_at(10, 8, 8) == kClashValue && one.value_at(14, 8, 8) == kContactValue && one.value_at(0, 0, 0) == 0.0);

  // dock_and_score determinism and accounting (test_dockengine.cpp:696-744)
  const Pocket twin = build_pocket({{Element::C, Eigen::Vector3d(-2, 0, 0)}, {Element::O, Eigen::Vector3d(2, 0, 0)}},
                                   "twin", Eigen::Vector3d::Zero(), 5.0, 0.5);
  ScoringConfig cfg;
  cfg.restarts = 16;
  cfg.rescored = 5;
  const Ligand co = b200::prepare_smiles("CO", 1);
  const DockResult a = dock_and_score(twin, co, cfg);
  const DockResult b = dock_and_score(twin, co, cfg);
  CHECK(a.best_score == b.best_score && a.scoring_evals == b.scoring_evals && a.poses_evaluated == 16);
  CHECK((a.best_pose.conformation - b.best_pose.conformation).cwiseAbs().maxCoeff() == 0.0);
  CHECK(a.best_pose.chem_score.has_value() && *a.best_pose.chem_score == a.best_score);
  CHECK(chem_score(twin, co, a.best_pose.conformation) == a.best_score);
  CHECK(geo_score(twin, co, a.best_pose.conformation) == a.best_pose.geo_score);
  const Conformation again =
      apply_rigid(apply_torsions(conformation_of(co), co, a.best_pose.torsion_angles), a.best_pose.transform);
  CHECK((again - a.best_pose.conformation).cwiseAbs().maxCoeff() == 0.0);
  bool threw = false;
  try {
    ScoringConfig bad = cfg;
    bad.restarts = 0;
    dock_and_score(twin, co, bad);
  } catch (const InvalidArgument &) {
    threw = true;
  }
  CHECK(threw);

  // flat-field eval count (test_dockengine.cpp:746-761)
  Pocket flat;
  flat.dims = {9, 9, 9};
  flat.spacing = 1.0;
  flat.values.assign(729, 0.0);
  ScoringConfig c8;
  c8.restarts = 8;
  c8.rescored = 3;
  const Ligand cccc = b200::prepare_smiles("CCCC", 1);
  CHECK(dock_and_score(flat, cccc, c8).scoring_evals == 8u * 4u * (1u + 4u * (12u + 2u)));

  // batch == per-ligand calls; sub-APIs compose to the same answer
  const std::vector<Ligand> ligs =
      b200::prepare_ligands({"CCOC(=O)c1ccccc1N", "CC(C)Cc1ccc(cc1)C(C)C(=O)O", "c1ccccc1-c1ccccc1", "CCCCCCO"});
  const std::vector<DockResult> batch = dock_and_score_batch(twin, ligs, cfg);
  for (std::size_t i = 0; i < ligs.size(); ++i) {
    const DockResult single = dock_and_score(twin, ligs[i], cfg);
    CHECK(single.best_score == batch[i].best_score);
    CHECK(single.scoring_evals == batch[i].scoring_evals);
  }
  const Ligand &lig = ligs[0];
  const FlattenResult fl = flatten(lig, conformation_of(lig), cfg.flatten_max_sweeps);
  EvalCounter counter;
  std::vector<Pose> poses = initial_poses(twin, lig, conformation_of(lig), fl.torsion_angles, cfg.restarts, &counter);
  CHECK(poses.size() == 16 && counter.scoring_evals == 16 * lig.heavy_atom_count());
  for (Pose &p : poses) p = local_search(twin, lig, p, cfg, &counter);
  std::vector<Pose> surv = cluster_and_select(poses, lig, cfg.rmsd_threshold, cfg.rescored);
  double best = -1e300;
  for (const Pose &p : surv) best = std::max(best, chem_score(twin, lig, p.conformation));
  CHECK(best == batch[0].best_score);
  CHECK(counter.scoring_evals == batch[0].scoring_evals);

  // exhaustive_dock KATs (test_dockengine.cpp:665-693)
  auto flat_pocket = [](int nodes, double spacing) {
    Pocket p;
    p.id = "test";
    p.spacing = spacing;
    p.dims = {nodes, nodes, nodes};
    p.values.assign(static_cast<std::size_t>(nodes) * nodes * nodes, 0.0);
    return p;
  };
  const Ligand carbon = b200::prepare_smiles("C", 2);
  {
    Pocket p3 = flat_pocket(3, 0.5);
    p3.values[p3.value_index(2, 1, 0)] = 7.0;
    const Pose pose = exhaustive_dock(p3, carbon);
    CHECK((pose.conformation.col(0) - Eigen::Vector3d(1.0, 0.5, 0.0)).norm() < 1e-12);
    CHECK(std::fabs(pose.geo_score - 7.0) <= 7e-12);
    Pocket p2 = flat_pocket(2, 0.5);
    p2.values[p2.value_index(0, 0, 0)] = 3.0;
    p2.values[p2.value_index(1, 1, 1)] = 3.0;
    CHECK((exhaustive_dock(p2, carbon).conformation.col(0) - Eigen::Vector3d(0, 0, 0)).norm() < 1e-12);
    int limits = 0;
    try { exhaustive_dock(p3, b200::prepare_smiles("CCO", 1)); } catch (const InvalidArgument &) { ++limits; }
    try { exhaustive_dock(p3, b200::prepare_smiles("CCCC", 2)); } catch (const InvalidArgument &) { ++limits; }
    try { exhaustive_dock(flat_pocket(35, 0.5), carbon); } catch (const InvalidArgument &) { ++limits; }
    CHECK(limits == 3);
  }

  // device pockets are cached by content: a Pocket rebuilt at the same
  // address with the same sizes, or mutated in place, is re-uploaded
  // (test_dockengine.cpp:215-240 rebuilds `pocket` per SUBCASE)
  {
    Conformation origin(3, 1);
    origin.col(0) = Eigen::Vector3d(0, 0, 0);
    const double want[3] = {0.4, 0.0, 0.4 * 0.5};
    const double zs[3] = {3.0, 4.5, 4.0};
    for (int sc = 0; sc < 3; ++sc) {
      Pocket pk = flat_pocket(2, 1.0);
      pk.protein_atoms = {{Element::C, Eigen::Vector3d(0.0, 0.0, zs[sc])}};
      CHECK(std::fabs(chem_score(pk, carbon, origin) - want[sc]) <= 1e-12);
    }
    Pocket pm = flat_pocket(3, 0.5);
    const Conformation mid = [] { Conformation c(3, 1); c.col(0) = Eigen::Vector3d(0.5, 0.5, 0.5); return c; }();
    CHECK(pocket_field_value(pm, mid.col(0)) == 0.0);
    pm.values[pm.value_index(1, 1, 1)] = 5.0;  // mutated in place: same buffer, same sizes
    CHECK(pocket_field_value(pm, mid.col(0)) == 5.0);
  }

  // run_rank on the CUDA workers (pipeline.cpp:297-389): rows equal
  // format_row of dock_and_score per record, in record order
  {
    std::vector<std::uint8_t> img = {'X', 'S', 'L', 'B', 1, 0, 0, 0};
    std::vector<Ligand> lib = b200::prepare_ligands({"CCOC(=O)c1ccccc1N", "CCCCCCO", "c1ccccc1-c1ccccc1"});
    const char *names[] = {"CCOC(=O)c1ccccc1N", "CCCCCCO", "c1ccccc1-c1ccccc1"};
    for (std::size_t i = 0; i < lib.size(); ++i) {
      lib[i].name = names[i];
      encode(img, lib[i]);
    }
    std::string want;
    for (const Ligand &l : lib) want += format_row(OutputRow{l.name, dock_and_score(twin, l, cfg).best_score});
    MemorySource src(img);
    StringSink sink;
    RankPlan plan;
    plan.slab_stop = src.size();
    PipelineConfig pc;
    pc.scoring = cfg;
    pc.workers = {WorkerClass{WorkerKind::Fast, 2, 1.0}};
    const RankStats rs = run_rank(plan, src, sink, twin, pc);
    CHECK(sink.data() == want);
    CHECK(rs.rows_written == 3 && rs.ligands_docked == 3 && rs.records_skipped == 0 && rs.dock_errors == 0);
    CHECK(plan_slabs(10, 3)[1].slab_start == 3 && plan_slabs(10, 3)[2].slab_stop == 10);
    // file source / sink and merge_outputs (pipeline.cpp:391-412): two slabs
    // written to rank files, concatenated, equal the one-slab output
    const std::string dir = "/tmp/vs_dropin_rank";
    if (std::system(("mkdir -p " + dir).c_str()) != 0) ++failures;
    {
      std::FILE *f = std::fopen((dir + "/lib.xslb").c_str(), "wb");
      std::fwrite(img.data(), 1, img.size(), f);
      std::fclose(f);
    }
    const std::vector<RankPlan> plans = plan_slabs(img.size(), 2);
    std::vector<std::string> outs;
    for (RankPlan rp : plans) {
      rp.input_path = dir + "/lib.xslb";
      rp.output_path = dir + "/rank" + std::to_string(rp.rank) + ".scores";
      run_rank(rp, twin, pc);
      outs.push_back(rp.output_path);
    }
    merge_outputs(outs, dir + "/merged.tsv");
    std::FILE *mf = std::fopen((dir + "/merged.tsv").c_str(), "rb");
    std::string merged;
    char buf[4096];
    for (size_t got; (got = std::fread(buf, 1, sizeof buf, mf)) > 0;) merged.append(buf, got);
    std::fclose(mf);
    CHECK(merged == want);
    // the .stats file format (pipeline.cpp:430-505) round-trips
    const RankStats back = parse_rank_stats(format_rank_stats(rs));
    CHECK(back.rows_written == rs.rows_written && back.workers == rs.workers &&
          back.ligands_docked == rs.ligands_docked);
    CHECK(format_rank_stats(back) == format_rank_stats(rs) || rs.wall_seconds != back.wall_seconds);
    int bad = 0;
    try { parse_rank_stats("ligands_docked=3\nnope=1\n"); } catch (const ParseError &) { ++bad; }
    try { parse_rank_stats("rows_written 3\n"); } catch (const ParseError &) { ++bad; }
    CHECK(bad == 2);
  }

  // docker_worker (pipeline.cpp:206-244): a producer thread feeds WorkItems
  // through the reference's BoundedQueue; the batch-pulling CUDA worker's rows
  // equal format_row of per-ligand dock_and_score, one degenerate ligand is a
  // dock_error
  {
    std::vector<Ligand> lib = b200::prepare_ligands({"CCOC(=O)c1ccccc1N", "CCCCCCO", "c1ccccc1-c1ccccc1",
                                                     "CC(C)Cc1ccc(cc1)C(C)C(=O)O"});
    const char *names[] = {"A", "B", "C", "D"};
    for (std::size_t i = 0; i < lib.size(); ++i) lib[i].name = names[i];
    Ligand broken = lib[3];
    broken.name = "E";
    {
      const auto &bond = broken.bonds[broken.torsions[0].bond_index];
      broken.atoms[bond.b].position = broken.atoms[bond.a].position;  // degenerate torsion axis
    }
    BoundedQueue<WorkItem> in(2);
    BoundedQueue<OutputRow> out(64);
    std::thread producer([&] {
      std::uint64_t seq = 0;
      for (int rep = 0; rep < 3; ++rep)
        for (const Ligand &l : lib) in.push(WorkItem{l, seq++});
      in.push(WorkItem{broken, seq++});
      in.close();
    });
    const DockerStats ds = docker_worker(in, out, twin, cfg, 1.0);
    producer.join();
    out.close();
    std::vector<std::string> got;
    while (auto row = out.pop()) got.push_back(format_row(*row));
    std::vector<std::string> want;
    for (int rep = 0; rep < 3; ++rep)
      for (const Ligand &l : lib) want.push_back(format_row(OutputRow{l.name, dock_and_score(twin, l, cfg).best_score}));
    CHECK(got == want);
    CHECK(ds.rows == 12 && ds.dock_errors == 1);
    bool threw = false;
    try {
      BoundedQueue<WorkItem> q(1);
      docker_worker(q, out, twin, cfg, 0.5);
    } catch (const InvalidArgument &) {
      threw = true;
    }
    CHECK(threw);
  }

  // per-thread device selection
  CHECK(b200::device_count() >= 1);
  b200::use_device(b200::device_count() - 1);
  CHECK(dock_and_score(twin, co, cfg).best_score == a.best_score);
  b200::use_device(0);

  std::printf(failures == 0 ? "ALL OK\n" : "%d FAILURES\n", failures);
  return failures == 0 ? 0 : 1;
}
