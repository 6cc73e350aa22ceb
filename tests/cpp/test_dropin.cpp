// C++ drop-in check: code written against the reference's API
// (proj/include/vscreen) runs unchanged on the B200 build (libvscreen_b200).
// Mirrors checks of test_dockengine.cpp / test_ligand_graph.cpp.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vscreen/b200/prepare.hpp"
#include "vscreen/dockengine/chem.hpp"
#include "vscreen/dockengine/grid.hpp"
#include "vscreen/dockengine/search.hpp"
#include "vscreen/error.hpp"

using namespace vscreen;

static int failures = 0;
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

  std::printf(failures == 0 ? "ALL OK\n" : "%d FAILURES\n", failures);
  return failures == 0 ? 0 : 1;
}
