// Drop-in for search.hpp:17-79 (every declaration, exhaustive_dock included),
// plus the batch entry point this build adds.
// dock_and_score / dock_and_score_batch / flatten / local_search run on the
// B200 through libvsdock.so; results match the reference's (bit-exact up to
// the correctly rounded torsion sin/cos).
#pragma once

#include <span>
#include <vector>

#include "vscreen/dockengine/grid.hpp"
#include "vscreen/dockengine/pose.hpp"
#include "vscreen/molmodel/ligand.hpp"
#include "vscreen/molmodel/pocket.hpp"

namespace vscreen {

struct FlattenResult {
  Conformation conformation;
  std::vector<double> torsion_angles;
};

FlattenResult flatten(const Ligand &ligand, const Conformation &base, int max_sweeps = 20);
Eigen::Vector3d fibonacci_axis(int i, int k);
double fibonacci_rotation_angle(int i);
std::vector<Pose> initial_poses(const Pocket &pocket, const Ligand &ligand, const Conformation &base,
                                const std::vector<double> &flat_angles, int k, EvalCounter *counter = nullptr);
Pose local_search(const Pocket &pocket, const Ligand &ligand, Pose pose, const ScoringConfig &config,
                  EvalCounter *counter = nullptr);
std::vector<Pose> cluster_and_select(const std::vector<Pose> &poses, const Ligand &ligand, double threshold,
                                     std::size_t top);
DockResult dock_and_score(const Pocket &pocket, const Ligand &ligand, const ScoringConfig &config = {});
// search.hpp:74-79: brute-force test oracle (0.25 A lattice x 512 Fibonacci
// orientations, ties keep the earliest point then orientation); rigid
// ligands of <= 5 atoms, pockets <= 16 A per side, else InvalidArgument.
// Field values come from the B200 sampler; the scan order is the reference's.
Pose exhaustive_dock(const Pocket &pocket, const Ligand &ligand);

// B200 batch entry point (no reference counterpart; the reference docks one
// ligand per call from W threads, pipeline.cpp:206-244).  Ligands that the
// reference would reject (InvalidArgument) come back with a non-finite
// best_score and an empty best_pose; `errors` (optional) receives the message.
std::vector<DockResult> dock_and_score_batch(const Pocket &pocket, std::span<const Ligand> ligands,
                                             const ScoringConfig &config = {},
                                             std::vector<std::string> *errors = nullptr);

}  // namespace vscreen
