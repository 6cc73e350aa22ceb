// Drop-in for grid.hpp:17-48.  On this build build_pocket, pocket_field_value
// and geo_score execute on the B200 (libvsdock.so sub-APIs).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "vscreen/geometry/transform.hpp"
#include "vscreen/molmodel/ligand.hpp"
#include "vscreen/molmodel/pocket.hpp"

namespace vscreen {

struct EvalCounter {
  std::uint64_t scoring_evals = 0;
};

inline constexpr double kClashValue = -10.0;
inline constexpr double kContactValue = 1.0;
inline constexpr double kClashDistance = 1.5;
inline constexpr double kContactDistance = 4.0;

Pocket build_pocket(const std::vector<ProteinAtom> &protein, const std::string &id, const Eigen::Vector3d &center,
                    double radius, double spacing);
double pocket_field_value(const Pocket &pocket, const Eigen::Vector3d &point);
double geo_score(const Pocket &pocket, const Ligand &ligand, const Conformation &conf, EvalCounter *counter = nullptr);

}  // namespace vscreen
