// Drop-in for chem.hpp:14-26 (chem_score runs on the B200).
#pragma once

#include "vscreen/geometry/transform.hpp"
#include "vscreen/molmodel/ligand.hpp"
#include "vscreen/molmodel/pocket.hpp"

namespace vscreen {

double chem_score(const Pocket &pocket, const Ligand &ligand, const Conformation &conf);
double chem_pair_weight(ChemClass a, ChemClass b);

}  // namespace vscreen
