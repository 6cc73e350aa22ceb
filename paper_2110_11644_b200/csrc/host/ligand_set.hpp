// Host container behind the opaque vs_ligand_set of vs_prep.h / vs_codec.h:
// a SoA ligand batch (vs_ligand_batch view) plus per-entry status, error
// text and name.  Filled by SMILES preparation (prep.cpp) and by the GPU
// record decoder (cuda/codec.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

struct vs_ligand_set {
  std::vector<int32_t> status;
  std::vector<std::string> errors;
  std::vector<std::string> names;
  std::vector<int32_t> atom_off, bond_off, tors_off, right_off;
  std::vector<double> xyz;
  std::vector<uint8_t> elem, heavy, border;
  std::vector<uint16_t> ba, bb, tbond, ratoms;
};
