// B200 build extras (no reference counterpart): SMILES -> prepared Ligand
// through the native input side (include/vs_prep.h) and the GPU flatten,
// i.e. the reference's prepare_ligand (prep.cpp:37-44) with an optional f32
// wire quantisation (binary_codec.cpp:254-264).
#pragma once

#include <string>
#include <vector>

#include "vscreen/molmodel/ligand.hpp"

namespace vscreen::b200 {

// mode 1: hydrogens + embedding + torsions (unflattened); 2: heavy graph +
// torsions, zero coordinates; 3: heavy graph embedded.  Throws ParseError.
Ligand prepare_smiles(const std::string &smiles, int mode = 1);

// prepare_ligand: mode 1 + GPU flatten (+ quantise_to_wire when quantize).
std::vector<Ligand> prepare_ligands(const std::vector<std::string> &smiles, bool quantize = true);

// Device selection for the reference-API calls made by THIS thread (the
// reference's W docker threads can each pin one GPU, pipeline.cpp:343-363).
// Default: $VS_DEVICE, else 0.  One vs_context (stream) per device.
void use_device(int device);
int device_count();

}  // namespace vscreen::b200
