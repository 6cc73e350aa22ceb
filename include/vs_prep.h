/*
 * vs_prep.h — input side of the dock path (libvsdock.so, host code).
 *
 * Ligand preparation the reference performs before dock_and_score
 * (prep.cpp:37-44 prepare_ligand = parse_smiles -> add_hydrogens ->
 * embed_3d -> detect_torsions -> flatten), split so that the only compute-
 * heavy step, flatten, runs on the GPU (vs_flatten_batch in vs_dock.h):
 *
 *   mode 1: parse_smiles (smiles.cpp:37-211) + add_hydrogens
 *           (hydrogens.cpp:33-72) + embed_3d (embed.cpp:82-419) +
 *           detect_torsions (ligand.cpp:126-139) -- coordinates unflattened;
 *   mode 2: detect_torsions(parse_smiles(s)) -- heavy-atom graph, zero
 *           coordinates (no hydrogens);
 *   mode 3: mode 2 plus embed_3d of the heavy-atom graph (the fixtures of
 *           the reference's tests, e.g. test_dockengine.cpp:301-313).
 *
 * Plus the seeded synthetic drug-like SMILES generator used by the bench
 * (~30 heavy atoms, ~6 rotatable bonds, reference
 * SMILES subset).
 */
#ifndef VS_PREP_H
#define VS_PREP_H

#include "vs_dock.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vs_ligand_set vs_ligand_set;

/* Prepare n SMILES on nthreads host threads.  Always returns a set (unless
 * out of memory); entries that fail to parse/prepare have status != 0 and
 * zero atoms, and their message is available from vs_ligand_set_error. */
vs_status vs_prep_smiles_batch(int32_t n, const char *const *smiles, int32_t mode, int32_t nthreads,
                               vs_ligand_set **out);
/* Borrowed SoA view of the set (valid until vs_ligand_set_free). */
vs_status vs_ligand_set_view(const vs_ligand_set *set, vs_ligand_batch *view, const int32_t **status);
const char *vs_ligand_set_error(const vs_ligand_set *set, int32_t i);
/* Name of entry i (the SMILES for prepared sets, the record name for
 * decoded ones: the string the reference writes as the output row key). */
const char *vs_ligand_set_name(const vs_ligand_set *set, int32_t i);
void vs_ligand_set_free(vs_ligand_set *set);

/* Graph analysis of ligand i of a batch (host): detect_torsions
 * (ligand.cpp:126-139) writes the rotatable bond indices (ascending) to
 * bonds_out (capacity n_bonds) and one right-set membership byte per atom per
 * torsion to right_mask_out (n_torsions * n_atoms); returns the torsion
 * count.  vs_bridge_bonds (ligand.cpp:57-99) writes one flag per bond. */
int32_t vs_detect_torsions(const vs_ligand_batch *b, int32_t i, uint16_t *bonds_out, uint8_t *right_mask_out);
int32_t vs_bridge_bonds(const vs_ligand_batch *b, int32_t i, uint8_t *bridge_out);

/* Deterministic synthetic drug-like SMILES: candidates are assembled from
 * ring/linker/substituent fragments with a seeded xoshiro256** stream and
 * kept when the prepared graph has heavy atoms in [min_heavy, max_heavy]
 * and detect_torsions count in [min_rot, max_rot].  Writes n
 * NUL-terminated strings back to back into buf (capacity cap bytes) and
 * returns the number of bytes used, or -1 if cap is too small. */
int64_t vs_synth_smiles(int32_t n, uint64_t seed, int32_t min_heavy, int32_t max_heavy, int32_t min_rot,
                        int32_t max_rot, char *buf, int64_t cap);
/* The same with a grammar choice: 0 = the drug-like grammar above
 * (vs_synth_smiles), 1 = wide (adds larger rigid fused systems and flexible
 * chain linkers/tails, for the BASELINE configs[2] size sweep).  Returns -2
 * when the window is unreachable. */
int64_t vs_synth_smiles_ex(int32_t n, uint64_t seed, int32_t min_heavy, int32_t max_heavy, int32_t min_rot,
                           int32_t max_rot, int32_t grammar, char *buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* VS_PREP_H */
