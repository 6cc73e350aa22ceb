/*
 * vs_dock.h — C ABI of the B200 dock-and-score path (libvsdock.so).
 *
 * This is the drop-in boundary for the reference's hot path
 *   DockResult vscreen::dock_and_score(const Pocket&, const Ligand&,
 *                                      const ScoringConfig&)
 *   (/root/reference/proj/include/vscreen/dockengine/search.hpp:71-72,
 *    implementation src/dockengine/search.cpp:238-276)
 * and the public sub-APIs beneath it (search.hpp:28-79, grid.hpp:35-48,
 * chem.hpp:21-26).  Plain pointers and sizes only; no C++ or torch types.
 * The C++ drop-in headers under include/vscreen/ and the Python package
 * paper_2110_11644_b200 are thin layers over these entry points.
 *
 * Error convention (reference: C++ exceptions, error.hpp:14-52).  Every call
 * returns a vs_status.  Whole-call failures (bad config -> InvalidArgument,
 * search.cpp:240-243; CUDA errors; missing device) fail the call and set a
 * thread-local message readable with vs_last_error_message().  Failures the
 * reference raises per ligand (empty conformation transform.cpp:50,
 * degenerate torsion axis transform.cpp:62, torsion index out of range
 * transform.cpp:57/67, no heavy atoms transform.cpp:111) mark only that
 * ligand's slot (vs_dock_result.status) — the batch continues, as the
 * reference's docker workers count dock_errors and carry on
 * (pipeline.cpp:218-238).
 *
 * Threading: calls on distinct vs_context objects may run concurrently;
 * one vs_context serialises its own calls (it owns one CUDA stream).
 */
#ifndef VS_DOCK_H
#define VS_DOCK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VS_ABI_VERSION 1

typedef enum vs_status {
  VS_OK = 0,
  VS_ERR_INVALID_ARGUMENT = 1, /* reference InvalidArgument (whole call) */
  VS_ERR_NO_DEVICE = 2,        /* no CUDA device / extension unusable    */
  VS_ERR_CUDA = 3,             /* CUDA runtime failure                   */
  VS_ERR_LIMIT = 4,            /* input exceeds a documented device limit */
  VS_ERR_INTERNAL = 5
} vs_status;

/* Per-ligand outcome (vs_dock_result.status and friends). */
typedef enum vs_ligand_status {
  VS_LIG_OK = 0,
  VS_LIG_EMPTY = 1,           /* "empty conformation" (transform.cpp:50)        */
  VS_LIG_DEGENERATE_AXIS = 2, /* "degenerate torsion axis" (transform.cpp:62)   */
  VS_LIG_BAD_TORSION = 3,     /* torsion bond / atom index out of range         */
  VS_LIG_NO_HEAVY = 4,        /* "no heavy atoms" (transform.cpp:111)           */
  VS_LIG_TOO_LARGE = 5,       /* exceeds VS_MAX_* device limits (see below)     */
  VS_LIG_NONFINITE = 6,       /* non-finite best score (pipeline.cpp:224-229)   */
  VS_LIG_BAD_RECORD = 7       /* vs_dock_records: the record failed to decode   */
} vs_ligand_status;

/* Device limits of the sm_100a kernels (per ligand).  The reference caps
 * sizes only through u16 counts (binary_codec.cpp:130-132); drug-like
 * ligands (<= 80 heavy atoms, <= 15 rotors) sit far inside these. */
#define VS_MAX_ATOMS 256
#define VS_MAX_HEAVY 128
#define VS_MAX_TORSIONS 31
#define VS_MAX_RESTARTS 65536 /* k <= ~7000: select state in shared memory, beyond in global */

/* Element codes: wire-stable, elements.hpp:14-26. */
enum {
  VS_ELEM_C = 0, VS_ELEM_N = 1, VS_ELEM_O = 2, VS_ELEM_S = 3, VS_ELEM_P = 4,
  VS_ELEM_F = 5, VS_ELEM_CL = 6, VS_ELEM_BR = 7, VS_ELEM_I = 8, VS_ELEM_H = 9,
  VS_ELEM_OTHER = 10
};

/* Search knobs: ScoringConfig, pose.hpp:33-48 (same fields, same defaults). */
typedef struct vs_scoring_config {
  int32_t restarts;          /* 256 */
  int32_t rescored;          /* 30 */
  double rmsd_threshold;     /* 3.0 A */
  double step_translation;   /* 1.0 A */
  double step_rotation;      /* 20 deg in rad */
  double step_torsion;       /* 20 deg in rad */
  double min_translation;    /* 0.1 A */
  int32_t max_iterations;    /* 200 */
  int32_t flatten_max_sweeps;/* 20 */
} vs_scoring_config;

/* Rigid binding site: Pocket, pocket.hpp:28-57.  values is x-fastest,
 * value_index = ix + dims[0]*(iy + dims[1]*iz) (pocket.hpp:36-41). */
typedef struct vs_pocket_desc {
  double origin[3];
  double spacing;
  int32_t dims[3];
  const double *values;            /* dims[0]*dims[1]*dims[2] */
  int32_t n_protein;
  const uint8_t *protein_element;  /* n_protein */
  const double *protein_xyz;       /* 3*n_protein, (x,y,z) per atom */
} vs_pocket_desc;

/* A batch of ligands in structure-of-arrays form: Ligand, ligand.hpp:19-71.
 * Ligand i owns atoms [atom_offset[i], atom_offset[i+1]), bonds
 * [bond_offset[i], ...), torsions [torsion_offset[i], ...).  Atom and bond
 * indices inside a ligand are local (0-based), as in the reference.  Torsion
 * t (global index) rotates right_atoms[right_offset[t] .. right_offset[t+1])
 * (TorsionalBond::right_set, ascending) about bond torsion_bond[t]. */
typedef struct vs_ligand_batch {
  int32_t n_ligands;
  const int32_t *atom_offset;     /* n_ligands+1 */
  const double *xyz;              /* 3*n_atoms_total */
  const uint8_t *element;         /* n_atoms_total */
  const uint8_t *is_heavy;        /* n_atoms_total (0/1) */
  const int32_t *bond_offset;     /* n_ligands+1 */
  const uint16_t *bond_a;         /* n_bonds_total */
  const uint16_t *bond_b;
  const uint8_t *bond_order;      /* 1..4 (BondOrder, ligand.hpp:19-25) */
  const int32_t *torsion_offset;  /* n_ligands+1 */
  const uint16_t *torsion_bond;   /* n_torsions_total, local bond index */
  const int32_t *right_offset;    /* n_torsions_total+1 */
  const uint16_t *right_atoms;    /* right_offset[n_torsions_total] */
} vs_ligand_batch;

/* One ligand's DockResult (pose.hpp:50-56) minus the heap parts, which are
 * written to caller arrays (vs_dock_batch best_angles / best_conformation). */
typedef struct vs_dock_result {
  int32_t status;            /* vs_ligand_status */
  int32_t n_survivors;       /* poses re-scored by chem_score */
  double best_score;         /* DockResult::best_score (chem score)   */
  double best_geo_score;     /* best_pose.geo_score                   */
  double rotation[4];        /* best_pose.transform.rotation (x,y,z,w) */
  double translation[3];     /* best_pose.transform.translation        */
  uint64_t poses_evaluated;  /* DockResult::poses_evaluated (= restarts) */
  uint64_t scoring_evals;    /* DockResult::scoring_evals (grid samples) */
  int32_t clash_pairs;       /* best pose: chem pairs with d < 2.0 A (chem.cpp:42) */
  int32_t oob_samples;       /* best pose: heavy atoms outside the grid box (grid.cpp:64-66) */
} vs_dock_result;

/* One pose for the local_search / initial_poses entry points (Pose,
 * pose.hpp:23-29).  angles/conformation live in caller arrays indexed by the
 * ligand's torsion/atom offsets. */
typedef struct vs_pose {
  double rotation[4];        /* x,y,z,w */
  double translation[3];
  double geo_score;
} vs_pose;

typedef struct vs_context vs_context;
typedef struct vs_pocket vs_pocket;

/* ---- library / device ------------------------------------------------- */
int vs_abi_version(void);
int vs_device_count(void);
const char *vs_last_error_message(void);
void vs_scoring_config_default(vs_scoring_config *cfg);

vs_status vs_context_create(int device, vs_context **out);
vs_status vs_context_destroy(vs_context *ctx);
/* Milliseconds of device time of the last vs_dock_batch on this context
 * (CUDA events around its kernels on the context stream) and the number of
 * kernel launches it issued. */
vs_status vs_context_last_timing(vs_context *ctx, double *kernel_ms, int32_t *launches);
/* Per-stage device milliseconds of the last vs_dock_batch: setup, flatten,
 * search (initial_poses + local_search), select (cluster + chem + best). */
vs_status vs_context_stage_timing(vs_context *ctx, double stage_ms[4]);

/* ---- pocket: uploaded once, device resident -------- */
vs_status vs_pocket_create(vs_context *ctx, const vs_pocket_desc *desc, vs_pocket **out);
/* build_pocket (grid.cpp:15-57) on the GPU: protein -> steric grid. */
vs_status vs_pocket_build(vs_context *ctx, int32_t n_protein, const uint8_t *protein_element,
                          const double *protein_xyz, const double center[3], double radius,
                          double spacing, vs_pocket **out);
/* Shape of a device pocket, and a copy of its grid values (may be NULL). */
vs_status vs_pocket_info(const vs_pocket *p, double origin[3], double *spacing, int32_t dims[3],
                         int32_t *n_protein);
vs_status vs_pocket_download(vs_context *ctx, const vs_pocket *p, double *values);
vs_status vs_pocket_destroy(vs_pocket *p);

/* ---- the hot path ------------------------------------------------------ */
/* dock_and_score over a batch (search.cpp:238-276).  results: n_ligands.
 * best_angles: n_torsions_total (may be NULL).  best_conformation:
 * 3*n_atoms_total (may be NULL). */
vs_status vs_dock_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                        const vs_scoring_config *cfg, vs_dock_result *results,
                        double *best_angles, double *best_conformation);

/* vs_dock_batch plus, when counters != NULL, the SURVEY.md Appendix B work
 * counters per ligand (9 each: S, A_rigid, A_tors, R_build, P_flat, P_chem,
 * P_rmsd, clash_pairs, oob_samples), reproduced from the run's integers in
 * the oracle's (reference-order) accounting. */
vs_status vs_dock_batch_ex(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                           const vs_scoring_config *cfg, vs_dock_result *results, double *best_angles,
                           double *best_conformation, uint64_t *counters);

/* ---- sub-APIs beneath dock_and_score (same kernels, exposed for parity) -- */
/* pocket_field_value (grid.cpp:59-91) at n points (3*n doubles). */
vs_status vs_field_values(vs_context *ctx, const vs_pocket *pocket, int64_t n, const double *xyz,
                          double *out);
/* geo_score (grid.cpp:93-104) of each ligand at the given conformation
 * (3*n_atoms_total); evals (may be NULL) receives the per-ligand count. */
vs_status vs_geo_score_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                             const double *conformation, double *out, uint64_t *evals);
/* chem_score (chem.cpp:31-46). */
vs_status vs_chem_score_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                              const double *conformation, double *out);
/* flatten (search.cpp:27-69) of each ligand from its stored coordinates.
 * conformation_out: 3*n_atoms_total; angles_out: n_torsions_total;
 * status_out: n_ligands (may be NULL). */
vs_status vs_flatten_batch(vs_context *ctx, const vs_ligand_batch *batch, int32_t max_sweeps,
                           double *conformation_out, double *angles_out, int32_t *status_out);
/* initial_poses (search.cpp:84-107) of ONE ligand (batch->n_ligands == 1)
 * from its stored (base) coordinates and the given flat angles: k poses
 * (poses_out[k]) and conformations (conformations_out[k * 3 * n_atoms]);
 * evals receives k * n_heavy. */
vs_status vs_initial_poses(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                           const double *flat_angles, int32_t k, vs_pose *poses_out, double *conformations_out,
                           uint64_t *evals, int32_t *status_out);
/* cluster_and_select (search.cpp:195-236) of n_poses poses of ONE ligand
 * (geo scores + conformations n_poses * 3 * n_atoms): writes the selected
 * pose indices in output order (leaders, then followers) and their count. */
vs_status vs_cluster_select(vs_context *ctx, const vs_ligand_batch *batch, int32_t n_poses, const double *geo,
                            const double *conformations, double threshold, int32_t top, int32_t *order_out,
                            int32_t *count_out);
/* local_search (search.cpp:109-193) of one pose per ligand.  poses,
 * angles (n_torsions_total) and conformation (3*n_atoms_total) are read as
 * the start pose and overwritten with the result; evals (may be NULL)
 * receives the per-ligand scoring_evals. */
vs_status vs_local_search_batch(vs_context *ctx, const vs_pocket *pocket, const vs_ligand_batch *batch,
                                const vs_scoring_config *cfg, vs_pose *poses, double *angles,
                                double *conformation, uint64_t *evals, int32_t *status_out);

/* dock_and_score of every ligand of the batch against each of n_pockets
 * pockets (BASELINE configs[4]: many pockets x one library).  The
 * ligand-only stages (setup, flatten) run once per ligand, then the search
 * and selection per pocket; results hold n_pockets x n_ligands entries,
 * pocket-major, each identical to vs_dock_batch with that pocket. */
vs_status vs_dock_batch_multi(vs_context *ctx, const vs_pocket *const *pockets, int32_t n_pockets,
                              const vs_ligand_batch *batch, const vs_scoring_config *cfg, vs_dock_result *results);

/* ---- measurement helper ------------------------------------------------- */
/* Measured FP64 DADD ops/s, FP64 DFMA flop/s and FP32 FFMA flop/s of the
 * device (the roofline denominators of this CUDA-core path). */
int vs_measure_peaks(int device, double out[3]);
/* Random-gather rate (loads/s) of elem_bytes-byte loads (2, 4, 16, 32) over a
 * ws_bytes L1/L2-resident working set: the sampler's gather roofline. */
int vs_measure_gather(int device, int64_t ws_bytes, int32_t elem_bytes, double *loads_per_s);

/* Device self-test of the branch-free square root used by the kernels
 * (dmath.cuh dsqrt) against the IEEE sqrt: n inputs drawn from seed (random
 * doubles over the whole exponent range, squares of random doubles +- a few
 * ulps -- the rounding-boundary cases -- and distances in [1e-4, 1e4] A^2).
 * Writes the number of bitwise mismatches and the first bad input.
 * Returns 0 on success (test ran), nonzero on a CUDA failure. */
int vs_selftest_sqrt(int device, uint64_t n, uint64_t seed, uint64_t *mismatches, double *first_bad);

/* Same for the shared-reciprocal division (dmath.cuh drecip/ddiv_r) against
 * IEEE a / b: random operands over the fast-path range, quotients next to
 * rounding midpoints, and unit-vector components over norms (signed zeros
 * included). */
int vs_selftest_div(int device, uint64_t n, uint64_t seed, uint64_t *mismatches, double *first_bad);

#ifdef __cplusplus
}
#endif
#endif /* VS_DOCK_H */
