// Kernel launch interface of the dock path (kernels.cu).  Host driver code
// (driver.cu) fills these argument blocks and calls the launchers.
#pragma once

#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#include "dmath.cuh"

namespace vsd {

// Per-ligand derived layout written by k_setup.  Offsets into the batch
// arrays come from the caller's atom/torsion offset arrays.
struct lig_meta {
  int n_atoms;
  int n_heavy;
  int m;
  int status;   // vs_ligand_status
  int r_all;    // sum_t |right_set(t)|          (counter model, Appendix B)
  int r_heavy;  // sum_t |right_set(t) ∩ heavy|
  int d_total;  // sum_t |D_t ∩ heavy| (stage-t prefix positions the search keeps)
};

// Device copy of one batch (vs_ligand_batch) plus derived arrays.
struct batch_dev {
  int n_lig;
  const int *pre_status;   // n or NULL: nonzero = reject the ligand (records that failed to decode)
  const int *atom_off;     // n+1
  const int *bond_off;     // n+1
  const int *tors_off;     // n+1
  const int *ditem_base;   // n (capacity m*N per ligand)
  const double *xyz;       // 3*atoms
  const uint8_t *elem;
  const uint8_t *heavy;
  const uint16_t *bond_a;
  const uint16_t *bond_b;
  const uint16_t *tors_bond;
  const int *right_off;    // torsions+1
  const uint16_t *right_atoms;
  // derived (k_setup)
  lig_meta *meta;          // n
  uint32_t *atom_tmask;    // atoms: bit t <=> atom in right_set(t)
  uint16_t *heavy_list;    // atoms capacity: local atom index of heavy h
  uint32_t *heavy_dmask;   // atoms capacity: bit t <=> heavy h in D_t
  uint16_t *tors_a;        // torsions: local atom index of bond.a (pivot)
  uint16_t *tors_b;        // torsions: local atom index of bond.b
  int *d_count;            // torsions: |D_t ∩ heavy|
  int *d_off;              // torsions: offset of D_t items in the ligand list
  uint16_t *ditems;        // ditem_base[l] + ...: heavy indices of D_t items
  uint32_t *titems;        // 2*ditem_base[l] + ...: torsion-neighbour items h | (2t+s) << 8 | pd << 14
};

// FP32 screen of the search (search.cu): one 32-bit word per
// cell at node index ix + dx * (iy + dy * iz); byte i (x-pair i = corners
// (2i, 2i + 1), i.e. (y, z) = (i & 1, i >> 1)) holds 8 * (c0 | c1 << 2), the
// offset of that pair's (a, b - a) float2 in the pair table; bit 31 = NU: the
// 4x4x4 nodes around the cell are not all equal (a point within the screen's
// error bound of one in a !NU cell has exactly the cell's constant value).
// Only for pockets with <= 4 distinct node values (2-bit codes).
struct screen_grid {
  const uint32_t *__restrict__ w;  // NULL: no screen (the search runs in FP64 only)
  float pair[32];                  // 16 x (a, b - a), FP32
  float G;                         // Lipschitz bound, sum over axes, per cell unit: 3 (vmax - vmin)
  float J;                         // largest jump at a box face: max |v - (-10)|
  float eval;                      // FP32 interpolation error bound (NU cells)
  float uni;                       // error of a uniform cell's FP32 value (0 when the palette is FP32-exact)
  float v3;                        // 3 max |value|: per-item conversion errors of the row sums, / u
  float dx1, dy1, dz1;             // dims - 1
  float fdx, fdxy;                 // node strides dx, dx * dy (linear cell index, exact in FP32)
  uint32_t last;                   // largest valid word index
};

struct pocket_dev {
  grid_view g;
  screen_grid scr;
  packed_grid packed;       // cell-packed palette codes for the search sampler
  const double *palette;    // 16 values (device)
  double center[3];
  int n_protein;
  const double *pxyz;       // 3*P
  const uint8_t *pclass;    // P: 0 hydrophobic, 1 polar, 2 other (chem.cpp:24-29)
  // culling cells for chem_score
  double cmin[3];
  double cs;                // cell size
  int cdims[3];
  const int *cell_start;    // ncells+1
  const double2 *cell_rec;  // per cell entry two double2: (x, y), (z, class as a double), protein order
};

struct search_cfg {
  int k;
  int rescored;
  double rmsd_threshold;
  int max_iter;
  double step_t, step_r, step_q, min_t;
  int flatten_sweeps;
  int n_levels;             // spin table levels
  const double *spin;       // [n_levels][6][4] (x,y,z,w), glibc trig, host computed
  const double *stepsc;     // [n_levels][4] sin hi, sin lo, cos hi, cos lo of step_q * 2^-level
  const double *fibq;       // [k][4]
};

// Per-restart scratch (item = ligand * k + restart).
struct item_out {
  double *geo;              // items
  double *T;                // items * 7 (q xyzw, t xyz)
  double *ang;              // tors_off[l]*k + r*m + t
  double *conf;             // (atom_off[l]*k + r*N + a)*3; heavy_conf: heavy atom h at + 3*h
  int heavy_conf;           // dock path: restart conformations hold the heavy atoms only (select reads
                            // nothing else; the best pose's hydrogens are rematerialised)
  unsigned long long *evals;
  int *status;
  int *iters;               // items: local_search iterations
  int *adopts;              // items: adopted neighbours
};

struct flat_out {
  int *idx;                 // torsions: lattice index of the flat angle
  double *xyz;              // 3*atoms: flat conformation
  double *centroid;         // 3*n
  int *sweeps;              // n: flatten sweeps executed
};

struct dock_out {
  void *results;            // vs_dock_result[n]
  double *best_ang;         // torsions
  double *best_conf;        // 3*atoms
  unsigned long long *counters;  // n*9 (may be NULL): S, A_rigid, A_tors, R_build, P_flat, P_chem, P_rmsd, clash, oob
  const int *sweeps;        // flatten sweeps per ligand (flat_out.sweeps)
  int *best_idx;            // n: restart of the best pose, -1 without a result (k_best_conf input)
};

void set_lattice_table(const double *sc72, const double *lo72);
// serialises (max-dynamic-shared-memory attribute, launch) pairs across host threads
std::mutex &launch_mutex();
// load every kernel of the library on the current device (vs_context_create)
void preload_kernels();
void preload_kernels_search();
void preload_kernels_codec();
void set_lattice_table_search(const double *sc72, const double *lo72);

cudaError_t launch_setup(const batch_dev &b, int restarts, cudaStream_t s);
cudaError_t launch_flatten(const batch_dev &b, int max_sweeps, const flat_out &f, int nmax_atoms, int mmax,
                           cudaStream_t s, const int *lig_index = nullptr, int n_lig = 0);
cudaError_t launch_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const flat_out &f,
                          const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                          int num_sms, cudaStream_t s, int *launches, void *args_buf,
                          const int *lig_index = nullptr, int n_lig = 0, int dmax = 0);
// device buffer size the search launchers need for their argument block
cudaError_t launch_decode(const uint8_t *bytes, const int64_t *offs, int n, const int *atom_off, const int *bond_off,
                          const int *tors_off, const int64_t *rs_off, double *xyz, uint8_t *elem, uint8_t *heavy,
                          uint8_t *border, uint16_t *ba, uint16_t *bb, uint16_t *tbond, uint16_t *rslots, int *rcount,
                          int *status, cudaStream_t s, int *nheavy = nullptr);
cudaError_t launch_compact_right(const uint16_t *slots, const int64_t *rs_off, const int *rcount, const int *right_off,
                                 int n_tors, uint16_t *right_atoms, cudaStream_t s);
size_t search_scratch_bytes(int nmax_atoms, int nmax_heavy, int mmax, int num_sms);
// dynamic shared memory of one k_search CTA for the given ligand maxima
size_t search_smem_bytes(int N, int n, int m, int dtot, bool screen);
int search_warps_per_cta();
cudaError_t launch_select(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const item_out &o,
                          const dock_out &d, int nmax_atoms, cudaStream_t s, int *sel_scratch = nullptr);
// global scratch the select needs for restart counts whose per-ligand state
// exceeds shared memory (0 otherwise)
size_t select_scratch_bytes(int n_lig, int k);
// sub-API kernels
cudaError_t launch_field_values(const pocket_dev &p, int64_t n, const double *xyz, double *out, cudaStream_t s);
cudaError_t launch_geo_score(const batch_dev &b, const pocket_dev &p, const double *conf, double *out,
                             unsigned long long *evals, cudaStream_t s);
cudaError_t launch_chem_score(const batch_dev &b, const pocket_dev &p, const double *conf, double *out,
                              cudaStream_t s);
cudaError_t launch_build_pocket(const double *hxyz, int nh, double cx, double cy, double cz, double radius,
                                double ox, double oy, double oz, double h, int d0, int d1, int d2, double *values,
                                cudaStream_t s);
// initial_poses of each ligand from given (flat) angles: k items per ligand.
cudaError_t launch_initial_poses(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *angles,
                                 const item_out &o, int *work_counter, int nmax_atoms, int nmax_heavy, int mmax,
                                 int num_sms, cudaStream_t s, void *args_buf);
// cluster_and_select of np poses of ligand 0 (search.cpp:195-236).
cudaError_t launch_cluster(const batch_dev &b, int np, const double *geo, const double *confs, double threshold,
                           int top, int *order_out, int *count_out, cudaStream_t s);
// local_search of one supplied pose per ligand (item = ligand, k = 1).
cudaError_t launch_local_search(const batch_dev &b, const pocket_dev &p, const search_cfg &c, const double *pose_in,
                                const double *ang_in, const double *conf_in, const item_out &o, int *work_counter,
                                int nmax_atoms, int nmax_heavy, int mmax, int num_sms, cudaStream_t s,
                                void *args_buf);

}  // namespace vsd
