// Ligand record stream (".xslb") on the B200: host framing and encoding,
// GPU batched decode with the torsion partitions rebuilt from the graph.
//
// k_decode: one warp per record (binary_codec.cpp:165-222).  Lanes parse the
// atoms (f32 coordinates widened to double, element, heavy flag), bonds and
// torsion bond indices in parallel and validate them in the reference's
// order; the first failing check (lowest atom, then bond, then torsion)
// becomes the record status.  Each torsion's partition (ligand.cpp:110-124)
// is a reachability sweep from the bond's `a` atom with the bond removed,
// on a shared-memory bit set relaxed over the bond list until it stops
// changing (the reachable set is unique, so it equals the reference's BFS);
// the right set is the complement, written in ascending atom order with a
// ballot compaction.  The same sweep from atom 0 checks connectivity
// (ligand.cpp:52-56).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/vs_codec.h"
#include "kernels.cuh"

namespace vsd {

namespace {

constexpr int kDecWarps = 4;
constexpr int kDecMaxAtoms = 4096;  // shared-memory bit set per warp: 128 words

__device__ __forceinline__ uint32_t rd8(const uint8_t *p) { return __ldg(p); }
__device__ __forceinline__ uint32_t rd16(const uint8_t *p) { return rd8(p) | (rd8(p + 1) << 8); }
__device__ __forceinline__ uint32_t rd32(const uint8_t *p) { return rd16(p) | (rd16(p + 2) << 16); }

struct decode_args {
  const uint8_t *bytes;
  const int64_t *offs;
  int n;
  const int *atom_off, *bond_off, *tors_off;
  const int64_t *rs_off;  // per torsion: first right-set slot (n_atoms slots per torsion)
  double *xyz;
  uint8_t *elem, *heavy, *border;
  uint16_t *ba, *bb, *tbond, *rslots;
  int *rcount;  // per torsion: right-set size
  int *status;  // per record: in = host framing status, out = decode status
  int *nheavy;  // per record: heavy atoms (NULL: not needed)
};

// Reachability from `start` over the record's bonds, bond `skip` removed,
// into the warp's bit set `vis` (n_atoms bits).
__device__ void reach(uint32_t *vis, int na, int nb, const uint16_t *ba, const uint16_t *bb, int start, int skip,
                      int lane) {
  for (int w = lane; w < (na + 31) / 32; w += 32) vis[w] = 0u;
  __syncwarp();
  if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
  __syncwarp();
  bool changed = true;
  while (changed) {
    bool mine = false;
    for (int j = lane; j < nb; j += 32) {
      if (j == skip) continue;
      const int a = ba[j], b = bb[j];
      const bool va = (vis[a >> 5] >> (a & 31)) & 1u, vb = (vis[b >> 5] >> (b & 31)) & 1u;
      if (va && !vb) {
        atomicOr(&vis[b >> 5], 1u << (b & 31));
        mine = true;
      } else if (vb && !va) {
        atomicOr(&vis[a >> 5], 1u << (a & 31));
        mine = true;
      }
    }
    changed = __any_sync(0xffffffffu, mine);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(32 * kDecWarps) k_decode(decode_args A) {
  __shared__ uint32_t s_vis[kDecWarps][kDecMaxAtoms / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * kDecWarps + w;
  if (r >= A.n) return;
  if (A.status[r] != VS_REC_OK) return;  // framing already failed
  uint32_t *vis = s_vis[w];
  const uint8_t *p = A.bytes + A.offs[r];
  const int name_len = (int)rd16(p + 6);
  const uint8_t *q = p + 8 + name_len;
  const int na = (int)rd16(q), nb = (int)rd16(q + 2), nt = (int)rd16(q + 4);
  if (na > kDecMaxAtoms) {
    if (lane == 0) A.status[r] = VS_REC_TOO_LARGE;
    return;
  }
  const uint8_t *pa = q + 6, *pb = pa + 14 * (size_t)na, *pt = pb + 5 * (size_t)nb;
  const int a0 = A.atom_off[r], b0 = A.bond_off[r], t0 = A.tors_off[r];
  // atoms (binary_codec.cpp:189-203): element checked before finiteness
  unsigned long long first = ~0ull;  // (index << 4) | code of the first failure
  for (int i = lane; i < na; i += 32) {
    const uint8_t *e = pa + 14 * (size_t)i;
    const float x = __uint_as_float(rd32(e)), y = __uint_as_float(rd32(e + 4)), z = __uint_as_float(rd32(e + 8));
    const uint32_t code = rd8(e + 12), flags = rd8(e + 13);
    A.xyz[3 * (size_t)(a0 + i)] = (double)x;
    A.xyz[3 * (size_t)(a0 + i) + 1] = (double)y;
    A.xyz[3 * (size_t)(a0 + i) + 2] = (double)z;
    A.elem[a0 + i] = (uint8_t)code;
    A.heavy[a0 + i] = (flags & 1u) ? 1 : 0;
    int err = 0;
    if (code > 10u) err = VS_REC_BAD_ELEMENT;
    else if (!isfinite(x) || !isfinite(y) || !isfinite(z)) err = VS_REC_NONFINITE;
    if (err && first == ~0ull) first = ((unsigned long long)i << 4) | (unsigned long long)err;
  }
  if (A.nheavy) {
    int hc = 0;
    for (int i = lane; i < na; i += 32) hc += (rd8(pa + 14 * (size_t)i + 13) & 1u) ? 1 : 0;
    hc = __reduce_add_sync(0xffffffffu, hc);
    if (lane == 0) A.nheavy[r] = hc;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, first, off);
    first = o < first ? o : first;
  }
  int st = first != ~0ull ? (int)(first & 15ull) : VS_REC_OK;
  // bonds (binary_codec.cpp:204-213): indices checked before the order
  if (st == VS_REC_OK) {
    unsigned long long fb = ~0ull;
    for (int j = lane; j < nb; j += 32) {
      const uint8_t *e = pb + 5 * (size_t)j;
      const uint32_t a = rd16(e), b = rd16(e + 2), order = rd8(e + 4);
      A.ba[b0 + j] = (uint16_t)a;
      A.bb[b0 + j] = (uint16_t)b;
      A.border[b0 + j] = (uint8_t)order;
      int err = 0;
      if (a >= (uint32_t)na || b >= (uint32_t)na || a == b) err = VS_REC_BAD_BOND;
      else if (order < 1u || order > 4u) err = VS_REC_BAD_BOND_ORDER;
      if (err && fb == ~0ull) fb = ((unsigned long long)j << 4) | (unsigned long long)err;
    }
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, fb, off);
      fb = o < fb ? o : fb;
    }
    if (fb != ~0ull) st = (int)(fb & 15ull);
  }
  __syncwarp();
  // torsions in order (binary_codec.cpp:214-221): index, then the partition
  for (int k = 0; k < nt && st == VS_REC_OK; ++k) {
    const uint32_t bi = rd16(pt + 2 * (size_t)k);
    if (lane == 0) A.tbond[t0 + k] = (uint16_t)bi;
    if (bi >= (uint32_t)nb) {
      st = VS_REC_BAD_TORSION_INDEX;
      break;
    }
    const int ea = A.ba[b0 + bi], eb = A.bb[b0 + bi];
    reach(vis, na, nb, A.ba + b0, A.bb + b0, ea, (int)bi, lane);
    if ((vis[eb >> 5] >> (eb & 31)) & 1u) {
      st = VS_REC_NOT_BRIDGE;
      break;
    }
    // right set = atoms not reachable from a, ascending (ligand.cpp:120-122)
    uint16_t *out = A.rslots + A.rs_off[t0 + k];
    int cnt = 0;
    for (int c0 = 0; c0 < na; c0 += 32) {
      const int i = c0 + lane;
      const bool right = i < na && !((vis[i >> 5] >> (i & 31)) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, right);
      if (right) out[cnt + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)i;
      cnt += __popc(bal);
    }
    if (lane == 0) A.rcount[t0 + k] = cnt;
    __syncwarp();
  }
  // connectivity (binary_codec.cpp:222, ligand.cpp:52-56)
  if (st == VS_REC_OK && na > 0) {
    reach(vis, na, nb, A.ba + b0, A.bb + b0, 0, -1, lane);
    bool all = true;
    for (int i = lane; i < na; i += 32) all &= ((vis[i >> 5] >> (i & 31)) & 1u) != 0u;
    if (!__all_sync(0xffffffffu, all)) st = VS_REC_DISCONNECTED;
  }
  if (lane == 0) A.status[r] = st;
}

// Right sets from the padded decode slots into the dock path's compact
// right_atoms (thread per torsion; failed records have count 0).
__global__ void k_compact_right(const uint16_t *slots, const int64_t *rs_off, const int *rcount, const int *right_off,
                                int n_tors, uint16_t *right_atoms) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tors) return;
  const uint16_t *src = slots + rs_off[t];
  uint16_t *dst = right_atoms + right_off[t];
  for (int i = 0; i < rcount[t]; ++i) dst[i] = src[i];
}

}  // namespace

cudaError_t launch_compact_right(const uint16_t *slots, const int64_t *rs_off, const int *rcount, const int *right_off,
                                 int n_tors, uint16_t *right_atoms, cudaStream_t s) {
  if (n_tors <= 0) return cudaSuccess;
  k_compact_right<<<(n_tors + 127) / 128, 128, 0, s>>>(slots, rs_off, rcount, right_off, n_tors, right_atoms);
  return cudaGetLastError();
}

cudaError_t launch_decode(const uint8_t *bytes, const int64_t *offs, int n, const int *atom_off, const int *bond_off,
                          const int *tors_off, const int64_t *rs_off, double *xyz, uint8_t *elem, uint8_t *heavy,
                          uint8_t *border, uint16_t *ba, uint16_t *bb, uint16_t *tbond, uint16_t *rslots, int *rcount,
                          int *status, cudaStream_t s, int *nheavy) {
  if (n <= 0) return cudaSuccess;
  decode_args A{bytes, offs, n, atom_off, bond_off, tors_off, rs_off, xyz, elem, heavy, border,
                ba, bb, tbond, rslots, rcount, status, nheavy};
  k_decode<<<(n + kDecWarps - 1) / kDecWarps, 32 * kDecWarps, 0, s>>>(A);
  return cudaGetLastError();
}

void preload_kernels_codec() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_decode);
  cudaFuncGetAttributes(&a, k_compact_right);
}

}  // namespace vsd

// ------------------------------------------------------------------ host
namespace {

uint32_t h16(const uint8_t *p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8); }
uint32_t h32(const uint8_t *p) { return h16(p) | (h16(p + 2) << 16); }
void put16(std::vector<uint8_t> &o, uint32_t v) {
  o.push_back((uint8_t)(v & 0xFF));
  o.push_back((uint8_t)(v >> 8));
}
void put32(std::vector<uint8_t> &o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((uint8_t)((v >> (8 * i)) & 0xFF));
}

}  // namespace

extern "C" int32_t vs_xslb_frame(const uint8_t *bytes, int64_t size, int64_t start, int32_t max_records,
                                 int64_t *offsets, int64_t *next) {
  if (!bytes || size < 0 || start < 0 || max_records < 0) return -1;
  int64_t at = start;
  int32_t n = 0;
  while (n < max_records && at + 6 <= size && bytes[at] == 0xD0 && bytes[at + 1] == 0xC5) {
    const int64_t end = at + 6 + (int64_t)h32(bytes + at + 2);
    if (end > size) break;
    if (offsets) offsets[n] = at;
    ++n;
    at = end;
  }
  if (next) *next = at;
  return n;
}

extern "C" int64_t vs_encode_records(const vs_ligand_batch *b, const char *const *names, uint8_t *out, int64_t cap) {
  if (!b) return 0;
  std::vector<uint8_t> o;
  for (int i = 0; i < b->n_ligands; ++i) {
    const int A0 = b->atom_offset[i], A1 = b->atom_offset[i + 1];
    const int B0 = b->bond_offset[i], B1 = b->bond_offset[i + 1];
    const int T0 = b->torsion_offset[i], T1 = b->torsion_offset[i + 1];
    const std::string name = names && names[i] ? names[i] : "";
    const size_t payload = 2 + name.size() + 6 + 14 * (size_t)(A1 - A0) + 5 * (size_t)(B1 - B0) + 2 * (size_t)(T1 - T0);
    o.push_back(0xD0);
    o.push_back(0xC5);
    put32(o, (uint32_t)payload);
    put16(o, (uint32_t)name.size());
    o.insert(o.end(), name.begin(), name.end());
    put16(o, (uint32_t)(A1 - A0));
    put16(o, (uint32_t)(B1 - B0));
    put16(o, (uint32_t)(T1 - T0));
    for (int a = A0; a < A1; ++a) {
      for (int c = 0; c < 3; ++c) {
        const float f = (float)b->xyz[3 * a + c];
        uint32_t bits;
        std::memcpy(&bits, &f, 4);
        put32(o, bits);
      }
      o.push_back(b->element[a]);
      o.push_back(b->is_heavy[a] ? 0x01 : 0x00);
    }
    for (int k = B0; k < B1; ++k) {
      put16(o, b->bond_a[k]);
      put16(o, b->bond_b[k]);
      o.push_back(b->bond_order ? b->bond_order[k] : 1);
    }
    for (int t = T0; t < T1; ++t) put16(o, b->torsion_bond[t]);
  }
  if ((int64_t)o.size() > cap || !out) return -(int64_t)o.size();
  std::memcpy(out, o.data(), o.size());
  return (int64_t)o.size();
}
