// Seeded synthetic drug-like SMILES in the reference's SMILES subset
// (smiles.hpp:26-31: organic atoms, aromatic c/n/o/s, branches, ring digits
// 1-9, no brackets/charges/stereo).  SURVEY.md §8d config 1/2 asks for
// ~30 heavy atoms and ~6 rotatable bonds as counted by detect_torsions.
//
// A candidate is a main chain of ring units joined by linkers, with optional
// ring substituents and a terminal tail:  [tail] R (L R)* [tail]
// Candidates whose heavy-atom / torsion counts fall outside the requested
// window are rejected, so the library is an exact draw from the window.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <cstring>
#include <string>
#include <vector>

#include "vs_prep.h"

namespace vsprep {
struct Mol;
}
// prep.cpp internals re-declared here to count atoms and torsions.
namespace vsprep_internal {
bool counts(const std::string &smiles, int *heavy, int *rot);
}

namespace {

struct Xoshiro {  // xoshiro256**
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    for (int i = 0; i < 4; ++i) {  // splitmix64 seeding
      seed += 0x9e3779b97f4a7c15ULL;
      uint64_t z = seed;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      s[i] = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  int below(int n) { return static_cast<int>(next() % static_cast<uint64_t>(n)); }
};

// Ring units: {prefix-with-attachment, exit form}.  '%' marks the ring digit.
// The exit form leaves a branch open so the main chain continues from a
// second ring atom (para/meta/ortho-like), e.g. "c%ccc(cc%)" then "<linker>".
struct RingUnit {
  const char *terminal;  // ring as the last unit
  const char *exits[3];  // ring with the chain continuing from another atom
  const char *subst;     // ring with one substituent slot '$' and chain exit
};
const RingUnit kRings[] = {
    {"c%ccccc%", {"c%ccc(cc%)", "c%cc(ccc%)", "c%c(cccc%)"}, "c%cc($)c(cc%)"},
    {"c%ccncc%", {"c%ccc(nc%)", "c%cc(ncc%)", "c%cnc(cc%)"}, "c%cc($)c(nc%)"},
    {"c%ccoc%", {"c%ccc(o%)", "c%cc(oc%)", "c%cc(co%)"}, "c%c($)cc(o%)"},
    {"c%ccsc%", {"c%ccc(s%)", "c%cc(sc%)", "c%cc(cs%)"}, "c%c($)cc(s%)"},
    {"C%CCCCC%", {"C%CCC(CC%)", "C%CC(CCC%)", "C%C(CCCC%)"}, "C%CC($)C(CC%)"},
    {"C%CCNCC%", {"C%CCN(CC%)", "C%CC(NCC%)", "C%CNC(CC%)"}, "C%CC($)N(CC%)"},
    {"C%CCOCC%", {"C%COC(CC%)", "C%CC(OCC%)", "C%COCC%"}, "C%OC($)C(CC%)"},
    {"C%CCCC%", {"C%CCC(C%)", "C%CC(CC%)", "C%C(CCC%)"}, "C%CC($)C(C%)"},
    {"c%cnccn%", {"c%cnc(cn%)", "c%cncc(n%)", "c%c(nccn%)"}, "c%c($)ncc(n%)"},
    // fused bicyclics: '&' is the second ring digit of the unit
    {"c%ccc&ccccc&c%", {"c%ccc&cc(ccc&c%)", "c%ccc&c(cccc&c%)", "c%cc(c&ccccc&c%)"}, "c%cc($)c&cc(ccc&c%)"},
    {"c%ccc&occc&c%", {"c%ccc&oc(cc&c%)", "c%cc(c&occc&c%)", "c%ccc&occ(c&c%)"}, "c%cc($)c&oc(cc&c%)"},
    {"C%CCc&ccccc&C%", {"C%CCc&cc(ccc&C%)", "C%CCc&c(cccc&C%)", "C%CC(c&ccccc&C%)"}, "C%CCc&cc($)c(cc&C%)"},
    {"c%ccc&ncccc&c%", {"c%ccc&ncc(cc&c%)", "c%ccc&nc(ccc&c%)", "c%cc(c&ncccc&c%)"}, "c%cc($)c&ncc(cc&c%)"},
};
// Wide grammar (vs_synth_smiles_ex grammar 1, the configs[2] size sweep):
// larger rigid fused systems ('^' = third ring digit) for heavy, low-rotor
// ligands, and flexible chain linkers / tails for small, many-rotor ones.
const RingUnit kRingsWide[] = {
    {"c%ccc&cc^ccccc^cc&c%", {"c%ccc&cc^ccc(cc^cc&c%)", "c%ccc&cc^cccc(c^cc&c%)", "c%cc(c&cc^ccccc^cc&c%)"},
     "c%cc($)c&cc^ccc(cc^cc&c%)"},
    {"c%ccc&c(c%)ccc^ccccc&^", {"c%ccc&c(c%)ccc^cccc(c&^)", "c%cc(c&c(c%)ccc^ccccc&^)", "c%ccc&c(c%)cc(c^ccccc&^)"},
     "c%cc($)c&c(c%)ccc^cccc(c&^)"},
    {"C%CCC&CCCCC&C%", {"C%CCC&CC(CCC&C%)", "C%CCC&C(CCCC&C%)", "C%CC(C&CCCCC&C%)"}, "C%CC($)C&CC(CCC&C%)"},
};
const char *kLinkersWide[] = {"CCCC", "CCCCC", "OCCO", "CCOCC", "CCCCCC", "CCNCC", "C", "CC", "", "O"};
const char *kTailsWide[] = {"CCCCC", "CCCCCCC", "OCCCC", "CCCCOC", "F", "Cl", "C", "Br"};
const char *kSubstWide[] = {"F", "Cl", "Br", "C", "CCCC", "OCCC"};

const char *kLinkers[] = {"",   "",    "C",      "CC",   "O",     "N",  "C(=O)N", "NC(=O)", "C(=O)O", "OC",
                          "CO", "S",   "CN",     "NC",   "C(=O)", "CC(=O)N", "OCC", "CCO", "C(C)N", "CCN"};
const char *kSubst[] = {"F", "Cl", "Br", "C", "O", "N", "OC", "C(=O)O", "C#N", "C(F)(F)F", "N(C)C", "CC", "C(=O)N", "OCC"};
const char *kTails[] = {"C", "CC", "CCC", "OC", "N(C)C", "CC(C)C", "OCC", "NC(=O)C", "CCO", "C(=O)OC", "CCN", "F", "Cl"};

std::string with_digit(const char *tmpl, int digit, const char *subst) {
  std::string out;
  for (const char *p = tmpl; *p; ++p) {
    if (*p == '%')
      out += static_cast<char>('0' + digit);
    else if (*p == '&')
      out += static_cast<char>('0' + digit + 1);
    else if (*p == '^')
      out += static_cast<char>('0' + digit + 2);
    else if (*p == '$')
      out += subst;
    else
      out += *p;
  }
  return out;
}

std::string candidate(Xoshiro &rng, int rmin, int rmax) {
  std::string s;
  if (rng.below(3) == 0) s += kTails[rng.below(static_cast<int>(sizeof(kTails) / sizeof(*kTails)))];
  const int rings = rmin + rng.below(rmax - rmin + 1);
  for (int r = 0; r < rings; ++r) {
    const RingUnit &u = kRings[rng.below(static_cast<int>(sizeof(kRings) / sizeof(*kRings)))];
    const int digit = 1;  // each unit closes its rings before the next opens: digits 1, 2 are reused
    const bool last = r + 1 == rings;
    const bool tail_after = last && rng.below(3) == 0;
    if (last && !tail_after) {
      s += with_digit(u.terminal, digit, "");
    } else if (rng.below(3) == 0) {
      s += with_digit(u.subst, digit, kSubst[rng.below(static_cast<int>(sizeof(kSubst) / sizeof(*kSubst)))]);
    } else {
      s += with_digit(u.exits[rng.below(3)], digit, "");
    }
    if (!last)
      s += kLinkers[rng.below(static_cast<int>(sizeof(kLinkers) / sizeof(*kLinkers)))];
    else if (tail_after)
      s += kTails[rng.below(static_cast<int>(sizeof(kTails) / sizeof(*kTails)))];
  }
  return s;
}

template <typename T, size_t N>
constexpr int count_of(const T (&)[N]) {
  return static_cast<int>(N);
}

std::string candidate_wide(Xoshiro &rng, int rmin, int rmax) {
  std::string s;
  if (rng.below(2) == 0) s += kTailsWide[rng.below(count_of(kTailsWide))];
  const int rings = rmin + rng.below(rmax - rmin + 1);
  for (int r = 0; r < rings; ++r) {
    const bool big = rng.below(3) == 0;
    const RingUnit &u = big ? kRingsWide[rng.below(count_of(kRingsWide))] : kRings[rng.below(count_of(kRings))];
    const bool last = r + 1 == rings;
    const bool tail_after = last && rng.below(2) == 0;
    if (last && !tail_after) {
      s += with_digit(u.terminal, 1, "");
    } else if (rng.below(3) == 0) {
      s += with_digit(u.subst, 1, kSubstWide[rng.below(count_of(kSubstWide))]);
    } else {
      s += with_digit(u.exits[rng.below(3)], 1, "");
    }
    if (!last)
      s += rng.below(2) ? kLinkersWide[rng.below(count_of(kLinkersWide))] : kLinkers[rng.below(count_of(kLinkers))];
    else if (tail_after)
      s += kTailsWide[rng.below(count_of(kTailsWide))];
  }
  return s;
}

}  // namespace

// Blocks of 256 accepted SMILES, each from its own xoshiro stream
// (seed, block) -- deterministic for any thread count.
extern "C" int64_t vs_synth_smiles_ex(int32_t n, uint64_t seed, int32_t min_heavy, int32_t max_heavy,
                                      int32_t min_rot, int32_t max_rot, int32_t grammar, char *buf, int64_t cap) {
  constexpr int kBlock = 256;
  const int nblocks = (n + kBlock - 1) / kBlock;
  std::vector<std::vector<std::string>> blocks(static_cast<size_t>(nblocks));
  std::atomic<int> next{0};
  std::atomic<bool> unreachable{false};
  auto work = [&] {
    for (int bi = next++; bi < nblocks; bi = next++) {
      Xoshiro rng(seed * 0x9e3779b97f4a7c15ULL + static_cast<uint64_t>(bi) + 1);
      const int want = std::min(kBlock, n - bi * kBlock);
      // ring units scale with the requested size (2-3 for ~30 heavy atoms)
      const int rmin = grammar ? 1 : std::max(1, min_heavy / 13);
      const int rmax = grammar ? std::max(2, max_heavy / 8) : std::max(rmin + 1, max_heavy / 11);
      auto &out = blocks[static_cast<size_t>(bi)];
      int64_t tries = 0;
      while (static_cast<int>(out.size()) < want) {
        // give up on windows the grammar cannot reach (nothing accepted in
        // 200k candidates) or reaches too rarely
        if (++tries > 4000LL * kBlock || (out.empty() && tries > 200000) || unreachable) {
          unreachable = true;
          return;
        }
        std::string s = grammar ? candidate_wide(rng, rmin, rmax) : candidate(rng, rmin, rmax);
        int heavy = 0, rot = 0;
        if (!vsprep_internal::counts(s, &heavy, &rot)) continue;
        if (heavy < min_heavy || heavy > max_heavy || rot < min_rot || rot > max_rot) continue;
        out.push_back(std::move(s));
      }
    }
  };
  const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nblocks));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto &th : pool) th.join();
  if (unreachable) return -2;
  int64_t used = 0;
  for (const auto &blk : blocks)
    for (const auto &s : blk) {
      const int64_t need = static_cast<int64_t>(s.size()) + 1;
      if (used + need > cap) return -1;
      std::memcpy(buf + used, s.c_str(), static_cast<std::size_t>(need));
      used += need;
    }
  return used;
}

extern "C" int64_t vs_synth_smiles(int32_t n, uint64_t seed, int32_t min_heavy, int32_t max_heavy, int32_t min_rot,
                                   int32_t max_rot, char *buf, int64_t cap) {
  return vs_synth_smiles_ex(n, seed, min_heavy, max_heavy, min_rot, max_rot, 0, buf, cap);
}
