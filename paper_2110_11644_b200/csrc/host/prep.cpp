// Input side of the dock path: SMILES -> hydrogen-complete graph -> 3D
// embedding -> rotatable-bond partition (include/vs_prep.h).
//
// Restates, for bit-identical coordinates, the reference's
//   parse_smiles    smiles.cpp:37-211
//   add_hydrogens   hydrogens.cpp:33-72
//   embed_3d        embed.cpp:44-419 (ring finder, natural-extension placer)
//   detect_torsions ligand.cpp:15-139 (bridges, heavy degree, BFS partition)
// using the Eigen 3.4 evaluation order of SURVEY.md Appendix A for the few
// reductions involved (norm/dot = (a0 + a1) + a2, generic cross product).
// Host-only; compiled -ffp-contract=off so no a*b+c is fused.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "vs_prep.h"

namespace vsprep {

constexpr double kPi = 3.14159265358979323846;

struct V3 {
  double x = 0, y = 0, z = 0;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator-(V3 a) { return {-a.x, -a.y, -a.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double sqn(V3 a) { return dot(a, a); }
inline double norm(V3 a) { return std::sqrt(sqn(a)); }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 normalized(V3 a) {
  const double n = sqn(a);
  if (n > 0.0) {
    const double r = std::sqrt(n);
    return {a.x / r, a.y / r, a.z / r};
  }
  return a;
}

enum : uint8_t { C = 0, N = 1, O = 2, S = 3, P = 4, F = 5, Cl = 6, Br = 7, I = 8, H = 9, Other = 10 };
enum : uint8_t { Single = 1, Double = 2, Triple = 3, Aromatic = 4 };

struct Mol {
  std::string name;
  std::vector<uint8_t> elem, heavy;
  std::vector<V3> pos;
  std::vector<uint16_t> ba, bb;
  std::vector<uint8_t> order;
  std::vector<uint16_t> tors;
  std::vector<std::vector<uint16_t>> right;
  std::size_t n() const { return elem.size(); }
};

struct PrepError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using Adj = std::vector<std::vector<std::pair<uint16_t, uint16_t>>>;
Adj adjacency(const Mol &m) {  // ligand.cpp:15-25
  Adj g(m.n());
  for (std::size_t i = 0; i < m.ba.size(); ++i) {
    g[m.ba[i]].emplace_back(m.bb[i], static_cast<uint16_t>(i));
    g[m.bb[i]].emplace_back(m.ba[i], static_cast<uint16_t>(i));
  }
  return g;
}
std::vector<uint8_t> reachable(const Adj &g, uint16_t start, int skip) {  // ligand.cpp:30-46
  std::vector<uint8_t> seen(g.size(), 0);
  std::vector<uint16_t> st{start};
  seen[start] = 1;
  while (!st.empty()) {
    const uint16_t at = st.back();
    st.pop_back();
    for (auto [nx, b] : g[at]) {
      if (static_cast<int>(b) == skip || seen[nx]) continue;
      seen[nx] = 1;
      st.push_back(nx);
    }
  }
  return seen;
}
bool connected(const Mol &m) {  // ligand.cpp:50-55
  if (m.n() == 0) return false;
  const auto s = reachable(adjacency(m), 0, -1);
  return std::all_of(s.begin(), s.end(), [](uint8_t v) { return v != 0; });
}
std::vector<uint8_t> bridge_bonds(const Mol &m) {  // ligand.cpp:57-99, iterative low-link
  const Adj g = adjacency(m);
  std::vector<uint8_t> br(m.ba.size(), 0);
  std::vector<int> disc(m.n(), -1), low(m.n(), 0);
  int timer = 0;
  struct Frame {
    uint16_t at;
    int in_bond;
    std::size_t next;
  };
  for (std::size_t root = 0; root < m.n(); ++root) {
    if (disc[root] != -1) continue;
    std::vector<Frame> st{{static_cast<uint16_t>(root), -1, 0}};
    disc[root] = low[root] = timer++;
    while (!st.empty()) {
      Frame &f = st.back();
      if (f.next < g[f.at].size()) {
        const auto [nx, b] = g[f.at][f.next++];
        if (static_cast<int>(b) == f.in_bond) continue;
        if (disc[nx] == -1) {
          disc[nx] = low[nx] = timer++;
          st.push_back({nx, static_cast<int>(b), 0});
        } else {
          low[f.at] = std::min(low[f.at], disc[nx]);
        }
      } else {
        const Frame done = f;
        st.pop_back();
        if (!st.empty()) {
          Frame &par = st.back();
          low[par.at] = std::min(low[par.at], low[done.at]);
          if (low[done.at] > disc[par.at]) br[static_cast<std::size_t>(done.in_bond)] = 1;
        }
      }
    }
  }
  return br;
}
int heavy_degree(const Mol &m, uint16_t a) {  // ligand.cpp:101-108
  int d = 0;
  for (std::size_t i = 0; i < m.ba.size(); ++i) {
    if (m.ba[i] == a && m.heavy[m.bb[i]]) ++d;
    if (m.bb[i] == a && m.heavy[m.ba[i]]) ++d;
  }
  return d;
}
void detect_torsions(Mol &m) {  // ligand.cpp:110-139
  m.tors.clear();
  m.right.clear();
  const auto br = bridge_bonds(m);
  const Adj g = adjacency(m);
  for (std::size_t i = 0; i < m.ba.size(); ++i) {
    if (m.order[i] != Single || !br[i]) continue;
    if (!m.heavy[m.ba[i]] || !m.heavy[m.bb[i]]) continue;
    if (heavy_degree(m, m.ba[i]) < 2 || heavy_degree(m, m.bb[i]) < 2) continue;
    const auto left = reachable(g, m.ba[i], static_cast<int>(i));
    std::vector<uint16_t> r;
    for (std::size_t a = 0; a < m.n(); ++a)
      if (!left[a]) r.push_back(static_cast<uint16_t>(a));
    m.tors.push_back(static_cast<uint16_t>(i));
    m.right.push_back(std::move(r));
  }
}

// ------------------------------------------------------------------ SMILES
// smiles.cpp:37-211: organic subset, branches, ring digits 1-9, - = # :.
class SmilesParser {
 public:
  explicit SmilesParser(const std::string &t) : t_(t) {}
  Mol run() {
    if (t_.empty()) fail("empty SMILES");
    while (pos_ < t_.size()) step();
    if (pending_) fail("dangling bond symbol");
    if (!branches_.empty()) fail("unclosed branch");
    for (int i = 0; i < 9; ++i)
      if (ring_atom_[i] >= 0) fail("unclosed ring bond " + std::to_string(i + 1));
    if (m_.n() == 0) fail("no atoms");
    if (!connected(m_)) fail("disconnected molecule");
    m_.name = t_;
    return std::move(m_);
  }

 private:
  [[noreturn]] void fail(const std::string &msg) { throw PrepError("SMILES: " + msg); }
  static uint8_t order_of(char c) { return c == '-' ? Single : c == '=' ? Double : c == '#' ? Triple : Aromatic; }
  void step() {
    const char c = t_[pos_];
    if (c == '(') {
      if (prev_ < 0 || pending_) fail("bad branch open");
      branches_.push_back(prev_);
      ++pos_;
    } else if (c == ')') {
      if (branches_.empty() || pending_) fail("bad branch close");
      prev_ = branches_.back();
      branches_.pop_back();
      ++pos_;
    } else if (c == '-' || c == '=' || c == '#' || c == ':') {
      if (prev_ < 0 || pending_) fail("misplaced bond symbol");
      pending_ = order_of(c);
      ++pos_;
    } else if (c >= '1' && c <= '9') {
      ring_digit(c - '1');
      ++pos_;
    } else if (std::strchr("[%/\\@+*.0", c) != nullptr) {
      fail(std::string("unsupported character '") + c + "'");
    } else {
      atom();
    }
  }
  void ring_digit(int slot) {
    if (prev_ < 0) fail("ring closure before any atom");
    if (ring_atom_[slot] < 0) {
      ring_atom_[slot] = prev_;
      ring_order_[slot] = pending_;
      pending_.reset();
      return;
    }
    if (ring_atom_[slot] == prev_) fail("ring bond to the same atom");
    std::optional<uint8_t> o = pending_;
    if (o && ring_order_[slot] && *o != *ring_order_[slot]) fail("ring bond order mismatch");
    if (!o) o = ring_order_[slot];
    bond(static_cast<uint16_t>(ring_atom_[slot]), static_cast<uint16_t>(prev_), o);
    ring_atom_[slot] = -1;
    ring_order_[slot].reset();
    pending_.reset();
  }
  void atom() {
    const char c = t_[pos_];
    uint8_t e;
    bool arom = false;
    const char nx = pos_ + 1 < t_.size() ? t_[pos_ + 1] : '\0';
    if (c == 'C' && nx == 'l') {
      e = Cl;
      pos_ += 2;
    } else if (c == 'B' && nx == 'r') {
      e = Br;
      pos_ += 2;
    } else {
      switch (c) {
        case 'C': e = C; break;
        case 'N': e = N; break;
        case 'O': e = O; break;
        case 'S': e = S; break;
        case 'P': e = P; break;
        case 'F': e = F; break;
        case 'I': e = I; break;
        case 'B': e = Other; break;
        case 'c': e = C; arom = true; break;
        case 'n': e = N; arom = true; break;
        case 'o': e = O; arom = true; break;
        case 's': e = S; arom = true; break;
        default: fail(std::string("unexpected character '") + c + "'");
      }
      ++pos_;
    }
    if (m_.n() >= 65535) fail("too many atoms");
    const auto idx = static_cast<uint16_t>(m_.n());
    m_.elem.push_back(e);
    m_.heavy.push_back(1);
    m_.pos.push_back({});
    aromatic_.push_back(arom);
    if (prev_ >= 0) bond(static_cast<uint16_t>(prev_), idx, pending_);
    pending_.reset();
    prev_ = idx;
  }
  void bond(uint16_t a, uint16_t b, std::optional<uint8_t> o) {
    for (std::size_t i = 0; i < m_.ba.size(); ++i)
      if ((m_.ba[i] == a && m_.bb[i] == b) || (m_.ba[i] == b && m_.bb[i] == a)) fail("duplicate bond");
    m_.ba.push_back(a);
    m_.bb.push_back(b);
    m_.order.push_back(o ? *o : (aromatic_[a] && aromatic_[b] ? Aromatic : Single));
  }

  std::string t_;
  std::size_t pos_ = 0;
  int prev_ = -1;
  std::optional<uint8_t> pending_;
  std::vector<int> branches_;
  int ring_atom_[9] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
  std::optional<uint8_t> ring_order_[9];
  std::vector<bool> aromatic_;
  Mol m_;
};

// ---------------------------------------------------------------- hydrogens
int standard_valence(uint8_t e) {  // elements.hpp:47-74
  switch (e) {
    case C: return 4;
    case N: return 3;
    case O: return 2;
    case S: return 2;
    case P: return 3;
    case F: case Cl: case Br: case I: case H: return 1;
    default: return 0;
  }
}
void add_hydrogens(Mol &m) {  // hydrogens.cpp:33-72
  const std::size_t n0 = m.n();
  std::vector<double> used(n0, 0.0);
  std::vector<bool> arom(n0, false);
  for (std::size_t i = 0; i < m.ba.size(); ++i) {
    const double w = m.order[i] == Single ? 1.0 : m.order[i] == Double ? 2.0 : m.order[i] == Triple ? 3.0 : 1.5;
    used[m.ba[i]] += w;
    used[m.bb[i]] += w;
    if (m.order[i] == Aromatic) arom[m.ba[i]] = arom[m.bb[i]] = true;
  }
  for (std::size_t i = 0; i < n0; ++i) {
    if (!m.heavy[i]) continue;
    const int val = standard_valence(m.elem[i]);
    if (val == 0) continue;
    const double free = static_cast<double>(val) - used[i];
    if (free < 0.0 && !arom[i]) throw PrepError("valence of atom " + std::to_string(i) + " exceeded");
    const int nh = std::max(0, static_cast<int>(std::floor(free)));
    for (int h = 0; h < nh; ++h) {
      const auto hi = static_cast<uint16_t>(m.n());
      m.elem.push_back(H);
      m.heavy.push_back(0);
      m.pos.push_back({});
      m.ba.push_back(static_cast<uint16_t>(i));
      m.bb.push_back(hi);
      m.order.push_back(Single);
    }
  }
}

// -------------------------------------------------------------------- embed
double bond_length(uint8_t a, uint8_t b, uint8_t order) {  // embed.cpp:397-412
  auto is = [&](uint8_t x, uint8_t y) { return (a == x && b == y) || (a == y && b == x); };
  double l = 1.5;
  if (is(C, C)) l = 1.54;
  else if (is(C, O)) l = 1.43;
  else if (is(C, N)) l = 1.47;
  else if (is(C, H)) l = 1.09;
  if (order != Single) l *= 0.87;
  return l;
}

V3 any_perpendicular(V3 u) {  // embed.cpp:33-37
  const V3 axis = std::abs(u.x) < 0.9 ? V3{1, 0, 0} : V3{0, 1, 0};
  return normalized(cross(u, axis));
}

class Embedder {  // embed.cpp:82-393
 public:
  explicit Embedder(const Mol &m) : m_(m), adj_(adjacency(m)) {
    const std::size_t n = m.n();
    pos_.assign(n, V3{});
    placed_.assign(n, false);
    parent_.assign(n, -1);
    slots_.assign(n, 0);
    sib_slots_.assign(n, 0);
    find_rings();
    atom_rings_.resize(n);
    for (std::size_t r = 0; r < rings_.size(); ++r)
      for (uint16_t a : rings_[r]) atom_rings_[a].push_back(r);
    ring_center_.resize(rings_.size());
    ring_normal_.resize(rings_.size());
    ring_placed_.assign(rings_.size(), false);
  }

  std::vector<V3> run() {
    if (m_.n() == 0) return pos_;
    placed_[0] = true;
    std::deque<uint16_t> q{0};
    while (!q.empty()) {
      const uint16_t at = q.front();
      q.pop_front();
      for (std::size_t r : atom_rings_[at])
        if (!ring_placed_[r]) place_ring(r, at, q);
      for (auto [nb, bi] : adj_[at]) {
        if (placed_[nb]) continue;
        place_child(at, nb, bi);
        q.push_back(nb);
      }
    }
    return pos_;
  }

 private:
  // Smallest cycle through each non-bridge bond, deduplicated by atom set
  // (embed.cpp:44-80).
  void find_rings() {
    const auto br = bridge_bonds(m_);
    std::set<std::vector<uint16_t>> seen;
    for (std::size_t bi = 0; bi < m_.ba.size(); ++bi) {
      if (br[bi]) continue;
      const uint16_t a = m_.ba[bi], b = m_.bb[bi];
      std::vector<int> par(m_.n(), -2);
      std::deque<uint16_t> fr{a};
      par[a] = -1;
      while (!fr.empty() && par[b] == -2) {
        const uint16_t at = fr.front();
        fr.pop_front();
        for (auto [nb, e] : adj_[at]) {
          if (e == bi || par[nb] != -2) continue;
          par[nb] = at;
          fr.push_back(nb);
        }
      }
      if (par[b] == -2) continue;
      std::vector<uint16_t> cyc;
      for (int at = b; at != -1; at = par[at]) cyc.push_back(static_cast<uint16_t>(at));
      std::reverse(cyc.begin(), cyc.end());
      std::vector<uint16_t> key = cyc;
      std::sort(key.begin(), key.end());
      if (seen.insert(key).second) rings_.push_back(std::move(cyc));
    }
  }

  double ideal_angle(uint16_t at) const {
    for (auto [nb, bi] : adj_[at]) {
      (void)nb;
      if (m_.order[bi] == Double || m_.order[bi] == Aromatic) return 120.0 * kPi / 180.0;
    }
    return 109.5 * kPi / 180.0;
  }

  V3 extend(V3 ref, V3 g, V3 p, double len, double theta, double phi) const {
    const V3 u = normalized(p - g);
    V3 n = cross(g - ref, u);
    if (sqn(n) < 1e-12)
      n = any_perpendicular(u);
    else
      n = normalized(n);
    const V3 mm = cross(n, u);
    const double ct = std::cos(theta), st = std::sin(theta), cp = std::cos(phi), sp = std::sin(phi);
    const V3 inner = cp * mm + sp * n;
    const V3 dir = (-ct) * u + st * inner;
    return p + len * dir;
  }

  int ring_ref(uint16_t p, uint16_t g) const {
    for (std::size_t r : atom_rings_[g]) {
      const auto &cyc = rings_[r];
      const std::size_t at = static_cast<std::size_t>(std::find(cyc.begin(), cyc.end(), g) - cyc.begin());
      const std::size_t k = cyc.size();
      const uint16_t next = cyc[(at + 1) % k];
      const uint16_t prev = cyc[(at + k - 1) % k];
      if (next == p && placed_[prev]) return prev;
      if (prev == p && placed_[next]) return next;
    }
    return -1;
  }

  void place_child(uint16_t p, uint16_t c, std::size_t bi) {
    const double len = bond_length(m_.elem[m_.ba[bi]], m_.elem[m_.bb[bi]], m_.order[bi]);
    const double theta = ideal_angle(p);
    const int slot = slots_[p]++;
    int g = parent_[p];
    if (g < 0 || !placed_[static_cast<std::size_t>(g)]) {
      g = -1;
      for (auto [nb, e] : adj_[p]) {
        (void)e;
        if (nb != c && placed_[nb]) {
          g = nb;
          break;
        }
      }
    }
    if (g < 0) {
      if (slot == 0)
        pos_[c] = pos_[p] + len * V3{1.0, 0.0, 0.0};
      else
        pos_[c] = pos_[p] + len * V3{std::cos(theta), std::sin(theta), 0.0};
      placed_[c] = true;
      parent_[c] = p;
      return;
    }
    const auto gu = static_cast<uint16_t>(g);
    bool sibling = false;
    int ref_atom = ring_ref(p, gu);
    if (ref_atom < 0 && parent_[gu] >= 0 && placed_[static_cast<std::size_t>(parent_[gu])] && parent_[gu] != p)
      ref_atom = parent_[gu];
    if (ref_atom < 0)
      for (auto [nb, e] : adj_[gu]) {
        (void)e;
        if (nb != p && placed_[nb]) {
          ref_atom = nb;
          break;
        }
      }
    if (ref_atom < 0)
      for (auto [nb, e] : adj_[p]) {
        (void)e;
        if (nb != c && nb != gu && placed_[nb]) {
          ref_atom = nb;
          sibling = true;
          break;
        }
      }
    const V3 ref = ref_atom >= 0 ? pos_[static_cast<std::size_t>(ref_atom)]
                                 : pos_[gu] + any_perpendicular(pos_[p] - pos_[gu]);
    static constexpr double kChild[6] = {180.0, 60.0, 300.0, 120.0, 240.0, 0.0};
    static constexpr double kSibling[6] = {120.0, 240.0, 60.0, 300.0, 0.0, 180.0};
    const double phi = sibling ? kSibling[std::min(sib_slots_[p]++, 5)] * kPi / 180.0
                               : kChild[std::min(slot, 5)] * kPi / 180.0;
    pos_[c] = extend(ref, pos_[gu], pos_[p], len, theta, phi);
    placed_[c] = true;
    parent_[c] = p;
  }

  void place_ring(std::size_t ri, uint16_t entry, std::deque<uint16_t> &q) {
    const auto &ring = rings_[ri];
    const std::size_t k = ring.size();
    ring_placed_[ri] = true;
    std::size_t edge = k;
    for (std::size_t j = 0; j < k; ++j) {
      const uint16_t u = ring[j], v = ring[(j + 1) % k];
      if (!placed_[u] || !placed_[v]) continue;
      if (edge == k) edge = j;
      if (u == entry || v == entry) {
        edge = j;
        break;
      }
    }
    std::vector<uint16_t> order(k);
    if (edge < k)
      ring_on_edge(ri, edge, order);
    else
      ring_fresh(ri, entry, order);
    for (std::size_t j = 1; j < k; ++j) {
      const uint16_t at = order[j];
      if (parent_[at] < 0 && at != 0) parent_[at] = order[j - 1];
    }
    for (std::size_t j = 0; j < k; ++j)
      if (just_placed_.count(order[j])) q.push_back(order[j]);
    just_placed_.clear();
  }

  double mean_ring_bond(const std::vector<uint16_t> &ring) const {
    const std::size_t k = ring.size();
    double total = 0.0;
    for (std::size_t j = 0; j < k; ++j) {
      const uint16_t u = ring[j], v = ring[(j + 1) % k];
      uint8_t o = Single;
      for (auto [nb, bi] : adj_[u])
        if (nb == v) o = m_.order[bi];
      total += bond_length(m_.elem[u], m_.elem[v], o);
    }
    return total / static_cast<double>(k);
  }

  void ring_fresh(std::size_t ri, uint16_t entry, std::vector<uint16_t> &order) {
    const auto &ring = rings_[ri];
    const std::size_t k = ring.size();
    const std::size_t shift = static_cast<std::size_t>(std::find(ring.begin(), ring.end(), entry) - ring.begin());
    for (std::size_t j = 0; j < k; ++j) order[j] = ring[(shift + j) % k];
    const double side = mean_ring_bond(ring);
    const double radius = side / (2.0 * std::sin(kPi / static_cast<double>(k)));
    V3 e1{1.0, 0.0, 0.0};
    if (parent_[entry] >= 0 && placed_[static_cast<std::size_t>(parent_[entry])]) {
      const V3 away = pos_[entry] - pos_[static_cast<std::size_t>(parent_[entry])];
      if (sqn(away) > 1e-12) e1 = normalized(away);
    }
    const V3 e2 = any_perpendicular(e1);
    const V3 center = pos_[entry] + radius * e1;
    for (std::size_t j = 0; j < k; ++j) {
      const uint16_t at = order[j];
      if (placed_[at]) continue;
      const double ang = kPi + 2.0 * kPi * static_cast<double>(j) / static_cast<double>(k);
      const V3 dir = std::cos(ang) * e1 + std::sin(ang) * e2;
      pos_[at] = center + radius * dir;
      placed_[at] = true;
      just_placed_.insert(at);
    }
    ring_center_[ri] = center;
    ring_normal_[ri] = normalized(cross(e1, e2));
  }

  void ring_on_edge(std::size_t ri, std::size_t edge, std::vector<uint16_t> &order) {
    const auto &ring = rings_[ri];
    const std::size_t k = ring.size();
    const uint16_t u = ring[edge], v = ring[(edge + 1) % k];
    for (std::size_t j = 0; j < k; ++j) order[j] = ring[(edge + k - j) % k];
    V3 normal = any_perpendicular(pos_[v] - pos_[u]);
    V3 prev_center = 0.5 * (pos_[u] + pos_[v]) + any_perpendicular(pos_[v] - pos_[u]);
    for (std::size_t r = 0; r < rings_.size(); ++r) {
      if (!ring_placed_[r] || r == ri) continue;
      const auto &ar = rings_[r];
      const bool hu = std::find(ar.begin(), ar.end(), u) != ar.end();
      const bool hv = std::find(ar.begin(), ar.end(), v) != ar.end();
      if (hu && hv) {
        normal = ring_normal_[r];
        prev_center = ring_center_[r];
        break;
      }
    }
    const V3 mid = 0.5 * (pos_[u] + pos_[v]);
    const V3 axis = normalized(pos_[v] - pos_[u]);
    const double side = norm(pos_[v] - pos_[u]);
    const double radius = side / (2.0 * std::sin(kPi / static_cast<double>(k)));
    V3 w = normalized(cross(normal, axis));
    if (dot(w, mid - prev_center) < 0.0) w = -w;
    const V3 center = mid + (radius * std::cos(kPi / static_cast<double>(k))) * w;
    const V3 ex = normalized(pos_[u] - center);
    V3 ey = pos_[v] - center;
    ey = ey - dot(ey, ex) * ex;
    if (sqn(ey) < 1e-12) ey = cross(normal, ex);
    ey = -normalized(ey);
    for (std::size_t j = 1; j + 1 < k; ++j) {
      const uint16_t at = order[j];
      if (placed_[at]) continue;
      const double ang = 2.0 * kPi * static_cast<double>(j) / static_cast<double>(k);
      const V3 dir = std::cos(ang) * ex + std::sin(ang) * ey;
      pos_[at] = center + radius * dir;
      placed_[at] = true;
      just_placed_.insert(at);
    }
    ring_center_[ri] = center;
    ring_normal_[ri] = normalized(cross(ex, ey));
  }

  const Mol &m_;
  Adj adj_;
  std::vector<std::vector<uint16_t>> rings_;
  std::vector<V3> pos_;
  std::vector<bool> placed_;
  std::vector<int> parent_, slots_, sib_slots_;
  std::vector<std::vector<std::size_t>> atom_rings_;
  std::vector<V3> ring_center_, ring_normal_;
  std::vector<bool> ring_placed_;
  std::set<uint16_t> just_placed_;
};

Mol prepare(const std::string &smiles, int mode) {
  Mol m = SmilesParser(smiles).run();
  if (mode == 2) {
    detect_torsions(m);
    return m;
  }
  if (mode == 3) {  // embed_3d of the heavy-atom graph (the reference tests' fixtures)
    m.pos = Embedder(m).run();
    detect_torsions(m);
    return m;
  }
  add_hydrogens(m);
  if (!connected(m)) throw PrepError("cannot embed a disconnected graph");
  m.pos = Embedder(m).run();
  detect_torsions(m);
  return m;
}

}  // namespace vsprep

namespace vsprep_internal {
// Heavy-atom and rotatable-bond counts of a SMILES as prepare_ligand would
// see them (hydrogens do not change which bonds qualify, ligand.cpp:126-139);
// false when the SMILES cannot be parsed or hydrogenated.
bool counts(const std::string &smiles, int *heavy, int *rot) {
  try {
    vsprep::Mol m = vsprep::SmilesParser(smiles).run();
    *heavy = static_cast<int>(m.n());
    vsprep::Mol h = m;
    vsprep::add_hydrogens(h);
    vsprep::detect_torsions(m);
    *rot = static_cast<int>(m.tors.size());
    return true;
  } catch (const std::exception &) {
    return false;
  }
}
}  // namespace vsprep_internal

// =================================================================== C API
#include "ligand_set.hpp"

extern "C" {

vs_status vs_prep_smiles_batch(int32_t n, const char *const *smiles, int32_t mode, int32_t nthreads,
                               vs_ligand_set **out) {
  if (n < 0 || !out || mode < 1 || mode > 3) return VS_ERR_INVALID_ARGUMENT;
  std::vector<vsprep::Mol> mols(static_cast<std::size_t>(n));
  auto *set = new vs_ligand_set;
  set->status.assign(static_cast<std::size_t>(n), 0);
  set->errors.assign(static_cast<std::size_t>(n), std::string());
  set->names.resize(static_cast<std::size_t>(n));
  for (int32_t i = 0; i < n; ++i) set->names[static_cast<std::size_t>(i)] = smiles[i] ? smiles[i] : "";
  std::atomic<int> next{0};
  auto work = [&] {
    for (int i = next++; i < n; i = next++) {
      try {
        mols[i] = vsprep::prepare(smiles[i], mode);
      } catch (const std::exception &e) {
        set->status[i] = 1;
        set->errors[i] = e.what();
        mols[i] = vsprep::Mol{};
      }
    }
  };
  const int nt = std::max(1, std::min<int>(nthreads, n));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto &th : pool) th.join();

  set->atom_off.push_back(0);
  set->bond_off.push_back(0);
  set->tors_off.push_back(0);
  set->right_off.push_back(0);
  for (const auto &m : mols) {
    for (std::size_t a = 0; a < m.n(); ++a) {
      set->xyz.push_back(m.pos[a].x);
      set->xyz.push_back(m.pos[a].y);
      set->xyz.push_back(m.pos[a].z);
    }
    set->elem.insert(set->elem.end(), m.elem.begin(), m.elem.end());
    set->heavy.insert(set->heavy.end(), m.heavy.begin(), m.heavy.end());
    set->ba.insert(set->ba.end(), m.ba.begin(), m.ba.end());
    set->bb.insert(set->bb.end(), m.bb.begin(), m.bb.end());
    set->border.insert(set->border.end(), m.order.begin(), m.order.end());
    for (std::size_t t = 0; t < m.tors.size(); ++t) {
      set->tbond.push_back(m.tors[t]);
      set->ratoms.insert(set->ratoms.end(), m.right[t].begin(), m.right[t].end());
      set->right_off.push_back(static_cast<int32_t>(set->ratoms.size()));
    }
    set->atom_off.push_back(static_cast<int32_t>(set->elem.size()));
    set->bond_off.push_back(static_cast<int32_t>(set->ba.size()));
    set->tors_off.push_back(static_cast<int32_t>(set->tbond.size()));
  }
  *out = set;
  return VS_OK;
}

vs_status vs_ligand_set_view(const vs_ligand_set *s, vs_ligand_batch *v, const int32_t **status) {
  if (!s || !v) return VS_ERR_INVALID_ARGUMENT;
  v->n_ligands = static_cast<int32_t>(s->status.size());
  v->atom_offset = s->atom_off.data();
  v->xyz = s->xyz.data();
  v->element = s->elem.data();
  v->is_heavy = s->heavy.data();
  v->bond_offset = s->bond_off.data();
  v->bond_a = s->ba.data();
  v->bond_b = s->bb.data();
  v->bond_order = s->border.data();
  v->torsion_offset = s->tors_off.data();
  v->torsion_bond = s->tbond.data();
  v->right_offset = s->right_off.data();
  v->right_atoms = s->ratoms.data();
  if (status) *status = s->status.data();
  return VS_OK;
}

const char *vs_ligand_set_error(const vs_ligand_set *s, int32_t i) {
  if (!s || i < 0 || static_cast<std::size_t>(i) >= s->errors.size()) return "";
  return s->errors[static_cast<std::size_t>(i)].c_str();
}

const char *vs_ligand_set_name(const vs_ligand_set *s, int32_t i) {
  if (!s || i < 0 || static_cast<std::size_t>(i) >= s->names.size()) return "";
  return s->names[static_cast<std::size_t>(i)].c_str();
}

void vs_ligand_set_free(vs_ligand_set *s) { delete s; }

static vsprep::Mol mol_of(const vs_ligand_batch *b, int32_t i) {
  vsprep::Mol m;
  for (int a = b->atom_offset[i]; a < b->atom_offset[i + 1]; ++a) {
    m.elem.push_back(b->element[a]);
    m.heavy.push_back(b->is_heavy[a] ? 1 : 0);
    m.pos.push_back({b->xyz ? b->xyz[3 * a] : 0.0, b->xyz ? b->xyz[3 * a + 1] : 0.0, b->xyz ? b->xyz[3 * a + 2] : 0.0});
  }
  for (int k = b->bond_offset[i]; k < b->bond_offset[i + 1]; ++k) {
    m.ba.push_back(b->bond_a[k]);
    m.bb.push_back(b->bond_b[k]);
    m.order.push_back(b->bond_order ? b->bond_order[k] : 1);
  }
  return m;
}

int32_t vs_detect_torsions(const vs_ligand_batch *b, int32_t i, uint16_t *bonds_out, uint8_t *right_mask_out) {
  if (!b || i < 0 || i >= b->n_ligands) return -1;
  vsprep::Mol m = mol_of(b, i);
  for (std::size_t k = 0; k < m.ba.size(); ++k)
    if (m.ba[k] >= m.n() || m.bb[k] >= m.n()) return -1;
  vsprep::detect_torsions(m);
  for (std::size_t t = 0; t < m.tors.size(); ++t) {
    if (bonds_out) bonds_out[t] = m.tors[t];
    if (right_mask_out) {
      std::memset(right_mask_out + t * m.n(), 0, m.n());
      for (uint16_t a : m.right[t]) right_mask_out[t * m.n() + a] = 1;
    }
  }
  return static_cast<int32_t>(m.tors.size());
}

int32_t vs_bridge_bonds(const vs_ligand_batch *b, int32_t i, uint8_t *bridge_out) {
  if (!b || i < 0 || i >= b->n_ligands) return -1;
  vsprep::Mol m = mol_of(b, i);
  for (std::size_t k = 0; k < m.ba.size(); ++k)
    if (m.ba[k] >= m.n() || m.bb[k] >= m.n()) return -1;
  const auto br = vsprep::bridge_bonds(m);
  for (std::size_t k = 0; k < br.size(); ++k) bridge_out[k] = br[k];
  return static_cast<int32_t>(br.size());
}

}  // extern "C"
