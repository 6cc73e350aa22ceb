// Campaign ranking merge (include/vs_rank.h vs_merge_rankings): the order of
// the reference's cmd_merge (merge.cpp:81-147) -- every row of every rank's
// score file, parsed back with from_chars, stable-sorted by (score desc,
// SMILES asc), written as the original row text -- at 10^7..10^8 rows.
//
// B200-host design: rows are parsed in parallel into 24-byte keys (score,
// view of the SMILES, original position), sorted as independent runs on all
// host threads (std::stable_sort per run), then combined with a k-way heap
// merge whose tie-break is the run index: runs are contiguous slices of the
// concatenated input in file order, so the result is exactly the
// concatenation's stable sort.  Optionally only the first top_k rows.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstring>
#include <queue>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "vs_rank.h"

extern "C" vs_status vs_internal_fail(vs_status s, const char *msg);

namespace {

struct Row {
  double score;
  const char *text;  // row start
  uint32_t smiles_len;
  uint32_t text_len;  // without the newline
};

// a before b in the ranking (merge.cpp:131-135)
inline bool before(const Row &a, const Row &b) {
  if (a.score != b.score) return a.score > b.score;
  const int c = std::memcmp(a.text, b.text, std::min(a.smiles_len, b.smiles_len));
  if (c != 0) return c < 0;
  return a.smiles_len < b.smiles_len;
}

}  // namespace

extern "C" vs_status vs_merge_rankings(const char *const *texts, const int64_t *lens, int32_t n_files, int64_t top_k,
                                       int32_t threads, vs_write_fn write, void *user, uint64_t *rows_out) {
  if ((n_files > 0 && (!texts || !lens)) || !write) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
  // ---- line boundaries per file (file order = the reference's rank order)
  struct Span {
    int file;
    int64_t begin, end;  // byte range of whole lines
  };
  std::vector<Span> spans;
  int64_t total_bytes = 0;
  for (int f = 0; f < n_files; ++f) total_bytes += lens[f];
  const int64_t target = std::max<int64_t>(total_bytes / (4 * threads) + 1, 1 << 16);
  for (int f = 0; f < n_files; ++f) {
    int64_t b = 0;
    while (b < lens[f]) {
      int64_t e = std::min(lens[f], b + target);
      while (e < lens[f] && texts[f][e - 1] != '\n') ++e;  // cut after a newline
      spans.push_back({f, b, e});
      b = e;
    }
  }
  // ---- parse + sort each span as a run, in parallel
  std::vector<std::vector<Row>> runs(spans.size());
  std::vector<std::string> errs(spans.size());
  auto work = [&](size_t i) {
    const Span &sp = spans[i];
    const char *t = texts[sp.file];
    std::vector<Row> &rs = runs[i];
    int64_t at = sp.begin;
    while (at < sp.end) {
      const char *nl = static_cast<const char *>(std::memchr(t + at, '\n', static_cast<size_t>(sp.end - at)));
      const int64_t e = nl ? nl - t : sp.end;
      if (e > at) {
        const char *line = t + at;
        const size_t len = static_cast<size_t>(e - at);
        const char *tab = static_cast<const char *>(std::memchr(line, '\t', len));
        if (!tab) {
          errs[i] = "score row without a tab";
          return;
        }
        Row r;
        const auto res = std::from_chars(tab + 1, line + len, r.score);
        if (res.ec != std::errc() || res.ptr != line + len) {
          errs[i] = "bad score '" + std::string(tab + 1, line + len) + "'";
          return;
        }
        r.text = line;
        r.smiles_len = static_cast<uint32_t>(tab - line);
        r.text_len = static_cast<uint32_t>(len);
        rs.push_back(r);
      }
      at = e + 1;
    }
    std::stable_sort(rs.begin(), rs.end(), before);
  };
  {
    std::vector<std::thread> pool;
    std::atomic<size_t> next{0};
    for (int k = 0; k < threads; ++k)
      pool.emplace_back([&] {
        for (size_t i; (i = next.fetch_add(1)) < spans.size();) work(i);
      });
    for (auto &th : pool) th.join();
  }
  for (const std::string &e : errs)
    if (!e.empty()) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, e.c_str());
  // ---- k-way merge, run index breaks exact ties (stability)
  auto later = [&](const std::pair<size_t, size_t> &a, const std::pair<size_t, size_t> &b) {
    const Row &ra = runs[a.first][a.second], &rb = runs[b.first][b.second];
    if (before(ra, rb)) return false;
    if (before(rb, ra)) return true;
    return a.first > b.first;
  };
  std::priority_queue<std::pair<size_t, size_t>, std::vector<std::pair<size_t, size_t>>, decltype(later)> heap(later);
  for (size_t i = 0; i < runs.size(); ++i)
    if (!runs[i].empty()) heap.push({i, 0});
  std::string buf;
  buf.reserve(8 << 20);
  uint64_t rows = 0;
  const uint64_t limit = top_k >= 0 ? static_cast<uint64_t>(top_k) : ~0ull;
  while (!heap.empty() && rows < limit) {
    const auto [ri, pos] = heap.top();
    heap.pop();
    const Row &r = runs[ri][pos];
    buf.append(r.text, r.text_len);
    buf += '\n';
    ++rows;
    if (pos + 1 < runs[ri].size()) heap.push({ri, pos + 1});
    if (buf.size() >= (8u << 20)) {
      if (write(user, buf.data(), static_cast<int64_t>(buf.size())) != 0)
        return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "write failed");
      buf.clear();
    }
  }
  if (!buf.empty() && write(user, buf.data(), static_cast<int64_t>(buf.size())) != 0)
    return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "write failed");
  if (rows_out) *rows_out = rows;
  return VS_OK;
}
