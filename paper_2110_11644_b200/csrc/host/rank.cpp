// One rank of the screening pipeline with CUDA workers (include/vs_rank.h):
// the reference's run_rank (pipeline.cpp:297-398) with the docker stage
// (pipeline.cpp:206-244) replaced by W CUDA workers per GPU that each dock a
// batch of raw records per vs_dock_records call (GPU decode + dock).
//
// Threads: the calling thread frames records (reader + splitter roles) and
// writes rows (writer role) in record order; the CUDA workers run the
// batches.  Framing is speculative: a batch is framed assuming every record
// decodes (next scan position = record end).  When the GPU reports a record
// that fails to decode, that record is a records_skipped, everything framed
// after it (the rest of its batch and every later batch in flight) is
// discarded, and framing restarts two bytes after its marker -- exactly the
// splitter's resynchronisation (pipeline.cpp:180-185) -- so the set and the
// order of docked records are the reference's.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "vs_codec.h"
#include "vs_dock.h"
#include "vs_rank.h"

extern "C" vs_status vs_internal_fail(vs_status s, const char *msg);

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

constexpr uint8_t kMark0 = 0xD0, kMark1 = 0xC5;  // record sync marker (binary_codec.hpp)

enum class Scan { Found, NeedMore, End };

bool mark_at(const uint8_t *b, size_t n, size_t at) { return at + 2 <= n && b[at] == kMark0 && b[at + 1] == kMark1; }

uint32_t le32(const uint8_t *p) {
  return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
         static_cast<uint32_t>(p[3]) << 24;
}

// Is the marker at `at` a record start?  Its length chain must land, for two
// hops, on another marker or exactly on the end of the data
// (binary_codec.cpp:89-111).  `final`: no more data will arrive.
Scan chain(const uint8_t *b, size_t n, size_t at, bool final) {
  size_t c = at;
  for (int hop = 0; hop < 2; ++hop) {
    if (c + 2 <= n && !mark_at(b, n, c)) return Scan::End;
    if (c + 6 > n) return final ? Scan::End : Scan::NeedMore;
    const size_t next = c + 6 + le32(b + c + 2);
    if (next > n) return final ? Scan::End : Scan::NeedMore;
    if (next == n) return Scan::Found;
    c = next;
  }
  if (c + 2 > n) return final ? Scan::End : Scan::NeedMore;
  return mark_at(b, n, c) ? Scan::Found : Scan::End;
}

// First record start at or after `from` (scan_record_start,
// binary_codec.cpp:224-238): a NeedMore candidate stops the scan.
Scan scan(const uint8_t *b, size_t n, size_t from, bool final, size_t *at) {
  for (size_t a = from; a + 2 <= n; ++a) {
    if (b[a] != kMark0 || b[a + 1] != kMark1) continue;
    const Scan r = chain(b, n, a, final);
    if (r == Scan::End) continue;  // false marker
    *at = a;
    return r;
  }
  return Scan::End;
}

struct Batch {
  std::vector<uint64_t> file_off;  // record starts in the source
  std::vector<int64_t> offs;       // record starts in `bytes`
  uint8_t *bytes = nullptr;        // pinned staging
  size_t cap = 0, used = 0;
  std::vector<vs_dock_result> res;
  std::vector<int32_t> rec_status;
  vs_status rc = VS_OK;
  std::string err;
  bool done = false;
  bool discard = false;
};

struct Worker {
  vs_context *ctx = nullptr;
  vs_pocket *pocket = nullptr;
  std::thread th;
};

struct Pool {
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  std::deque<Batch *> jobs;
  bool quit = false;
  double busy = 0.0;
};

void worker_loop(Worker *w, Pool *pool, const vs_scoring_config *cfg) {
  while (true) {
    Batch *b = nullptr;
    {
      std::unique_lock<std::mutex> lk(pool->mu);
      pool->cv_job.wait(lk, [&] { return pool->quit || !pool->jobs.empty(); });
      if (pool->jobs.empty()) return;
      b = pool->jobs.front();
      pool->jobs.pop_front();
    }
    const auto t0 = Clock::now();
    const int32_t n = static_cast<int32_t>(b->offs.size());
    b->res.assign(static_cast<size_t>(n), vs_dock_result{});
    b->rec_status.assign(static_cast<size_t>(n), 0);
    const vs_pocket *pk = w->pocket;
    b->rc = n ? vs_dock_records(w->ctx, &pk, 1, b->bytes, static_cast<int64_t>(b->used), b->offs.data(), n, cfg,
                                b->res.data(), b->rec_status.data())
              : VS_OK;
    if (b->rc != VS_OK) b->err = vs_last_error_message();
    const double dt = since(t0);
    {
      std::lock_guard<std::mutex> lk(pool->mu);
      b->done = true;
      pool->busy += dt;
    }
    pool->cv_done.notify_all();
  }
}

// format_row (pipeline.cpp:47-62): SMILES, tab, the score in fixed notation
// with 4 decimals (std::to_chars), newline.
void append_row(std::string &out, const char *smiles, size_t len, double score) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, score, std::chars_format::fixed, 4);
  out.append(smiles, len);
  out += '\t';
  out.append(buf, r.ptr);
  out += '\n';
}

}  // namespace

extern "C" void vs_rank_config_default(vs_rank_config *rc) {
  if (!rc) return;
  rc->n_devices = 0;
  rc->devices = nullptr;
  rc->workers_per_device = 2;
  rc->batch_records = 32768;
  rc->chunk_bytes = 1 << 20;
  rc->writer_buffer_bytes = 4 << 20;
}

extern "C" vs_status vs_run_rank(uint64_t source_size, vs_read_fn read, void *read_user, uint64_t slab_start,
                                 uint64_t slab_stop, const vs_pocket_desc *pocket, const vs_scoring_config *cfg,
                                 const vs_rank_config *rc_in, vs_write_fn write, void *write_user,
                                 vs_rank_stats *stats) {
  if (!read || !write || !pocket || !cfg) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "null argument");
  vs_rank_config cf;
  vs_rank_config_default(&cf);
  if (rc_in) cf = *rc_in;
  if (cf.workers_per_device < 1) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "need at least one worker");
  if (cf.chunk_bytes <= 0) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "chunk size must be positive");
  if (cf.batch_records <= 0) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "batch size must be positive");
  if (cf.writer_buffer_bytes <= 0) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "writer buffer must be positive");
  if (slab_start > slab_stop) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "slab start past slab stop");
  if (slab_stop > source_size) return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "slab exceeds the input size");
  const auto wall0 = Clock::now();
  vs_rank_stats st{};

  // ---- CUDA workers: W per device, each with its own context and pocket copy
  std::vector<int> devs;
  if (cf.devices && cf.n_devices <= 0)
    return vs_internal_fail(VS_ERR_INVALID_ARGUMENT, "a device list needs n_devices > 0");
  const int ndev = cf.n_devices > 0 ? cf.n_devices : vs_device_count();
  if (ndev <= 0) return vs_internal_fail(VS_ERR_NO_DEVICE, "no CUDA device");
  for (int i = 0; i < ndev; ++i) devs.push_back(cf.devices ? cf.devices[i] : i);
  Pool pool;
  std::vector<std::unique_ptr<Worker>> workers;
  vs_status rc_setup = VS_OK;
  for (int d : devs)
    for (int k = 0; k < cf.workers_per_device && rc_setup == VS_OK; ++k) {
      auto w = std::make_unique<Worker>();
      rc_setup = vs_context_create(d, &w->ctx);
      if (rc_setup == VS_OK) rc_setup = vs_pocket_create(w->ctx, pocket, &w->pocket);
      workers.push_back(std::move(w));
    }
  auto shutdown = [&] {
    {
      std::lock_guard<std::mutex> lk(pool.mu);
      pool.quit = true;
    }
    pool.cv_job.notify_all();
    for (auto &w : workers) {
      if (w->th.joinable()) w->th.join();
      if (w->pocket) vs_pocket_destroy(w->pocket);
      if (w->ctx) vs_context_destroy(w->ctx);
    }
  };
  if (rc_setup != VS_OK) {
    const std::string msg = vs_last_error_message();
    shutdown();
    return vs_internal_fail(rc_setup, msg.c_str());
  }
  for (auto &w : workers) w->th = std::thread(worker_loop, w.get(), &pool, cfg);
  st.workers = static_cast<int32_t>(workers.size());

  // ---- batches: two in flight per worker, pinned staging owned here
  const size_t inflight_max = 2 * workers.size();
  std::vector<std::unique_ptr<Batch>> slots(inflight_max);
  std::deque<Batch *> free_b, flight;
  vs_status rc = VS_OK;
  std::string err;
  for (auto &b : slots) {
    b = std::make_unique<Batch>();
    free_b.push_back(b.get());
  }
  auto release = [&] {
    for (auto &b : slots)
      if (b->bytes) vs_host_free(b->bytes);
  };

  // ---- framing window over the source: bytes [base, base + win.size())
  std::vector<uint8_t> win;
  uint64_t base = slab_start, next_read = slab_start;
  size_t from = 0;              // scan position in `win`
  bool eof = slab_start >= slab_stop;  // an empty slab owns no record starts
  bool framing_done = eof;
  double t_read = 0.0, t_split = 0.0, t_write = 0.0;
  auto read_chunk = [&]() -> bool {
    if (next_read >= source_size) {
      eof = true;
      return false;
    }
    const auto t0 = Clock::now();
    const size_t want = static_cast<size_t>(std::min<uint64_t>(cf.chunk_bytes, source_size - next_read));
    const size_t old = win.size();
    win.resize(old + want);
    const int64_t got = read(read_user, next_read, win.data() + old, static_cast<int64_t>(want));
    t_read += since(t0);
    if (got <= 0) {
      win.resize(old);
      eof = true;
      if (got < 0) {
        rc = VS_ERR_INVALID_ARGUMENT;
        err = "read failed";
      }
      return false;
    }
    win.resize(old + static_cast<size_t>(got));
    next_read += static_cast<uint64_t>(got);
    ++st.chunks_read;
    st.bytes_read += static_cast<uint64_t>(got);
    return true;
  };

  // Frame up to batch_records records into b (false: nothing framed).
  auto frame = [&](Batch *b) {
    const auto t0 = Clock::now();
    b->file_off.clear();
    b->offs.clear();
    b->used = 0;
    b->done = b->discard = false;
    while (!framing_done && static_cast<int32_t>(b->offs.size()) < cf.batch_records) {
      size_t at = 0;
      const Scan r = scan(win.data(), win.size(), from, eof, &at);
      if (r == Scan::NeedMore || (r == Scan::End && !eof)) {
        // NeedMore: the candidate needs the next chunk; End before the final
        // chunk: only the last byte can still start a marker
        from = r == Scan::NeedMore ? at : (win.empty() ? 0 : win.size() - 1);
        read_chunk();
        if (rc != VS_OK) break;
        continue;
      }
      if (r == Scan::End) {
        // final data: a clean tail, or markers that never frame
        // (find_record_start, binary_codec.cpp:240-252)
        for (size_t a = from; a + 2 <= win.size(); ++a)
          if (win[a] == kMark0 && win[a + 1] == kMark1) {
            rc = VS_ERR_INVALID_ARGUMENT;
            err = "corrupt record stream: sync marker without valid chain";
            break;
          }
        framing_done = true;
        break;
      }
      if (base + at >= slab_stop) {  // the next rank's record
        framing_done = true;
        break;
      }
      const size_t len = 6 + static_cast<size_t>(le32(win.data() + at + 2));
      if (b->used + len > b->cap) {
        if (!b->offs.empty()) break;  // full: this record starts the next batch
        const size_t cap = std::max<size_t>(len, static_cast<size_t>(cf.batch_records) * 512);
        if (b->bytes) vs_host_free(b->bytes);
        void *p = nullptr;
        const vs_status s = vs_host_alloc(cap, &p);
        if (s != VS_OK) {
          rc = s;
          err = vs_last_error_message();
          framing_done = true;
          break;
        }
        b->bytes = static_cast<uint8_t *>(p);
        b->cap = cap;
      }
      std::memcpy(b->bytes + b->used, win.data() + at, len);
      b->offs.push_back(static_cast<int64_t>(b->used));
      b->file_off.push_back(base + at);
      b->used += len;
      from = at + len;  // speculative: the record decodes
    }
    t_split += since(t0);
    return !b->offs.empty();
  };

  // Drop window bytes no in-flight record (nor a resync) can need.
  auto trim = [&] {
    uint64_t keep = base + from;
    for (Batch *b : flight)
      if (!b->file_off.empty()) keep = std::min(keep, b->file_off.front());
    if (keep > base + (1u << 20) && keep - base <= win.size()) {
      const size_t drop = static_cast<size_t>(keep - base);
      win.erase(win.begin(), win.begin() + static_cast<std::ptrdiff_t>(drop));
      base += drop;
      from -= drop;
    }
  };

  std::string out;
  out.reserve(static_cast<size_t>(cf.writer_buffer_bytes) + 256);
  auto flush = [&] {
    if (out.empty()) return;
    const auto t0 = Clock::now();
    if (write(write_user, out.data(), static_cast<int64_t>(out.size())) != 0 && rc == VS_OK) {
      rc = VS_ERR_INVALID_ARGUMENT;
      err = "write failed";
    }
    ++st.write_calls;
    st.bytes_written += out.size();
    out.clear();
    t_write += since(t0);
  };

  while (rc == VS_OK) {
    // keep the workers fed
    while (rc == VS_OK && !framing_done && !free_b.empty()) {
      Batch *b = free_b.front();
      if (!frame(b)) break;
      free_b.pop_front();
      flight.push_back(b);
      {
        std::lock_guard<std::mutex> lk(pool.mu);
        pool.jobs.push_back(b);
      }
      pool.cv_job.notify_one();
      ++st.batches;
    }
    if (flight.empty()) break;
    // retire the oldest batch, in record order
    Batch *b = flight.front();
    {
      std::unique_lock<std::mutex> lk(pool.mu);
      pool.cv_done.wait(lk, [&] { return b->done; });
    }
    flight.pop_front();
    free_b.push_back(b);
    if (b->discard) continue;
    if (b->rc != VS_OK) {
      rc = b->rc;
      err = b->err;
      break;
    }
    const auto t0 = Clock::now();
    size_t bad = b->offs.size();
    for (size_t i = 0; i < b->offs.size(); ++i) {
      const vs_dock_result &r = b->res[i];
      if (r.status == VS_LIG_BAD_RECORD) {
        bad = i;
        break;
      }
      if (r.status != VS_LIG_OK || !std::isfinite(r.best_score)) {
        ++st.dock_errors;
        continue;
      }
      const uint8_t *rec = b->bytes + b->offs[i];
      const size_t name_len = static_cast<size_t>(rec[6]) | static_cast<size_t>(rec[7]) << 8;
      append_row(out, reinterpret_cast<const char *>(rec + 8), name_len, r.best_score);
      ++st.rows_written;
      if (out.size() >= static_cast<size_t>(cf.writer_buffer_bytes)) flush();
    }
    t_write += since(t0);
    if (bad < b->offs.size()) {
      // a framed record that does not decode: skip it, void what was framed
      // after it, and rescan two bytes past its marker (pipeline.cpp:180-185)
      ++st.records_skipped;
      ++st.resyncs;
      for (Batch *o : flight) o->discard = true;
      from = static_cast<size_t>(b->file_off[bad] - base) + 2;
      framing_done = false;
    }
    trim();
  }
  // drain (error paths leave batches in flight)
  for (Batch *b : flight) {
    std::unique_lock<std::mutex> lk(pool.mu);
    pool.cv_done.wait(lk, [&] { return b->done; });
  }
  flush();
  shutdown();
  release();
  st.ligands_docked = st.rows_written;
  st.wall_seconds = since(wall0);
  st.reader_busy_seconds = t_read;
  st.splitter_busy_seconds = t_split;
  st.docker_busy_seconds = pool.busy;
  st.writer_busy_seconds = t_write;
  if (stats) *stats = st;
  if (rc != VS_OK) return vs_internal_fail(rc, err.c_str());
  return VS_OK;
}
