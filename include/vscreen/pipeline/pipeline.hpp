// Drop-in for the reference's rank pipeline (pipeline.hpp:16-160), B200
// build: run_rank keeps the reference's slab rule, record framing and
// resynchronisation, counters and row format, with the docker stage replaced
// by CUDA workers (include/vs_rank.h; records decoded and docked on the GPU
// in batches, several workers per GPU on their own streams).
//   * PipelineConfig::workers: the total count is the number of CUDA workers
//     per GPU (every visible GPU, or the calling thread's
//     vscreen::b200::use_device() when set); synthetic_slowdown must be >= 1
//     and is otherwise ignored (it emulates slow CPU workers).
//   * chunk / queue capacities keep their meaning where one exists
//     (chunk_bytes, writer_buffer_bytes); rows are written in record order.
//   * docker_worker (pipeline.cpp:206-244) is the batch-pulling CUDA worker:
//     it drains whatever WorkItems are queued (up to 65,536) into one
//     dock_and_score_batch call.  The other stage functions (stage_reader,
//     stage_splitter, stage_writer) are not part of this build: run_rank
//     fuses them around GPU record decode.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "vscreen/dockengine/pose.hpp"
#include "vscreen/molmodel/ligand.hpp"
#include "vscreen/molmodel/pocket.hpp"
#include "vscreen/pipeline/bounded_queue.hpp"
#include "vscreen/pipeline/io.hpp"

namespace vscreen {

struct Chunk {
  std::vector<std::uint8_t> bytes;
  std::uint64_t file_offset = 0;
};

struct WorkItem {
  Ligand ligand;
  std::uint64_t sequence_id = 0;
};

struct OutputRow {
  std::string smiles;
  double score = 0.0;
};

struct RankPlan {
  int rank = 0;
  int n_ranks = 1;
  std::uint64_t slab_start = 0;
  std::uint64_t slab_stop = 0;
  std::string input_path;
  std::string output_path;
};

enum class WorkerKind { Fast, Slow };

struct WorkerClass {
  WorkerKind kind = WorkerKind::Fast;
  int count = 1;
  double synthetic_slowdown = 1.0;
};

struct PipelineConfig {
  ScoringConfig scoring;
  std::vector<WorkerClass> workers = {WorkerClass{}};
  std::size_t chunk_bytes = 1 << 20;
  std::size_t chunk_queue_capacity = 8;
  std::size_t item_queue_capacity = 64;
  std::size_t row_queue_capacity = 64;
  std::size_t writer_buffer_bytes = std::size_t(4) << 20;
};

struct DockerStats {
  std::uint64_t rows = 0;
  std::uint64_t dock_errors = 0;
  double busy_seconds = 0.0;
};

struct RankStats {
  std::uint64_t ligands_docked = 0;
  std::uint64_t records_skipped = 0;
  std::uint64_t dock_errors = 0;
  std::uint64_t rows_written = 0;
  std::uint64_t chunks_read = 0;
  std::uint64_t bytes_read = 0;
  std::uint64_t write_calls = 0;
  std::uint64_t bytes_written = 0;
  int workers = 0;
  double wall_seconds = 0.0;
  double reader_busy_seconds = 0.0;
  double splitter_busy_seconds = 0.0;
  double docker_busy_seconds = 0.0;
  double writer_busy_seconds = 0.0;
  std::size_t chunk_queue_high_water = 0;
  std::size_t item_queue_high_water = 0;
  std::size_t row_queue_high_water = 0;
};

// pipeline.cpp:32-45
std::vector<RankPlan> plan_slabs(std::uint64_t file_size, int n_ranks);
// pipeline.cpp:47-62: "SMILES\t<score, fixed 4 decimals>\n"; InvalidArgument if non-finite
std::string format_row(const OutputRow &row);

// pipeline.cpp:430-505: the rank's .stats file, one `key=value` line per
// RankStats field (counts as integers, seconds fixed with 6 decimals);
// parse_rank_stats throws ParseError on a malformed line or unknown key.
std::string format_rank_stats(const RankStats &stats);
RankStats parse_rank_stats(std::string_view text);

// pipeline.cpp:206-244: pop WorkItems, dock them, push one OutputRow per
// ligand with a finite score (others count as dock_errors); stops when `in`
// is closed and drained or `out` is closed.  Batched on the GPU.
DockerStats docker_worker(BoundedQueue<WorkItem> &in, BoundedQueue<OutputRow> &out, const Pocket &pocket,
                          const ScoringConfig &scoring, double synthetic_slowdown);

// pipeline.cpp:297-389 / 391-396 on the B200 CUDA workers
RankStats run_rank(const RankPlan &plan, ByteSource &source, Sink &sink, const Pocket &pocket,
                   const PipelineConfig &config);
RankStats run_rank(const RankPlan &plan, const Pocket &pocket, const PipelineConfig &config);

// pipeline.cpp:398-412: concatenate rank outputs in order
void merge_outputs(const std::vector<std::string> &paths, const std::string &merged_path);

}  // namespace vscreen
