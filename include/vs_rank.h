/*
 * vs_rank.h — one rank of the screening pipeline on B200s (SURVEY.md §8(f)
 * rank 2): the reference's run_rank (pipeline.cpp:297-398: reader ->
 * splitter -> W docker workers -> writer) with its docker stage replaced by
 * CUDA workers.
 *
 *   reference                          this build
 *   stage_reader (chunks)              the same: chunked reads through a
 *                                      read callback (ByteSource::read_at)
 *   stage_splitter: scan_record_start  host framing only (sync marker + the
 *     + decode_record per record       2-hop length-chain rule); records go
 *                                      to the GPU as raw bytes, decoded there
 *   docker_worker: dock_and_score per  CUDA workers: W threads per GPU, each
 *     WorkItem, W threads              with its own vs_context (stream,
 *                                      device buffers) and library-owned
 *                                      pinned staging; one vs_dock_records
 *                                      call per batch of records, so batch
 *                                      i+1's upload/decode overlaps batch
 *                                      i's kernels on another stream
 *   stage_writer: format_row           the same rows (format_row,
 *                                      pipeline.cpp:47-62), in record order
 *
 * Semantics kept from the reference: a rank owns the records whose start
 * lies in [slab_start, slab_stop) (pipeline.cpp:32-45, 168-169); a framed
 * record that fails to decode counts as records_skipped and the scan
 * resumes two bytes after its marker (pipeline.cpp:180-185); a ligand whose
 * dock throws or scores non-finite counts as dock_errors and writes no row
 * (pipeline.cpp:218-238); a final marker without a valid chain fails the
 * rank ("corrupt record stream", binary_codec.cpp:240-252).  One deviation:
 * an invalid ScoringConfig fails the call up front, where the reference
 * turns every ligand into a dock_error (search.cpp:240-243 inside the
 * workers' try blocks).  Rows come out
 * in record order: the reference's row order is its workers' completion
 * order, identical to record order with one worker.
 */
#ifndef VS_RANK_H
#define VS_RANK_H

#include "vs_dock.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ByteSource::read_at (io.hpp): fill out[0..n) from `offset`; returns the
 * bytes read (0 at the end), < 0 on error. */
typedef int64_t (*vs_read_fn)(void *user, uint64_t offset, uint8_t *out, int64_t n);
/* Sink::write (io.hpp); nonzero return = error. */
typedef int32_t (*vs_write_fn)(void *user, const char *bytes, int64_t n);

typedef struct vs_rank_config {
  int32_t n_devices;          /* GPUs to use; 0 = every visible device */
  const int32_t *devices;     /* NULL: devices 0..n_devices-1 */
  int32_t workers_per_device; /* CUDA workers (contexts / streams) per GPU, >= 1 */
  int32_t batch_records;      /* records per vs_dock_records call (> 0) */
  int64_t chunk_bytes;        /* reader chunk (PipelineConfig::chunk_bytes) */
  int64_t writer_buffer_bytes;/* writer flush size (PipelineConfig::writer_buffer_bytes) */
} vs_rank_config;

/* RankStats (pipeline.hpp:96-115) */
typedef struct vs_rank_stats {
  uint64_t ligands_docked, records_skipped, dock_errors, rows_written;
  uint64_t chunks_read, bytes_read, write_calls, bytes_written;
  int32_t workers;
  double wall_seconds, reader_busy_seconds, splitter_busy_seconds, docker_busy_seconds, writer_busy_seconds;
  uint64_t batches, resyncs;  /* GPU batches docked; batches re-framed after a bad record */
} vs_rank_stats;

void vs_rank_config_default(vs_rank_config *rc);

/* run_rank(plan, source, sink, pocket, config) (pipeline.cpp:297-389) on the
 * configured GPUs.  Returns VS_OK, VS_ERR_INVALID_ARGUMENT (bad plan/config,
 * corrupt record stream; message in vs_last_error_message), or a device
 * error. */
vs_status vs_run_rank(uint64_t source_size, vs_read_fn read, void *read_user, uint64_t slab_start,
                      uint64_t slab_stop, const vs_pocket_desc *pocket, const vs_scoring_config *cfg,
                      const vs_rank_config *rc, vs_write_fn write, void *write_user, vs_rank_stats *stats);

/* The campaign ranking (cmd_merge, merge.cpp:81-147): every row of the
 * n_files score texts (rank order) stable-sorted by (printed score desc,
 * SMILES asc) and written as the original row text, one per line; only the
 * first top_k rows when top_k >= 0.  Parallel run sorts on `threads` host
 * threads (0 = all) + a stable k-way merge.  *rows_out = rows written. */
vs_status vs_merge_rankings(const char *const *texts, const int64_t *lens, int32_t n_files, int64_t top_k,
                            int32_t threads, vs_write_fn write, void *user, uint64_t *rows_out);

/* Pinned (page-locked) host memory for callers that stage their own batches. */
vs_status vs_host_alloc(size_t bytes, void **out);
void vs_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* VS_RANK_H */
