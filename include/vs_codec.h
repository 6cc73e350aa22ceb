/*
 * vs_codec.h — the ligand record stream of the reference (".xslb",
 * binary_codec.hpp:18-24) on the B200: batched GPU decode of framed records
 * into a ligand set, with the torsion partitions rebuilt from the graph
 * (decode_record, binary_codec.cpp:165-222; torsion_partition,
 * ligand.cpp:110-124; is_connected, ligand.cpp:52-56).
 * rank 1: the step before the dock path.
 *
 * Record: sync 0xD0 0xC5 | record_len u32 LE | name_len u16 | name |
 *   n_atoms u16 | n_bonds u16 | n_torsions u16 | per atom x,y,z f32, element
 *   u8, flags u8 (bit0 heavy) | per bond a u16, b u16, order u8 | per
 *   torsion bond_index u16.
 */
#ifndef VS_CODEC_H
#define VS_CODEC_H

#include "vs_dock.h"
#include "vs_prep.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Per-record decode status (the CodecError cases of decode_record, in the
 * order the reference checks them). */
typedef enum vs_record_status {
  VS_REC_OK = 0,
  VS_REC_BAD_MARKER = 1,        /* "bad sync marker" */
  VS_REC_TRUNCATED = 2,         /* "truncated record" */
  VS_REC_LENGTH_MISMATCH = 3,   /* "record length mismatch" */
  VS_REC_BAD_ELEMENT = 4,       /* "invalid element code" */
  VS_REC_NONFINITE = 5,         /* "non-finite coordinate" */
  VS_REC_BAD_BOND = 6,          /* "invalid bond" */
  VS_REC_BAD_BOND_ORDER = 7,    /* "invalid bond order" */
  VS_REC_BAD_TORSION_INDEX = 8, /* "invalid torsion bond index" */
  VS_REC_NOT_BRIDGE = 9,        /* "invalid torsion: torsion bond is not a bridge" */
  VS_REC_DISCONNECTED = 10,     /* "record graph is disconnected" */
  VS_REC_TOO_LARGE = 11         /* more than 4096 atoms: beyond the GPU decoder */
} vs_record_status;

/* Host framing (the length chain of binary_codec.cpp:166-181): walks the
 * records starting at byte `start` (a record start, e.g. after the 8-byte
 * file header or from find_record_start) and writes up to max_records record
 * offsets.  *next receives the offset after the last framed record.  Returns
 * the number of framed records; stops early at a bad marker or a record
 * extending past `size` (the next call, or the caller, sees it). */
int32_t vs_xslb_frame(const uint8_t *bytes, int64_t size, int64_t start, int32_t max_records, int64_t *offsets,
                      int64_t *next);

/* Decode the n records at `offsets` on the context's GPU into a new ligand
 * set (names = record names, status = vs_record_status, error = the
 * reference's CodecError message).  Invalid records yield an entry with zero
 * atoms.  Replaces a loop of decode_record (binary_codec.cpp:165). */
vs_status vs_decode_records(vs_context *ctx, const uint8_t *bytes, int64_t size, const int64_t *offsets, int32_t n,
                            vs_ligand_set **out);

/* Decode + dock in one call (the pipeline's CUDA worker: decode_record then
 * dock_and_score per record, pipeline.cpp:206-244): the records are framed on
 * the host, decoded on the GPU straight into the dock path's device inputs
 * (no host round trip of the decoded batch) and docked against each of the
 * n_pockets pockets.  results: n_pockets x n entries, pocket-major; a record
 * that fails to decode gets status VS_LIG_BAD_RECORD and its
 * vs_record_status in record_status (may be NULL). */
vs_status vs_dock_records(vs_context *ctx, const vs_pocket *const *pockets, int32_t n_pockets, const uint8_t *bytes,
                          int64_t size, const int64_t *offsets, int32_t n, const vs_scoring_config *cfg,
                          vs_dock_result *results, int32_t *record_status);

/* encode_record (binary_codec.cpp:129-163) of every ligand of a batch, back to
 * back, coordinates truncated to f32 (host).  names may be NULL (empty
 * names).  Returns the bytes written, or -(bytes needed) if cap is too small. */
int64_t vs_encode_records(const vs_ligand_batch *batch, const char *const *names, uint8_t *out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* VS_CODEC_H */
