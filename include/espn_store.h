/*
 * espn_store.h -- C-ABI of the on-disk embedding store: the
 * packed `<base>.espn` data file plus its `<base>.manifest` (binary) and
 * `<base>.manifest.json` twin, as specified for the reference's
 * embedding_store module (proj/include/espn/store.hpp:13-54).
 * It is the data format on the input side of the re-rank path: a store built
 * here (or by the reference) opens as an HBM table through
 * espn_store_read_table + espn_gpu_table_open (include/espn_gpu.h).
 *
 * Layout (all integers little-endian):
 *   data file     records back to back; record i starts at
 *                 manifest.records[i].byte_offset (a multiple of `alignment`),
 *                 holds the d_cls CLS values followed by token_count rows of d
 *                 values (value_width 2 = IEEE binary16, 4 = binary32), and is
 *                 zero-padded to the next record start (store.hpp:20-22); the
 *                 file ends on an `alignment` boundary.
 *   manifest      header {char magic[8] = "ESPNSTR1"; u32 version = 1; u32 d;
 *                 u32 d_cls; u32 value_width; u32 alignment; u32 reserved = 0;
 *                 u64 count} (40 bytes) followed by `count` records
 *                 {u64 byte_offset; u32 byte_length; u32 token_count}
 *                 (16 bytes each; ManifestRecord, store.hpp:13-18).
 *   manifest.json the same fields, for debuggability.
 * byte_length is the exact payload (d_cls + token_count * d) * value_width
 * (store.hpp:32-34); padding is not counted.
 *
 * Pure host code (no device needed); status codes are espn_status.
 */
#ifndef ESPN_STORE_H
#define ESPN_STORE_H

#include <stdint.h>

#include "espn_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t version;      /* 1 */
  uint32_t d;            /* BOW token dim */
  uint32_t d_cls;        /* CLS dim */
  uint32_t value_width;  /* 2 (fp16) or 4 (fp32) */
  uint32_t alignment;    /* 1, 512 or 4096 */
  uint64_t count;        /* documents, dense ids [0, count) */
} espn_store_header;

typedef struct {         /* ManifestRecord (store.hpp:13-18) */
  uint64_t byte_offset;
  uint32_t byte_length;
  uint32_t token_count;
} espn_manifest_record;

/* build_store (store.hpp:48-51): writes <base>.espn, <base>.manifest and
 * <base>.manifest.json.  rows: row_ptr[n_docs] * d fp32 values (CSR over
 * docs, row_ptr[0] == 0); cls: n_docs * d_cls fp32 values or NULL (zeros).
 * Pre: t >= 1 per doc, every value finite, alignment in
 * {1, 512, 4096}, value_width in {2, 4} -> else INVALID_INPUT /
 * INVALID_CONFIG; file errors -> IO.  Width 2 stores RNE binary16. */
ESPN_API int espn_store_build(const char* base, uint64_t n_docs, uint32_t d, uint32_t d_cls,
                              uint32_t value_width, uint32_t alignment, const uint64_t* row_ptr,
                              const float* rows, const float* cls);

/* load_manifest (store.hpp:54): header, and when records != NULL the
 * `count` records (caller-sized from a first call with records == NULL).
 * Bad magic / version / sizes / overlapping or misaligned records -> FORMAT. */
ESPN_API int espn_store_load_manifest(const char* base, espn_store_header* header,
                                      espn_manifest_record* records);

/* Reads every document's BOW rows into a CSR table in the GPU table's code
 * format: row_ptr_out[count + 1] token offsets and codes_out[tokens * d]
 * 2-byte codes of `dtype` (fp16: width-2 stores are copied bit-exactly; other
 * conversions round to nearest even), plus, when cls_out != NULL, the CLS
 * vectors as fp32 (count * d_cls).  Short file -> IO; manifest errors ->
 * FORMAT.  The result feeds espn_table_desc.row_ptr / rows directly. */
ESPN_API int espn_store_read_table(const char* base, uint32_t dtype, uint64_t* row_ptr_out,
                                   uint16_t* codes_out, float* cls_out);

/* save_manifest (store.hpp:53): writes <base>.manifest (+ .manifest.json)
 * from a header and its `count` records. */
ESPN_API int espn_store_save_manifest(const char* base, const espn_store_header* header,
                                      const espn_manifest_record* records);

/* File-backed batched reads: StoreHandle / open_store / fetch_batch
 * (store.hpp:56-112), the reference's own retrieval path --
 * the NVMe tier on the host side.  Modes follow ReadMode (store.hpp:11):
 * DIRECT bypasses the page cache (O_DIRECT, aligned spans through an aligned
 * bounce buffer; needs alignment >= 512, else INVALID_CONFIG; a filesystem
 * without O_DIRECT -> IO), BUFFERED preads the exact payload, MMAP copies
 * from a shared mapping.  queue_depth reads are in flight (store.hpp:73-76). */
#define ESPN_READ_DIRECT 0u
#define ESPN_READ_BUFFERED 1u
#define ESPN_READ_MMAP 2u
typedef struct espn_store_reader espn_store_reader;
ESPN_API int espn_store_open(const char* base, uint32_t mode, uint32_t queue_depth, espn_store_reader** out,
                             espn_store_header* header);
ESPN_API int espn_store_close(espn_store_reader* reader);
/* The manifest records (header.count of them). */
ESPN_API int espn_store_records(const espn_store_reader* reader, espn_manifest_record* out);
/* Reads the records of ids[0..n) (duplicates allowed; unknown id ->
 * INVALID_INPUT listing the offenders) in request order: record i's payload
 * (byte_length bytes: CLS values then BOW rows, value_width each) lands at
 * out + out_off[i], out_off[n+1] being the prefix of payload sizes.  Counters
 * (store.hpp:61-65): bytes_read = payload bytes, aligned-rounded in direct
 * mode; blocks_read = sum of ceil(byte_length / block), block = alignment in
 * direct mode else 4096; wall_time in seconds.  out == NULL: offsets and
 * counters only.  Short read -> IO. */
ESPN_API int espn_store_fetch(espn_store_reader* reader, const uint32_t* ids, uint64_t n, uint8_t* out,
                              uint64_t* out_off, uint64_t capacity, uint64_t* bytes_read, uint64_t* blocks_read,
                              double* wall_time);

/* The BOW rows of docs [doc_begin, doc_begin + n) in the GPU table's code
 * format (fp16: width-2 stores copied bit-exactly; else round to nearest
 * even): row_ptr_out[n + 1] local token offsets, codes_out the rows (NULL:
 * offsets only).  Feeds espn_gpu_table_load_rows chunk by chunk, so a store
 * opens without ever being read whole. */
ESPN_API int espn_store_read_rows(espn_store_reader* reader, uint64_t doc_begin, uint64_t n, uint32_t dtype,
                                  uint64_t* row_ptr_out, uint16_t* codes_out);

/* Thread-local message of the last failing call of this library. */
ESPN_API const char* espn_store_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ESPN_STORE_H */
