/*
 * ndx.h -- C ABI of the B200 device layer (libndx.so).
 *
 * This is the thin C layer the C++ host runtime (include/ndactor/*.hpp,
 * libndactor.so) calls, and the surface any other FFI (ctypes, cgo, JNI)
 * binds.  It replaces the reference's CPU-simulated OpenCL device
 * (p/core/include/ndactor/device.hpp:26-86, p/core/src/device.cpp) and its
 * host-lambda "kernels" (p/core/include/ndactor/kernel.hpp:181-193) with CUDA
 * streams, events, stream-ordered allocations and sm_100a kernels.
 *
 * Conventions
 *   - Every function returns 0 on success, otherwise a cudaError_t value or
 *     one of the NDX_E_* codes below; ndx_error_string() names it.  Nothing
 *     throws across this boundary.
 *   - Pointers named d_* are device pointers, h_* host pointers.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Launches are asynchronous and thread-safe per stream.
 *
 * p/ = /root/reference/proj/ in the citations below.
 */
#ifndef NDX_H
#define NDX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NDX_E_INVALID 10001    /* bad argument (null pointer, size)       */
#define NDX_E_TOO_LARGE 10002  /* input exceeds the u32 index format      */
#define NDX_E_NO_DEVICE 10003  /* no CUDA device / extension unusable     */

const char* ndx_error_string(int code);
/* Version of the ABI; bumped on any signature change. */
int ndx_abi_version(void);

/* ---------------------------------------------------------------------------
 * Device, streams, events, memory.
 * Replace Device (device.hpp:26-86), Event (event.hpp:22-57) and the
 * Buffer storage (buffer.hpp:27-40) of the simulated backend.
 * ------------------------------------------------------------------------- */
int ndx_device_count(int* count);
int ndx_device_open(int ordinal);           /* cudaSetDevice + mempool setup */
int ndx_device_bind(int ordinal);           /* cudaSetDevice only (per host thread) */
/* cudaMalloc'd memory other processes can map (CUDA IPC, 64-byte handles):
 * the multi-GPU build reads peer shards' words over NVLink. */
int ndx_malloc_shared(void** p, size_t bytes);
int ndx_free_shared(void* p);
int ndx_ipc_handle(const void* p, void* handle64);
int ndx_ipc_open(const void* handle64, void** p);
int ndx_ipc_close(void* p);
int ndx_device_sm_count(int ordinal, int* sms);
int ndx_device_synchronize(void);

int ndx_stream_create(void** stream);       /* non-blocking stream */
int ndx_stream_destroy(void* stream);
int ndx_stream_synchronize(void* stream);
/* 0 = all work done, 1 = still running, else an error */
int ndx_stream_query(void* stream);

int ndx_event_create(void** event, int timing);
int ndx_event_destroy(void* event);
int ndx_event_record(void* event, void* stream);
int ndx_event_query(void* event);           /* 0 = complete, 1 = pending */
int ndx_event_synchronize(void* event);
int ndx_stream_wait_event(void* stream, void* event);
int ndx_event_elapsed_ms(void* start, void* stop, float* ms);

/* Stream-ordered allocation from the device's memory pool
 * (create_buffer / free_buffer, device.cpp:228-249). */
int ndx_malloc_async(void** d_ptr, size_t bytes, void* stream);
int ndx_free_async(void* d_ptr, void* stream);
int ndx_memset_async(void* d_ptr, int value, size_t bytes, void* stream);
int ndx_host_alloc(void** h_ptr, size_t bytes);   /* pinned */
int ndx_host_free(void* h_ptr);
/* enqueue_write_bytes / enqueue_read_bytes (device.cpp:253-283) */
int ndx_memcpy_h2d_async(void* d_dst, const void* h_src, size_t bytes, void* stream);
int ndx_memcpy_d2h_async(void* h_dst, const void* d_src, size_t bytes, void* stream);
int ndx_memcpy_d2d_async(void* d_dst, const void* d_src, size_t bytes, void* stream);

/* ---------------------------------------------------------------------------
 * WAH index build: the four device stages.
 * Replaces wah::build_index (p/core/src/wah_builder.cpp:38-307).
 *
 *   S1 plan   keys[n]              -> ctl (key range, histograms, sort plan)
 *   S2 sort   keys[n] + ctl        -> the sorted stream (stable by key; row ids
 *                                     made on the fly) in d_pairs, in one of
 *                                     two forms chosen on the device:
 *                                     rows form (keys within 2^16 of each
 *                                     other): u32 row ids, the values kept in
 *                                     ctl as the present keys and where each
 *                                     one's rows begin; pairs form (any other
 *                                     keys): u64 (key | row << 32)
 *   S3 emit   stream + ctl         -> words[<=2n], vstart[<=n], values[<=n],
 *                                     ctl.{words, distinct}
 *   S4 table  values, vstart, ctl  -> entries[3*D] (value, offset, length)
 *
 * `ctl` is a device block of ndx_wah_ctl_bytes() bytes; its first 24 bytes
 * are an ndx_wah_counts the host may read back after S3.  `status` is a
 * buffer of ndx_wah_status_bytes(n) bytes owned by the caller, zero-filled
 * ONCE after allocation and used for nothing else: it carries the sort's
 * decoupled look-back statuses, tagged per build so it never needs
 * clearing: its header keeps the tag counter and the high-water mark of the
 * statuses written, and the build whose 24-bit tags wrap (one in 2^21)
 * clears them all itself.  The emit's scratch (ndx_wah_emit_scratch_bytes(n)
 * bytes, 128-byte aligned) holds its per-tile aggregates and value-head
 * records and is cleared by the emit stage itself.  All sizes stay on the
 * device: no stage needs a host round trip.
 * n must be below 2^31 (the index format's word offsets are u32).
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t words;     /* W: compressed words in the index         */
  uint64_t distinct;  /* D: distinct values (index entries)        */
  uint32_t min_key;
  uint32_t max_key;
} ndx_wah_counts;

size_t ndx_wah_ctl_bytes(void);
size_t ndx_wah_status_bytes(uint64_t n);
size_t ndx_wah_emit_scratch_bytes(uint64_t n);

int ndx_wah_plan(const uint32_t* d_keys, uint64_t n, void* d_ctl, void* d_status,
                 void* stream);
int ndx_wah_sort(const uint32_t* d_keys, uint64_t n, uint32_t row_base, void* d_ctl,
                 uint64_t* d_pairs, uint64_t* d_tmp_pairs, void* d_status, void* stream);
int ndx_wah_emit(const uint64_t* d_pairs, uint64_t n, void* d_ctl, uint32_t* d_words,
                 uint32_t* d_vstart, uint32_t* d_values, void* d_emit_scratch,
                 void* stream);
int ndx_wah_table(const uint32_t* d_values, const uint32_t* d_vstart,
                  uint64_t n, const void* d_ctl, uint32_t* d_entries,
                  void* stream);

/* Result copy-out with no host round trip for the sizes: a kernel reads W and
 * D from ctl and writes the counts, min(W, words_cap) words and
 * min(3D, entries_cap) table words straight into host memory.  h_* must be
 * pinned (device-accessible) host memory; the data is there once the
 * stream reaches this point. */
int ndx_wah_copy_out(const void* d_ctl, const uint32_t* d_words, const uint32_t* d_entries,
                     ndx_wah_counts* h_counts, uint32_t* h_words, uint64_t words_cap,
                     uint32_t* h_entries, uint64_t entries_cap, void* stream);

/* ---------------------------------------------------------------------------
 * Query side: decode, bitwise ops, rows, encode.
 * A decoded bitmap is a chunk array: one u32 per 31-row chunk holding the
 * chunk's literal (bit i = row 31c + i).
 * ------------------------------------------------------------------------- */
/* decode (wah_words.cpp:21-34): chunks[c] for c < n_chunks, zero past the
 * end of the stream.  d_info[0] = chunks the words cover, d_info[1] = 1 if
 * a fill has length zero. */
size_t ndx_wah_decode_scratch_bytes(uint64_t n_words);
int ndx_wah_decode(const uint32_t* d_words, uint64_t n_words, uint32_t* d_chunks,
                   uint64_t n_chunks, void* d_scratch, uint32_t* d_info, void* stream);
/* out = a AND b / a OR b / a AND NOT b over n chunks. */
int ndx_chunks_and(const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n,
                   void* stream);
int ndx_chunks_or(const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n,
                  void* stream);
int ndx_chunks_andnot(const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n,
                      void* stream);
/* rows_for (wah_words.cpp:93-103) on a decoded bitmap: the rows of the set
 * bits below row_limit, ascending; *d_count = their number.  d_rows must
 * hold every set bit of the chunks. */
size_t ndx_chunks_rows_scratch_bytes(uint64_t n_chunks);
int ndx_chunks_rows(const uint32_t* d_chunks, uint64_t n_chunks, uint32_t row_limit,
                    uint32_t* d_rows, void* d_scratch, uint32_t* d_count, void* stream);
/* Canonical words of a chunk array (CanonicalWriter, wah.hpp:36-74): every
 * chunk (trim_trailing = 0, as encode() does) or up to the last set bit
 * (trim_trailing = 1, as an index bitmap).  d_words holds up to n_chunks
 * words; d_info[0] = word count, [1] error flags, [2] chunks encoded. */
size_t ndx_wah_encode_scratch_bytes(uint64_t n_chunks);
int ndx_wah_encode(const uint32_t* d_chunks, uint64_t n_chunks, int trim_trailing,
                   uint32_t* d_words, void* d_scratch, uint32_t* d_info, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU build: shards of rows [S_g, S_{g+1}),
 * S_g = 0 mod 31, are built with row_base = S_g; the pieces are then merged.
 * ------------------------------------------------------------------------- */
/* Per value of one shard's local index. */
typedef struct {
  uint32_t value;
  uint32_t f;         /* first chunk holding the value in this shard         */
  uint32_t l;         /* last chunk                                          */
  uint32_t a;         /* ones-fill length of the body's first word, or 0     */
  uint32_t z;         /* ones-fill length of the body's last word, or 0      */
  uint32_t body_off;  /* local word offset of the body (after the leading    */
  uint32_t body_len;  /*   zero-fill, which is `skip` words long: 0 or 1)    */
  uint32_t skip;
} ndx_shard_meta;

/* One piece of the merged index: `lead` (if nonzero) at dst, then src_len
 * words from src_off of the shard's (staged) words. */
typedef struct {
  uint64_t dst;
  uint32_t src_off;
  uint32_t src_len;
  uint32_t lead;
  uint32_t pad;
} ndx_piece;

/* meta[d] for each entry d of a local index built by the four stages
 * (d_pairs and d_ctl: that build's sorted stream and control block). */
int ndx_wah_shard_meta(const uint64_t* d_pairs, uint64_t n, const void* d_ctl, const uint32_t* d_entries,
                       uint64_t n_entries, const uint32_t* d_words, ndx_shard_meta* d_meta,
                       void* stream);
/* The same with the value count read from the device (d_ctl's
 * ndx_wah_counts) and at most `cap` records written (no host round trip). */
int ndx_wah_shard_meta_dev(const uint64_t* d_pairs, uint64_t n, const uint32_t* d_entries,
                           const void* d_ctl, uint64_t cap, const uint32_t* d_words, ndx_shard_meta* d_meta,
                           void* stream);
/* The merge plan on the device (same result as ndactor_merge_plan): shard
 * g's records at d_metas + g*stride, h_counts[g] of them (host array,
 * shards <= 64).  Writes the merged (value, offset, length) entries and one
 * ndx_piece per record at the same slot (dst absolute).  d_totals: [0]
 * entries, [1] words, [2] error flags (1 empty body, 2 overlapping shards). */
size_t ndx_merge_plan_scratch_bytes(uint64_t records);
int ndx_merge_plan(const ndx_shard_meta* d_metas, uint64_t stride, const uint64_t* h_counts,
                   uint32_t shards, uint32_t* d_entries, ndx_piece* d_pieces, uint64_t* d_totals,
                   void* d_scratch, void* stream);
/* Copies every piece of a device plan (slots g*stride + i, h_counts[g] per
 * shard) to out; h_src[g] is shard g's words (device pointers, host array). */
int ndx_wah_assemble_slots(const uint32_t* const* h_src, uint32_t shards, const ndx_piece* d_pieces,
                           uint64_t stride, const uint64_t* h_counts, uint32_t* d_out, void* stream);
/* Copies every piece to out (the merged words). */
int ndx_wah_assemble(const uint32_t* d_src, const ndx_piece* d_pieces, uint64_t n_pieces,
                     uint32_t* d_out, void* stream);

/* The per-step device work of the multi-GPU build with the
 * shard counts on the device -- no host round trip between the metadata
 * all-gather and the word exchange.  d_metas: shard g's records in slots
 * [g*cap, g*cap + d_counts[g].distinct) (the all-gathered ndx_wah_counts of
 * every shard).  Writes the merged (value, offset, length) table, the pieces
 * in merged (destination) order with the source shard in `pad`, d_totals
 * {D, W, error flags (1 empty body, 2 overlapping shards, 4 metadata
 * capacity exceeded, 8 slice capacity exceeded), records} and the G+1 owner
 * bounds (rank h owns words [b_h, b_h+1), cut at value boundaries). */
size_t ndx_dist_plan_scratch_bytes(uint32_t shards, uint64_t cap);
int ndx_dist_plan(const ndx_shard_meta* d_metas, uint64_t cap, const ndx_wah_counts* d_counts, uint32_t shards,
                  uint32_t* d_entries, ndx_piece* d_merged, uint64_t* d_totals, uint64_t* d_bounds,
                  void* d_scratch, void* stream);
/* Rank `rank`'s owned slice of the merged words (all_words: the whole
 * array), copied from every shard's words; h_shard_words[g] may point into
 * another GPU's memory (IPC-mapped, read over NVLink).  out_cap: capacity of
 * d_out in words; out_hint: expected slice size (grid sizing). */
int ndx_dist_pull(const uint32_t* const* h_shard_words, uint32_t shards, const ndx_piece* d_merged,
                  uint64_t max_records, uint64_t* d_totals, const uint64_t* d_bounds, uint32_t rank, int all_words,
                  uint32_t* d_out, uint64_t out_cap, uint64_t out_hint, void* stream);

/* ---------------------------------------------------------------------------
 * Device primitives behind the reference's public WAH device API
 * (p/core/include/ndactor/wah_device.hpp:17-50).
 * ------------------------------------------------------------------------- */
/* scan_exclusive (wah_scan.cpp:14-95): out[i] = sum(in[0..i)) mod 2^32. */
size_t ndx_scan_scratch_bytes(uint64_t n);
int ndx_scan_exclusive_u32(const uint32_t* d_in, uint32_t* d_out, uint64_t n,
                           void* d_scratch, void* stream);

/* sort_pairs (wah_radix.cpp:16-127): stable by key, in place. */
size_t ndx_sort_pairs_scratch_bytes(uint64_t n);
int ndx_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_payloads, uint64_t n,
                       void* d_scratch, void* stream);

/* The three compaction stages (wah_stages.cpp:29-163), same protocol:
 * cfg is u32[2]; cfg[0] = k on the way in, cfg[1] = output length. */
int ndx_compact_prepare(uint32_t* d_cfg, const uint32_t* d_a,
                        const uint32_t* d_b, uint64_t k, uint32_t* d_out,
                        void* stream);
/* counts[t] = nonzeros in data[4096 t, 4096 t + 4096) (wah_stages.cpp:59-91) */
int ndx_compact_count(const uint32_t* d_data, uint64_t n, uint32_t* d_counts,
                      void* stream);
/* order-preserving scatter of nonzeros; cfg[1] = total (wah_stages.cpp:93-156) */
size_t ndx_compact_move_scratch_bytes(uint64_t n);
int ndx_compact_move(uint32_t* d_cfg, const uint32_t* d_data, uint64_t n,
                     const uint32_t* d_counts, uint32_t* d_out,
                     void* d_scratch, void* stream);

/* out = a x b for n x n row-major fp32 matrices, the k sum in ascending order
 * with separately rounded multiply and add (bit-identical to the reference's
 * triple loop): the matmul actor of the paper's facade-overhead protocol
 * (p/core/src/bench_protocols.cpp, acceptance.cpp checks 6-7). */
int ndx_matmul_f32(const float* d_a, const float* d_b, float* d_out, uint64_t n, void* stream);

/* One-CTA, one-warp `p[0] += 1` kernel: the dispatch-overhead probe of
 * BASELINE config 2 (p/benchmarks/bench_device.cpp:14-24). */
int ndx_tiny_increment(uint32_t* d_p, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NDX_H */
