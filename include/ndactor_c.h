/*
 * ndactor_c.h -- C ABI of the C++ host runtime (libndactor.so).
 *
 * The C++ API (include/ndactor/*.hpp) is the reference's own surface
 * (p/core/include/ndactor/*.hpp).  These extern "C" entry points expose the
 * same operations to non-C++ callers (the ctypes/cgo/JNI stubs of
 * INTEGRATION.md) with plain pointers and sizes.  Every function returns 0
 * on success or a nonzero code; ndactor_last_error() describes the last
 * failure on the calling thread.  Nothing throws across this boundary.
 */
#ifndef NDACTOR_C_H
#define NDACTOR_C_H

#include <stddef.h>
#include <stdint.h>

#include "ndx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A runtime = one ActorSystem + one Device (CUDA ordinal) + the four build
 * stage actors (plan, sort, emit, table) chained table*emit*sort*plan. */
typedef struct ndactor_runtime ndactor_runtime;

int ndactor_runtime_create(int device_ordinal, unsigned workers, ndactor_runtime** out);
void ndactor_runtime_destroy(ndactor_runtime* rt);
const char* ndactor_last_error(void);
/* The runtime device's in-order stream (cudaStream_t), for callers that
 * time or order their own work against it. */
void* ndactor_runtime_stream(ndactor_runtime* rt);
int ndactor_runtime_synchronize(ndactor_runtime* rt);

/* wah::build_index (p/core/src/wah_builder.cpp:38-307) through the actor
 * chain: host values in, host index out.  `words`/`entries` are caller
 * buffers (pinned host memory is fastest) of at least 2n and 3n u32; the
 * entries are (value, offset, length) triples.  Bit-exact with the
 * reference's reference_index.  row_base offsets the row ids (shards). */
int ndactor_wah_build_index(ndactor_runtime* rt, const uint32_t* values, uint64_t n,
                            uint32_t row_base, uint32_t* words, uint64_t words_cap,
                            uint32_t* entries, uint64_t entries_cap,
                            uint64_t* n_words, uint64_t* n_entries);

/* Pipelined variant of ndactor_wah_build_index for a stream of columns:
 * returns at once.  Three streams keep both PCIe directions and the SMs busy:
 * the upload of `values` (pinned host memory) on its own stream, the build
 * on the device stream, and the result copy on an egress stream.  The build
 * ends with a copy of the counts to pinned memory; an egress thread then
 * issues exactly min(W, words_cap) words and min(3D, entries_cap) table
 * words of device-to-host copy (copy engines, no SMs).  So step i's result
 * copy overlaps step i+1's upload and build.  At most two builds in flight:
 * call ndactor_wah_wait(ticket) before reusing a ticket's buffers.  The
 * inputs must stay untouched until then.  counts->words / ->distinct give
 * the true sizes even if the capacities were too small. */
int ndactor_wah_build_index_async(ndactor_runtime* rt, const uint32_t* values, uint64_t n,
                                  uint32_t* words, uint64_t words_cap, uint32_t* entries,
                                  uint64_t entries_cap, ndx_wah_counts* counts, uint64_t* ticket);
int ndactor_wah_wait(ndactor_runtime* rt, uint64_t ticket);

/* The same chain on keys already resident on the device (d_keys: n u32, not
 * modified; row ids start at row_base).  The result stays on the device:
 * *d_counts points at an ndx_wah_counts {words, distinct, min, max},
 * *d_words at the words, *d_entries at the (value, offset, length) triples.
 * The pointers stay valid until the next call on this runtime.  Returns as
 * soon as the work is enqueued on ndactor_runtime_stream (no host sync). */
int ndactor_wah_build_index_device(ndactor_runtime* rt, const uint32_t* d_keys, uint64_t n,
                                   uint32_t row_base, uint32_t** d_words, uint32_t** d_entries,
                                   void** d_counts);

/* BASELINE config 2: `iters` one-warp kernels issued (a) raw, back to back
 * with the C ABI on the runtime stream, (b) as compute-actor requests where
 * each request is issued from the previous reply (in_out reference, replies
 * leave before the kernel runs).  Both end with one synchronisation; host
 * wall time in milliseconds.  `check` receives the final counter (2*iters). */
int ndactor_dispatch_probe(ndactor_runtime* rt, uint64_t iters, double* raw_ms, double* actor_ms,
                           uint64_t* check);
/* Same, with the breakdown: out[0] raw total ms, out[1] raw host enqueue ms,
 * out[2] actor total ms, out[3] actor chain with a no-op launcher (pure host
 * cost of `iters` hops), out[4] final counter value. */
int ndactor_dispatch_probe_ex(ndactor_runtime* rt, uint64_t iters, double* out);

/* Synthetic columns, bit-identical to the reference's generators:
 * std::mt19937(seed) + uniform_int_distribution<u32>(0, cardinality-1)
 * (p/tools/ndcli.cpp:144-148) and the Zipf stream of SURVEY.md App. C
 * (mt19937_64(seed), uniform_real_distribution<double>(0,1), inverse CDF). */
void ndactor_gen_uniform(uint32_t seed, uint64_t n, uint32_t cardinality, uint32_t* out);
void ndactor_gen_zipf(uint64_t seed, uint64_t n, uint32_t k, double s, uint32_t* out);
/* The instance stream of the reference's acceptance gate
 * (p/tests/acceptance.cpp:56-63). */
void ndactor_gen_instances(uint32_t seed, uint32_t count, const uint32_t* cards,
                           uint32_t ncards, uint32_t max_rows, uint64_t* sizes,
                           uint32_t* out);

/* Multi-GPU build (include/ndactor/wah_shard.hpp).
 * bounds[0..shards]: row shard bounds, inner ones multiples of 31. */
int ndactor_shard_bounds(uint64_t n, uint32_t shards, uint64_t* bounds);
/* Merge plan over the shards' metadata (ndx_wah_shard_meta of each shard,
 * counts[g] records each; shard g starts at metas + g*stride, or the shards
 * are concatenated when stride is 0).  Writes the merged (value, offset,
 * length) entries (capacity: sum of counts) and one ndx_piece per input
 * record at the same position (dst absolute in the merged words; src_off
 * local to the shard's words). */
int ndactor_merge_plan(uint32_t shards, const ndx_shard_meta* metas, const uint64_t* counts,
                       uint64_t stride, uint32_t* entries, ndx_piece* pieces,
                       uint64_t* n_entries, uint64_t* n_words);

/* FNV-1a-64 of the "WAH1" serialization of an index (row_count, entries as
 * (value, offset, length) triples, words) -- the digest of SURVEY.md App. C
 * and tests/golden/digests.json, computed without a serialized copy. */
uint64_t ndactor_index_digest(uint32_t row_count, const uint32_t* entries, uint64_t n_entries,
                              const uint32_t* words, uint64_t n_words);

/* The multi-GPU build behind the actor API (include/ndactor/wah_dist.hpp):
 * one ndactor_dist per rank (one process per GPU), NCCL loaded by the
 * runtime.  Rank 0 makes the id, every rank gets a copy (any host channel),
 * then every rank calls ndactor_dist_create (collective).  A step enqueues
 * the shard build, the metadata all-gather, the merge plan and the word
 * exchange on the runtime stream and returns; ndactor_dist_outputs gives the
 * device results: totals {D, W, error flags, records}, bounds[0..G], the
 * merged (value, offset, length) table (replicated), the rank's slice of
 * the merged words [bounds[rank], bounds[rank+1]) (after a gather_all step:
 * all W words, on every rank that asked), and the rank's local words. */
typedef struct ndactor_dist ndactor_dist;
int ndactor_nccl_unique_id(uint8_t* id128);
int ndactor_dist_create(ndactor_runtime* rt, int rank, int nranks, const uint8_t* id128, uint64_t local_cap,
                        uint32_t meta_cap, uint64_t slice_cap, ndactor_dist** out);
int ndactor_dist_step(ndactor_dist* d, const uint32_t* d_keys, uint64_t n_local, uint64_t row_base, int gather_all);
int ndactor_dist_outputs(ndactor_dist* d, uint64_t** d_totals, uint64_t** d_bounds, uint32_t** d_entries,
                         uint32_t** d_slice, uint32_t** d_local_words);
void ndactor_dist_destroy(ndactor_dist* d);

/* "WAH1" index file (p/core/src/wah_index_io.cpp:30-87). */
int ndactor_write_index_file(const char* path, uint32_t row_count, const uint32_t* entries,
                             uint64_t n_entries, const uint32_t* words, uint64_t n_words);

#ifdef __cplusplus
}
#endif
#endif /* NDACTOR_C_H */
