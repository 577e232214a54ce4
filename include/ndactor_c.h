/*
 * ndactor_c.h -- C ABI of the C++ host runtime (libndactor.so).
 *
 * The C++ API (include/ndactor/*.hpp) is the reference's own surface
 * (p/core/include/ndactor/*.hpp); these extern "C" entry points expose the
 * same operations to non-C++ callers (ctypes / cgo / JNI stubs in
 * INTEGRATION.md) with plain pointers and sizes.  Return 0 on success,
 * otherwise an error code; ndactor_last_error() describes the last failure
 * on the calling thread.
 */
#ifndef NDACTOR_C_H
#define NDACTOR_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

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

#ifdef __cplusplus
}
#endif
#endif /* NDACTOR_C_H */
