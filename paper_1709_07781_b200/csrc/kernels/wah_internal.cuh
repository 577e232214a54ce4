// Device-resident control block shared by the four build stages.
// It travels between the stage actors as the `cfg` MemRef -- the B200
// analogue of the paper's "configuration array" (PAPER.md:394,
// p/core/src/wah_stages.cpp:33-34 uses cfg u32[2] the same way).
#pragma once
#include <cstdint>

namespace ndx {

enum SortMode : uint32_t { kModeNone = 0, kModeWide = 1, kModeBytes = 2, kModeAB = 3 };

constexpr int kWideMaxBits = 11;                 // single pass up to 2048 buckets
constexpr int kWideBuckets = 1 << kWideMaxBits;
constexpr int kMaxRowsValues = 1 << 16;          // compact mode: keys share their top 16 bits

struct SortPlan {
  uint32_t mode;           // SortMode
  uint32_t complete;       // plan final (bytes 2/3 histograms not pending)
  uint32_t need_hi;        // bytes 2/3 vary: second histogram pass required
  uint32_t base;           // wide mode: digit = key - base; compact mode: the keys' top 16 bits
  uint32_t wide_bits;      // wide mode: digit width (0..11)
  uint32_t nseg;           // compact mode: row segments (2^24 rows each)
  uint32_t npasses;        // number of scatter passes that run
  uint32_t byte_active[4]; // bytes mode: byte k gets a pass
  uint32_t byte_order[4];  // bytes mode: execution index of byte k's pass
  uint32_t bucket_start_wide[kWideBuckets];
  uint32_t bucket_start_byte[4][256];
};

// Layout is part of the C ABI for the first 32 bytes (ndx_wah_counts in
// include/ndx.h); everything below `zero_end` is cleared at every build.
struct Ctl {
  uint64_t words;      // W, written by the emit stage
  uint64_t distinct;   // D, written by the emit stage
  uint32_t min_key;    // written by the plan stage
  uint32_t max_key;
  uint32_t n_lo, n_hi; // row count of the build
  // ---- scratch (zeroed) ----
  uint32_t max_seen;   // max(key)
  uint32_t max_not;    // max(~key) -> min = ~max_not
  uint32_t tile_ctr[16];
  uint32_t grid_bar[2];  // cooperative sort launch: arrivals, generation
  uint32_t hist_byte[4][256];
  uint32_t hist_wide[kWideBuckets];
  uint32_t rows_form;  // 1: the sort wrote row ids only (values from vs / pk below)
  uint64_t vs_agg[kMaxRowsValues / 1024];  // k_vs: present keys per block of 1024 | ready bit
  uint32_t zero_end;
  // ---- written by the plan kernel ----
  uint32_t epoch;      // look-back status tag of this build (from the sort scratch counter)
  uint32_t row_hi;     // largest row id of the build (row_base + n - 1), written by the sort
  SortPlan plan;
  // ---- the sorted stream's values in rows form (wide and compact modes) ----
  // The wide pass and pass B write row ids only; the values are the present
  // keys in order, pk[i] holding rows [vs[i], vs[i+1]) of the stream
  // (vs[nvals] = n).  Written by k_vs after the last pass from vs16
  // (compact mode: where each low-16-bit key starts, present or not --
  // written, every entry, by the pass-B tile holding its start).
  uint32_t nvals;
  uint32_t vs[kMaxRowsValues + 1];
  uint32_t pk[kMaxRowsValues];
  uint32_t vs16[kMaxRowsValues];
};

}  // namespace ndx
