// Dispatch / combine plan of the expert-parallel exchange (world > 1), from the all-gathered
// representative counts c[P][E] (P:143 dispatch, P:144 combine; layouts R14/R15).
//
// ONE definition, compiled for both sides: the device count-exchange kernel (exchange.cu,
// xcnt_plan_kernel + xplan_rows_kernel) derives the layout the kernels use with it, and the host export
// luffy_exchange_plan (api.cu) runs the very same code, so the gloo world-2 test
// (tests/test_multirank_cpu.py) covers the plan the product ships.
//
//   src_soff[q][e]  padded send offsets of rank q: expert asc, each segment rounded up to kRowAlign (R15)
//   roff[el]        padded expert-layout offsets of rank `me`: local expert asc; within a segment the
//                   source ranks' rows in rank order (R15)
//   dst_base[e]     first row, in the owner's expert layout, of the rows `me` sends to expert e
//   xplan_row(r)    inverse map for the combine: (source rank, source send slot) of expert-layout row r
//                   of `me`, (-1, -1) for padding
#pragma once
#include <stdint.h>

#include "luffy.h"

#if defined(__CUDACC__)
#define LUFFY_HD __host__ __device__ __forceinline__
#else
#define LUFFY_HD inline
#endif

namespace luffy {

LUFFY_HD int32_t xplan_pad(int64_t rows) {
  return (int32_t)((rows + LUFFY_ROW_ALIGN - 1) / LUFFY_ROW_ALIGN * LUFFY_ROW_ALIGN);
}

// Work split over `nthr` cooperating threads (tid in [0, nthr)); every output element has one writer and
// only `c` is read, so the threads need no synchronisation.  Host: tid = 0, nthr = 1.
LUFFY_HD void xplan_body(const int32_t* c, int P, int E, int me, int32_t* cnt_all, int32_t* roff, int32_t* dst_base,
                         int32_t* src_soff, int tid, int nthr) {
  const int El = E / P;
  if (cnt_all)
    for (int i = tid; i < P * E; i += nthr) cnt_all[i] = c[i];
  for (int q = tid; q < P; q += nthr) {
    int32_t o = 0;
    for (int e = 0; e < E; ++e) {
      src_soff[q * (E + 1) + e] = o;
      o += xplan_pad(c[q * E + e]);
    }
    src_soff[q * (E + 1) + E] = o;
  }
  if (tid == 0) {
    int32_t o = 0;
    for (int el = 0; el < El; ++el) {
      roff[el] = o;
      int64_t rows = 0;
      for (int q = 0; q < P; ++q) rows += c[q * E + me * El + el];
      o += xplan_pad(rows);
    }
    roff[El] = o;
  }
  for (int e = tid; e < E; e += nthr) {
    // owner p = e / El lays out expert e after its experts el' < e % El (each padded), then the rows of
    // the source ranks q < me
    const int p = e / El, el = e % El;
    int32_t base = 0;
    for (int j = 0; j < el; ++j) {
      int64_t rows = 0;
      for (int q = 0; q < P; ++q) rows += c[q * E + p * El + j];
      base += xplan_pad(rows);
    }
    for (int q = 0; q < me; ++q) base += c[q * E + e];
    dst_base[e] = base;
  }
}

// (source rank, source send slot) of expert-layout row r of `me`; returns false for padding rows.
LUFFY_HD bool xplan_row(int64_t r, const int32_t* cnt_all, const int32_t* roff, const int32_t* src_soff, int P, int E,
                        int me, int32_t* rank_of, int32_t* slot_of) {
  const int El = E / P;
  int el = 0;
  while (el + 1 <= El && roff[el + 1] <= r) ++el;
  const int e = me * El + el;
  int64_t i = r - roff[el];
  int q = 0;
  while (q < P && i >= cnt_all[q * E + e]) {
    i -= cnt_all[q * E + e];
    ++q;
  }
  if (q < P) {
    *rank_of = q;
    *slot_of = src_soff[q * (E + 1) + e] + (int32_t)i;
    return true;
  }
  *rank_of = -1;
  *slot_of = -1;
  return false;
}

}  // namespace luffy
