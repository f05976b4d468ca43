/*
 * TEST INFRASTRUCTURE ONLY — not part of the product path.
 *
 * Plain-C result types shared by the two CPU checkers under oracle/:
 *   - coopbatch_oracle.c : a plain-C restatement of the reference algorithm
 *                          (prefix ob_*), and
 *   - ref_capi.cpp       : an extern "C" shim over the reference's own C++
 *                          sources compiled into oracle/_ref (prefix rf_*).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.
 *
 * Layouts mirror the reference value types:
 *   ob_block    <-> coopbatch::BipartiteBlock  (samplers.hpp:30-38)
 *   ob_stack    <-> coopbatch::LayerStack      (samplers.hpp:42-49)
 *   ob_exchange <-> coopbatch::ExchangeRecord  (coop.hpp:25-37)
 *   ob_coop     <-> coopbatch::CoopSampleResult(coop.hpp:39-43)
 *   ob_sched    <-> coopbatch::SeedSchedule    (rng.hpp:93-111)
 */
#ifndef COOPBATCH_OB_TYPES_H
#define COOPBATCH_OB_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SamplerKind order of samplers.hpp:15 */
enum { OB_FULL = 0, OB_NS = 1, OB_LABOR0 = 2 };

typedef struct ob_sched {
  uint64_t kappa;
  uint64_t z1;
  uint64_t z2;
  uint64_t iteration;
} ob_sched;

typedef struct ob_block {
  int32_t layer;
  uint64_t n_dst, n_src, n_edges;
  uint32_t* dst;      /* [n_dst]                         */
  uint32_t* src;      /* [n_src] sorted unique           */
  uint32_t* edges;    /* [2*n_edges] (src_idx, dst_idx)  */
  uint32_t* dst_pos;  /* [n_dst] position of dst in src  */
} ob_block;

typedef struct ob_stack {
  int32_t num_layers;
  ob_block* blocks;
} ob_stack;

typedef struct ob_exchange {
  int32_t layer;
  uint32_t num_parts;
  uint64_t* send_counts;      /* [P*P], row p = sender          */
  uint64_t* owner_row_counts; /* [P]                            */
  uint64_t* loc_len;          /* [P] = |src_location[p]|        */
  uint32_t** loc_part;        /* [P][loc_len[p]]                */
  uint64_t** loc_row;         /* [P][loc_len[p]]                */
} ob_exchange;

typedef struct ob_coop {
  uint32_t num_parts;
  int32_t num_layers;
  ob_stack* stacks;        /* [P]        */
  ob_exchange* exchanges;  /* [L]        */
  uint64_t* owner_len;     /* [P]        */
  uint32_t** owner_sets;   /* [P][owner_len[p]] */
} ob_coop;

#ifdef __cplusplus
}
#endif
#endif
