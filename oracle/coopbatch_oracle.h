/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference (arxiv 2310.12403 "coopbatch", C++20,
 * /root/reference/proj) for the cooperative sample + dedup + feature-gather
 * path. Every function cites the reference file:line it restates. Parity of
 * this restatement is pinned against the reference's own sources compiled
 * into oracle/_ref (see oracle/Makefile, tests/test_oracle_vs_reference.py)
 * and against the committed golden vectors in tests/golden/.
 *
 * Conventions: return 0 on success, nonzero on a contract violation (the
 * reference's coopbatch::InputError); ob_last_error() holds the message.
 */
#ifndef COOPBATCH_ORACLE_H
#define COOPBATCH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "ob_types.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* ob_last_error(void);
void ob_free(void* p);

/* rng.hpp:17-48 */
uint64_t ob_mix64(uint64_t x);
uint64_t ob_hash_bits(uint64_t seed, const uint64_t* ids, int n_ids);
double ob_hash_uniform(uint64_t seed, const uint64_t* ids, int n_ids);
/* rng.cpp:7-52 */
double ob_phi(double x);
double ob_inverse_phi(double p);
double ob_normal_from_bits(uint64_t bits);
double ob_labor_variate(const ob_sched* sched, int layer, uint32_t t);
/* rng.cpp:69-86 */
void ob_sched_make(uint64_t kappa, uint64_t root_seed, ob_sched* out);
void ob_sched_advance(ob_sched* s);

/* Hash-keyed R-MAT (new; the reference has no R-MAT — DESIGN.md §Graph).
 * Allocates *indptr (n+1) and *indices (m_target) with malloc. */
int ob_rmat(uint64_t n, uint64_t m_target, uint64_t seed, uint64_t** indptr,
            uint32_t** indices);
/* Same graph as ob_rmat, built in parallel by destination bucket (large m). */
int ob_rmat_par(uint64_t n, uint64_t m_target, uint64_t seed, uint64_t** indptr,
                uint32_t** indices);
/* graph.cpp:17-48 (stable counting sort by dst, duplicates kept) */
int ob_build_csr(const uint32_t* src, const uint32_t* dst, uint64_t m,
                 uint64_t n, uint64_t* indptr, uint32_t* indices);

/* partition.cpp:10-20 */
int ob_partition_random(uint64_t n, uint32_t parts, uint64_t seed,
                        uint32_t* owner);

/* samplers.cpp:323-338 dispatch (FULL / NS / LABOR-0) */
int ob_sample_block(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                    const uint32_t* seeds, uint64_t n_seeds, int kind,
                    uint32_t fanout, const ob_sched* sched, int layer,
                    ob_block* out);
/* samplers.cpp:340-354; fanouts[l] applies at block l (NULL -> fanout) */
int ob_expand(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
              const uint32_t* seeds, uint64_t n_seeds, int num_layers, int kind,
              const uint32_t* fanouts, const ob_sched* sched, ob_stack* out);
/* coop.cpp:25-106 */
int ob_coop_sample(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                   const uint32_t* owner, uint32_t parts,
                   const uint32_t* seeds_flat, const uint64_t* seeds_off,
                   int num_layers, int kind, const uint32_t* fanouts,
                   const ob_sched* sched, ob_coop* out);
void ob_block_free(ob_block* b);
void ob_stack_free(ob_stack* s);
void ob_coop_free(ob_coop* c);

/* coop.cpp:359-376 value formula, cast once to the table dtype
 * (0 = f64 as stored by the reference, 1 = fp32, 2 = fp16 bits). */
void ob_feature_rows(uint64_t seed, uint32_t dim, int dtype, const uint32_t* ids,
                     uint64_t n_ids, void* out);

/* cache.cpp:8-32 */
typedef struct ob_lru ob_lru;
ob_lru* ob_lru_new(uint64_t capacity);
int ob_lru_access(ob_lru* c, uint32_t key); /* 1 = miss, 0 = hit */
void ob_lru_free(ob_lru* c);
/* cache.cpp:74-84 */
void ob_access_order(const uint32_t* ids, uint64_t n, uint64_t key,
                     uint32_t* out);
/* cache.cpp:123-133 */
uint64_t ob_stack_fingerprint(const ob_stack* s);
/* cli.cpp:121-139 */
int ob_draw_from_pool(const uint32_t* pool, uint64_t n_pool, uint64_t count,
                      uint64_t seed, uint64_t tag, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
