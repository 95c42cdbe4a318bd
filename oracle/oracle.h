/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY (see oracle.c).  Declarations of the
 * plain CPU oracle.  Not included by, and shares nothing with, the CUDA path.
 */
#ifndef TSV_ORACLE_H
#define TSV_ORACLE_H
#include <stdint.h>

#define ORACLE_STATUS_BAD_TOKEN 1
#define ORACLE_STATUS_BAD_K 2
#define ORACLE_STATUS_NO_WEIGHT 4

#define ORACLE_POLICY_DRAFT 0
#define ORACLE_POLICY_PLD 1
#define ORACLE_EST_TESTED 0
#define ORACLE_EST_PROPOSED 1

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float oracle_u_acc(uint32_t x);
float oracle_u_race(uint32_t x);
float oracle_E(float u);
void oracle_E_table(float* out);

int32_t oracle_verify(const float* p, const float* q, int64_t ld, int32_t V,
                      const int32_t* row_offsets, const int32_t* draft_tokens,
                      const uint32_t* request_ids, uint64_t seed, uint32_t step,
                      int32_t B, int32_t k_max,
                      const float* inj_u_acc, const float* inj_E,
                      int32_t* num_accepted, int32_t* out_tokens);

int32_t oracle_verify_greedy(const float* p, int64_t ld, int32_t V, const int32_t* row_offsets,
                             const int32_t* draft_tokens, int32_t B, int32_t k_max,
                             int32_t* num_accepted, int32_t* out_tokens);

void oracle_softmax_rows(const float* z, int64_t ld, int32_t V, int32_t rows, float temperature,
                         float* p_out);

int32_t oracle_fit_latency(const double* ctx_tokens, const double* batched_tokens, const double* ms, int32_t n,
                           double out[3], double* r2);

void oracle_sim_target(const int32_t* proposals, int32_t K, const int32_t* k_req, int32_t B, float alpha_true,
                       int32_t V, int64_t ld, float* p_out, int32_t* row_offsets, int32_t* drafts);
void oracle_context_append(const int32_t* ctx_in, int32_t L, int32_t B, const int32_t* out_tokens,
                           const int32_t* num_accepted, int32_t k_max, int32_t* ctx_out, int32_t* ctx_len);

void oracle_lookup(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                   int32_t n_min, int32_t n_max, int32_t K,
                   int32_t* proposals, int32_t* proposal_len);

double oracle_expected_len(double alpha, int32_t k);
double oracle_forward_time(const double model[3], double n_context, double n_batched);
int32_t oracle_choose_k(const double* alpha, int32_t alpha_per_request,
                        const int32_t* ctx_len, const int32_t* cap, int32_t B, int32_t k_max,
                        int32_t policy, const double target[3], const double draft[3],
                        double pld_cost_ms, int64_t kv_free_slots, double* goodput_out);
void oracle_update(double* alpha, int32_t per_request, const int32_t* num_accepted,
                   const int32_t* row_offsets, int32_t B, double decay, int32_t estimator);

#endif
