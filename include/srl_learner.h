/* srl_learner.h — the learner-side consumer of a harvested update group on the
 * GPU (sm_100a).  PAPER.md §2, P:57-85:
 *   Eq. (1) P:59-69  clipped surrogate objective, with pi_theta_old = the
 *           behaviour log-probabilities the rollout cached per token (P:180:
 *           "every token can use the exact log probability value that was used
 *           to generate each token during importance sampling") and DAPO's
 *           clip-higher bounds [1 - eps_low, 1 + eps_high];
 *   Eq. (2) P:74-80  GAE: A_t = sum_l (gamma lambda)^l delta_{t+l},
 *           delta_t = r_t + gamma V(s_{t+1}) - V(s_t);
 *   Eq. (3) P:81-85  Reinforce++: A_i = (R_i - mu_batch) / sigma_batch
 *           (population std; sigma = 0 -> all zeros).
 * The group itself (tokens, behaviour logprobs and generating versions,
 * concatenated over resumed segments) comes from srl_harvest_finished or, on
 * the device, srl_harvest_device (srl.h).
 *
 * Conventions (as srl_ops.h): every pointer is a DEVICE pointer; calls are
 * asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream);
 * the return value is 0, or < 0 for a rejected argument / launch failure
 * (srl_last_error()), in which case nothing is written.  A ragged group is
 * described by tok_off[n + 1] (int64, tok_off[0] = 0): trajectory i owns tokens
 * [tok_off[i], tok_off[i+1]).  Arithmetic is fp64 inside the kernels on fp32
 * inputs, with fixed reduction orders: results are bit-reproducible.
 */
#ifndef SRL_LEARNER_H
#define SRL_LEARNER_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Eq. (3): rewards[n] -> adv[n] (one block; n in [2, 65536]). */
int32_t srl_learner_reinforcepp(const float* rewards, int32_t n, float* adv, void* stream);

/* per_tok[t] = per_traj[i] for every token t of trajectory i (a sequence-level
 * advantage such as Eq. (3)'s applied to each of its tokens). */
int32_t srl_learner_expand(const float* per_traj, const int64_t* tok_off, int32_t n, float* per_tok, void* stream);

/* Eq. (2) per trajectory: rewards[tok_off[n]] (per token), values laid out with
 * one bootstrap entry per trajectory -- V(s_0..s_T) of trajectory i at
 * values[tok_off[i] + i .. tok_off[i+1] + i] -- gamma, lambda in [0, 1];
 * adv[tok_off[n]].  One CTA per trajectory, a parallel affine scan of the
 * backward recursion. */
int32_t srl_learner_gae(const float* rewards, const float* values, const int64_t* tok_off, int32_t n, float gamma,
                        float lambda, float* adv, void* stream);

/* Eq. (1) over n tokens: ratio[t] = exp(new_lp - old_lp); term = min(ratio A,
 * clip(ratio, 1 - eps_low, 1 + eps_high) A); dterm[t] = d term / d new_lp (ratio A on
 * the unclipped branch -- ties included -- else 0); *objective (device double) =
 * mean term.  workspace: srl_learner_ppo_workspace() bytes.  ratio / dterm may be
 * NULL.  Non-finite inputs are not checked on the device (the oracle rejects them). */
int64_t srl_learner_ppo_workspace(int64_t n);
int32_t srl_learner_ppo_objective(const float* new_lp, const float* old_lp, const float* adv, int64_t n,
                                  float eps_low, float eps_high, float* ratio, float* dterm, double* objective,
                                  void* workspace, void* stream);

/* Token staleness histogram: hist[d] = #tokens with
 * v_update - versions[t] = d, d clamped to [0, nbins - 1] (the last bin collects
 * everything >= nbins - 1).  hist[nbins] is zeroed by the call. */
int32_t srl_learner_staleness(const int32_t* versions, int64_t n, int32_t v_update, int32_t nbins, int32_t* hist,
                              void* stream);

#ifdef __cplusplus
}
#endif
#endif
