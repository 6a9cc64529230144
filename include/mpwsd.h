/*
 * mpwsd.h -- C-ABI of the B200-native MP-WSD two-stage decoder
 * (libmpwsd.so, built for sm_100a).
 *
 * This is the drop-in boundary for the reference's decoder API
 * (feclab.decoders, /root/reference/pkg/src/feclab/decoders.py):
 *
 *   mpw_set_code         <- LinearCode tables: inner info set, effective
 *                           generator, CRC (codebook.py:71-132, 261-279)
 *   mpw_set_patterns     <- CodeWeightSphere.member_words[1:] (wsphere.py:73-112)
 *   mpw_scl_batch        <- scl_decode(llrs, code, list_size)   decoders.py:181-268
 *   mpw_mpwsd_batch      <- mp_wsd(y, init_list, sphere, params) decoders.py:455-514
 *                           (also wsd_trajectory :420-452, wsd_step :401-417)
 *   mpw_two_stage_batch  <- two_stage_decode(y, code, SclStage(L), params, sphere,
 *                           sigma)                               decoders.py:520-583
 *   *_f64 variants       <- the same with the reference's float64 y (decoders.py:411,
 *                           466, 538 coerce y to float64)
 *
 * Conventions
 *   - Plain pointers and sizes; no framework types.  Buffers of the *_batch
 *     calls are DEVICE pointers on the handle's device (caller-owned);
 *     mpw_two_stage_batch_host takes HOST pointers and does the copies.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Packed bit vectors: bit j of a length-n vector is bit (j % 32) of uint32
 *     word j / 32, nw = max(1, n / 32) words per vector (the reference's uint64
 *     layout viewed as little-endian uint32, binlin.py:1-8).  Host-side code
 *     and pattern inputs are in the reference's uint64 layout.
 *   - Return 0 on success or a negative MPW_ERR_*; mpw_last_error() gives the
 *     message (thread-local).  No exception crosses the ABI.  Errors mirror the
 *     reference's ValueErrors (crc_gated without CRC, decoders.py:540-541; bad
 *     WsdParams, :80-86) plus device limits (MPW_ERR_UNSUPPORTED).
 *   - A handle is used by one host thread at a time (its stage-2 scratch and
 *     staging buffers are per handle); concurrent callers use one handle per
 *     thread, as the Python drop-in does (the reference's sweep calls the
 *     decoders from a thread pool, simharness.py:318-330).  Handles on
 *     different devices are independent.
 */
#ifndef MPWSD_H_
#define MPWSD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPW_ABI_VERSION 2

#define MPW_OK 0
#define MPW_ERR_ARG (-1)
#define MPW_ERR_STATE (-2)
#define MPW_ERR_UNSUPPORTED (-3)
#define MPW_ERR_CUDA (-4)
#define MPW_ERR_NO_DEVICE (-5)

/* activation_mode (decoders.py:78, 539) */
#define MPW_MODE_CRC_GATED 0
#define MPW_MODE_ALWAYS_ON 1

/* hop kernel selection */
#define MPW_HOP_AUTO 0
#define MPW_HOP_GATHER 1  /* shared-memory gather-sum on CUDA cores */
#define MPW_HOP_TENSOR 2  /* tcgen05, one fp16 limb of t, certified top-6 */
#define MPW_HOP_TENSOR_2LIMB 3 /* tcgen05, fp16 hi+lo limbs of t, certified top-6 */
#define MPW_HOP_TENSOR_I8 4 /* tcgen05 kind::i8, per-frame int8 quantisation of t, certified top-14 (N = 128, 256) */
#define MPW_HOP_TENSOR_I8_ASYNC 5 /* kind::i8 with asynchronous rows: continuous P stream, group-minimum scan, worker-warp decisions (N = 128, 256; float32 and float64 received words) */

/* counters (int64, accumulated by mpw_two_stage_batch; caller zeroes) */
#define MPW_CTR_FRAMES 0
#define MPW_CTR_ERRORS 1      /* decoded codeword != tx codeword (simharness.py:311) */
#define MPW_CTR_ACTIVATIONS 2 /* stage == mp_wsd (simharness.py:309) */
#define MPW_CTR_ITERATIONS 3  /* sum of iterations_used over trajectories */
#define MPW_CTR_EVALS 4       /* pattern-metric evaluations = |P| * iterations */
#define MPW_CTR_NEAR_TIE 5    /* frames carrying a near-tie report flag (bits 1|2|4) */
#define MPW_CTR_UNRESOLVED 6  /* frames carrying MPW_FLAG_UNRESOLVED */
#define MPW_NUM_COUNTERS 8

/* per-frame flags.  Hop decisions are certified: fp32 (or fp16-limb tensor)
 * scores whose top-2 gap or accept margin fall inside the error window are
 * re-scored in float64, so bits 1|2|4 only REPORT near-ties (exact relative
 * ED gap < 1e-5, the BASELINE north-star definition); bit 8 marks a scan in
 * which a third candidate was also inside the window (decision not certified). */
#define MPW_FLAG_TIE_ARGMIN 1 /* exact top-2 hop candidates within 1e-5 relative ED */
#define MPW_FLAG_TIE_ACCEPT 2 /* exact ED change of the best hop within 1e-5 relative of 0 */
#define MPW_FLAG_TIE_FINAL 4  /* two distinct final centres within 1e-5 relative (float64) */
#define MPW_FLAG_UNRESOLVED 8 /* >= 3 hop candidates inside the certification window */
#define MPW_FLAG_TIE_STAGE1 16 /* OSD: list order decided by candidates within the rounding bound */

typedef struct mpw_handle mpw_handle;

int mpw_version(void);
const char* mpw_last_error(void);

int mpw_create(int device, mpw_handle** out);
void mpw_destroy(mpw_handle* h);

/* Code tables.  info_set: kp ascending positions of the inner polar code;
 * gen_words: k x ceil(n/64) uint64 rows of the effective generator (the CA
 * generator for CRC-concatenated codes); crc_poly bit i = coefficient of x^i
 * (including x^crc_deg).  is_ca = 0 for a plain polar code (no gate, anchors
 * are the list codewords as-is, decoders.py:574-575). */
int mpw_set_code(mpw_handle* h, int n, int k, int kp, const int32_t* info_set,
                 const uint64_t* gen_words, int is_ca, int crc_deg, uint32_t crc_poly);

/* Pattern set P: np x ceil(n/64) uint64 words, the nonzero sphere members in
 * member order (pattern index = member index - 1). */
int mpw_set_patterns(mpw_handle* h, const uint64_t* pattern_words, int np);

/* Stage 1 alone.  Either y (F x n float32 received words; LLRs are 2y/sigma^2
 * in float64, decoders.py:550) or llr (F x n float64 LLRs, the scl_decode
 * argument) is given.  Outputs (any may be NULL): list_n[F];
 * list_u/list_cw: F x L x nw; list_pm: F x L float64, list in ascending PM. */
int mpw_scl_batch(mpw_handle* h, const float* y, const double* llr, int F, double sigma, int L,
                  int32_t* list_n, uint32_t* list_u, uint32_t* list_cw, double* list_pm,
                  void* stream);

/* Stage 2 alone from given anchors (F x A x nw); n_anchor[F] may be NULL (= A).
 * Outputs: best F x nw, best_ed F (float64 canonical), iters F x A,
 * hops F x A x T (accepted member index per hop, -1 = none; may be NULL),
 * flags F (may be NULL). */
int mpw_mpwsd_batch(mpw_handle* h, const float* y, const uint32_t* anchors, const int32_t* n_anchor,
                    int F, int A, int T, int variant, uint32_t* best, double* best_ed,
                    int32_t* iters, int32_t* hops, uint8_t* flags, void* stream);
/* Same with float64 received words (F x n): the screens run on their fp32
 * rounding with error bounds widened by the rounding, every exact re-scoring
 * and reported ED uses the float64 values (variant AUTO, TENSOR_I8_ASYNC, TENSOR
 * or GATHER). */
int mpw_mpwsd_batch_f64(mpw_handle* h, const double* y, const uint32_t* anchors, const int32_t* n_anchor,
                        int F, int A, int T, int variant, uint32_t* best, double* best_ed,
                        int32_t* iters, int32_t* hops, uint8_t* flags, void* stream);

/* The full two-stage path.  stage[F]: 0 = stage1_crc_pass, 1 = mp_wsd.
 * tx_cw (F x nw, may be NULL) enables the error counter.  best_msg[F]
 * (k <= 64 bits, may be NULL) = code.message_of(best).  anchors_out
 * (F x A x nw, may be NULL) returns the projected anchors. */
int mpw_two_stage_batch(mpw_handle* h, const float* y, int F, double sigma, int L, int A, int T,
                        int mode, int variant, const uint32_t* tx_cw, uint32_t* best,
                        uint64_t* best_msg, double* best_ed, uint8_t* stage, int32_t* iters,
                        int32_t* hops, uint32_t* anchors_out, uint8_t* flags,
                        unsigned long long* counters, void* stream);
/* Same with float64 received words (F x n): stage 1 from the float64 LLRs
 * 2.0 * y / (sigma * sigma) (decoders.py:550), stage 2 as mpw_mpwsd_batch_f64. */
int mpw_two_stage_batch_f64(mpw_handle* h, const double* y, int F, double sigma, int L, int A, int T,
                            int mode, int variant, const uint32_t* tx_cw, uint32_t* best,
                            uint64_t* best_msg, double* best_ed, uint8_t* stage, int32_t* iters,
                            int32_t* hops, uint32_t* anchors_out, uint8_t* flags,
                            unsigned long long* counters, void* stream);

/* Two-stage decode with order-k OSD as stage 1 (decoders.py:274-317, 555-556;
 * the paper's RM initialiser).  list_cap <= 0 means no cap.  OSD candidates
 * are codewords of the code itself: in crc_gated mode the first (minimum-ED)
 * entry passes the gate; in always_on mode the first A entries are the
 * anchors, unprojected (decoders.py:573-576).  Outputs as mpw_two_stage_batch;
 * flags gain MPW_FLAG_TIE_STAGE1 when two OSD candidates that decide the
 * list order are within the float64 rounding bound. */
int mpw_two_stage_osd_batch(mpw_handle* h, const float* y, int F, int order, int list_cap, int A,
                            int T, int mode, int variant, const uint32_t* tx_cw, uint32_t* best,
                            uint64_t* best_msg, double* best_ed, uint8_t* stage, int32_t* iters,
                            int32_t* hops, uint32_t* anchors_out, uint8_t* flags,
                            unsigned long long* counters, void* stream);

/* Order-k OSD list (decoders.py:274-317) for F frames (device buffers):
 * list_n[F], list_cw[F x M x nw], list_ed[F x M] in ascending squared-ED
 * order, ties to the lower candidate index, M = min(list_cap, C) (list_cap <= 0:
 * M = C = sum_{w<=order} C(k, w)).  flags[F] (may be NULL): MPW_FLAG_TIE_STAGE1
 * when adjacent entries within the first M + 1 are closer than the rounding
 * bound.  k <= 63, order <= 16, n in {32, 64, 128, 256}. */
int mpw_osd_batch(mpw_handle* h, const float* y, int F, int order, int list_cap, int32_t* list_n,
                  uint32_t* list_cw, double* list_ed, uint8_t* flags, void* stream);

/* Same with HOST buffers; H2D/D2H copies are made on `stream` and the call
 * returns after the results are on the host. */
int mpw_two_stage_batch_host(mpw_handle* h, const float* y_host, int F, double sigma, int L, int A,
                             int T, int mode, int variant, const uint32_t* tx_host,
                             uint32_t* best_host, uint64_t* msg_host, double* ed_host,
                             uint8_t* stage_host, int32_t* iters_host, uint8_t* flags_host,
                             unsigned long long* counters_host, void* stream);

/* Per-kernel CUDA-event timing of mpw_two_stage_batch: ms_out[4] =
 * {stage 1, stage 2 hops, finalize, frame epilogue}. */
int mpw_set_timing(mpw_handle* h, int enable);
/* Options: "scl_generic" (1 = force the warp-per-frame stage-1 kernel instead of
 * the lane-per-path one; both are bit-exact), "timing" (same as mpw_set_timing);
 * tensor-hop variants for A/B runs and tests: "i8_cluster" (2 = CTA pairs
 * sharing the P stream), "i8_pair" (1 = cta_group::2 pair MMAs), "f16_cluster"
 * (0 = single CTAs for the 1-limb N = 256 shape), "hop_experiment" (profiling
 * and test bits of the hop kernels, e.g. 2048 = int8 window overflow at 4 keys;
 * for the asynchronous-row hop: 32 = cycles per tile of the production kernel
 * on stderr, other non-zero values = the instrumented build), "ar_hit_cap"
 * (asynchronous-row hop: hit-list entries per scan thread and cycle, 0 = the
 * compiled maximum; small values force the re-scan path in tests). */
int mpw_set_option(mpw_handle* h, const char* key, int value);
int mpw_read_timing(mpw_handle* h, double* ms_out, long long* launches_out, int reset);
/* Asynchronous-row hop: out[0] = 256-pattern tiles streamed, out[1] = SM clock cycles of
 * the streaming loop, both summed over the CTAs of every launch since the last reset
 * (synchronises the device).  cycles / tiles against 1,024 (the MMA time of a tile) and
 * scans x tiles-per-scan against tiles x 128 rows (the rows' live share) explain the
 * bench's roofline fraction. */
int mpw_hop_tile_stats(mpw_handle* h, unsigned long long* out, int reset);

/* Device-side channel generator for bulk sweeps: frames [first_frame,
 * first_frame + F) of the counter-based Philox4x32-10 stream (seed, snr_idx):
 * uniform message bits, codeword through the code's generator, BPSK + AWGN
 * (float64 Box-Muller, rounded to float32).  Outputs (device): y F x n,
 * tx F x nw (may be NULL), msg F (k <= 64, may be NULL).  Mirrors
 * paper_2602_08501_b200.channel.keyed_inputs_host. */
int mpw_channel_batch(mpw_handle* h, uint64_t seed, int snr_idx, long long first_frame, int F,
                      double sigma, float* y, uint32_t* tx, uint64_t* msg, void* stream);

int mpw_num_patterns(mpw_handle* h);
/* Number of kernels this handle has launched (all entry points). */
long long mpw_launch_count(mpw_handle* h);
int mpw_tensor_path_ready(mpw_handle* h);
/* The hop variant MPW_HOP_AUTO resolves to for the current code and pattern set. */
int mpw_hop_auto_variant(mpw_handle* h);

/* Host-side pattern-set generation (off the timed path). */
int64_t mpw_enumerate_lowweight(const uint64_t* gen, int k, int n, int cap, int64_t* spectrum,
                                uint64_t* out, int64_t out_cap, int nthreads);
/* Same on the GPU (exhaustive, k <= 40) for the code set on `h`: the reference's
 * enumerate_spectrum / build_sphere (wsphere.py:115-208).  spectrum[n+1]
 * (host, may be NULL) gets the full weight distribution A_w; out (host,
 * out_cap x ceil(n/64) words) the codewords with 1 <= weight <= cap, in no
 * particular order (the caller sorts into CWS1 member order).  Returns the
 * number of such codewords (may exceed out_cap: only out_cap are written). */
int64_t mpw_enumerate_lowweight_gpu(mpw_handle* h, int cap, int64_t* spectrum, uint64_t* out,
                                    int64_t out_cap);
int64_t mpw_collect_lowweight(const uint64_t* gen, int k, int n, int cap, int64_t iterations,
                              uint64_t seed, int p_max, uint64_t* out, int64_t out_cap,
                              int nthreads);

#ifdef __cplusplus
}
#endif

#endif /* MPWSD_H_ */
