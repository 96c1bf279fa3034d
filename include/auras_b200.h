/*
 * auras_b200.h -- C ABI of the B200-native Auras hot path.
 *
 * Plain C: device pointers, host pointers, sizes and an opaque cudaStream_t
 * passed as `void *`.  No torch / C++ types cross this boundary.  Every entry
 * point launches asynchronously on the given stream and returns 0 on success
 * or a negative AURAS_E_* code (the Python host maps codes onto the
 * reference's FramepipeError tree, fp/errors.py:4-95).
 *
 * Each function names the reference interface it replaces.  Reference paths
 * are relative to /root/reference; fp/ = pkg/src/framepipe/.
 */
#ifndef AURAS_B200_H
#define AURAS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
#define AURAS_OK 0
#define AURAS_E_CUDA (-1)          /* CUDA runtime error (see auras_last_error) */
#define AURAS_E_ARG (-2)           /* invalid argument / unsupported shape       */
#define AURAS_E_ARCH (-3)          /* device is not sm_100                      */

/* Last error message (thread-local, static storage). */
const char *auras_last_error(void);
/* ABI version; bumped whenever a struct below changes layout. */
int auras_abi_version(void);
/* 1 when the loaded device is compute capability 10.0 (B200). */
int auras_device_ok(int device);

/* -------------------------------------------------- public-context ring
 * Replaces ContextStore (fp/context.py:98-175).  The ring lives in HBM:
 *   payload  : K slots of `slot_bytes` bytes (written by producer kernels)
 *   meta     : int64[K][2] = {frame, version} per slot, released last
 *   state    : int64[4]    = {global version, last frame, publish count, err}
 */

/* ContextStore.publish (fp/context.py:129-143): release-store the slot's
 * {frame, version} after the payload stores that precede it on `stream`;
 * bumps the device version counter.  `expected_version` is the host mirror's
 * version; a mismatch sets state[3]. */
int auras_ring_commit(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                      int64_t expected_version, void *stream);

/* ContextStore.fetch_entry / latest_entry (fp/context.py:145-164), resolved
 * on the device: acquire-load the slot meta of frame `target`; if it does not
 * hold `target` fall back to the newest slot (fp/executor.py:314-316).  Writes
 * {slot, version, frame} to `out` (int64[3]) for in-kernel consumers and
 * appends `version` at `version_log[log_index]`. */
int auras_ring_fetch(const int64_t *meta, const int64_t *state, int capacity, int64_t target,
                     int64_t *out, int64_t *version_log, int64_t log_index, void *stream);

/* Disaggregated variant (perception GPU != generation GPU): the same commit
 * with a system-scope release so a consumer on another GPU (or a peer-mapped
 * reader) observes the payload before the version. */
/* Stress test of the ring's publish/fetch ordering (test support; replaces the
 * threaded torn-read test of t/test_context_store.py:148-183 / fp/verify.py:83-123
 * on the device).  One writer block publishes n_versions into a `capacity`-slot
 * ring of `words` fp64 words with commit_slot's order while `readers` blocks
 * fetch the newest entry seqlock-style.  Synchronous.  counts_host receives
 * [readers][4] = {consistent reads, retries, torn reads, version regressions}. */
int auras_ring_stress(int capacity, int words, int n_versions, int readers, unsigned long long *counts_host);
/* Action emission (replaces the host-side copy of GenerationModel.finish's result,
 * fp/policy.py:230-246): pinned host memory mapped into the device address space; kernels write
 * through *dev, the host reads *host once the writing kernel completed. */
int auras_host_mapped_alloc(size_t bytes, void **host, void **dev);
int auras_host_mapped_free(void *host);

int auras_ring_commit_sys(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                          int64_t expected_version, void *stream);

/* Enable peer access from `device` to `peer` (idempotent). */
int auras_enable_peer(int device, int peer);

/* Asynchronous pitched copy of `rows` x `width` bytes between device buffers
 * that may live on different GPUs (unified addressing; NVLink P2P once
 * auras_enable_peer was called), enqueued on `stream`.  Used to ship a
 * perception GPU's staged context slots into the generation GPU's ring. */
int auras_peer_copy(void *dst, int64_t dst_pitch, const void *src, int64_t src_pitch, int64_t width,
                    int64_t rows, void *stream);

/* Copy `bytes` from device `src` into slot `slot` of the payload ring
 * (ContextStore.publish of a host-built PublicContext). */
int auras_ring_write(void *payload, int64_t slot_bytes, int slot, const void *src,
                     int64_t bytes, void *stream);

/* -------------------------------------------------- toy refinement policy
 * The reference's own conditioning policy (fp/policy.py:217-246, 279-297) in
 * fp64 on the device, bit-exact with numpy: x <- x + eta*(H - x). */

/* PerceptionModel.start + identity apply_layers (fp/policy.py:76-85): store
 * the 4-vector observation (host values, passed by value) into lane `lane`. */
int auras_toy_ingest(double *latent, int lane, const double obs[4], double *x_state,
                     const double x0[2], void *stream);

/* PerceptionModel.finalize + ContextStore.publish (fp/policy.py:285-290,
 * fp/context.py:129-143): H = latent[:2] - latent[2:4] into ring slot
 * frame % capacity, then commit {frame, version}. */
int auras_toy_publish(const double *latent, int lane, double *ring_payload, int64_t *meta,
                      int64_t *state, int capacity, int64_t frame, int64_t version,
                      void *stream);

/* The stage iteration loop (fp/executor.py:325-331): for each of `n` active
 * requests run iters[i] refinement steps on lane lanes[i], all reading the
 * single context fetched by auras_ring_fetch (`fetched` = {slot,version,frame}). */
int auras_toy_generate(double *x_state, const int *lanes, const int *iters, int n, double eta,
                       const double *ring_payload, const int64_t *fetched, void *stream);

/* GenerationModel.finish norm clip (fp/policy.py:240-244) into out[2]. */
int auras_toy_finish(const double *x_state, int lane, double max_action, double *out,
                     void *stream);

/* Scripted token policy (fp/policy.py:110-161, 300-327): tokens[lane][p] for
 * p in [starts[i], starts[i] + counts[i]) of each request lane, from the
 * displacement in the fetched ring slot (`fetched` = {slot, version, frame});
 * replaces GenerationModel.step for autoregressive contexts (:217-228). */
int auras_ar_generate(int *tokens, int l_a, const int *lanes, const int *starts, const int *counts, int n,
                      const double *ring_payload, const int64_t *fetched, double max_action, void *stream);
/* GenerationModel.finish for token policies: the lane's l_a tokens -> out (as doubles). */
int auras_ar_finish(const int *tokens, int lane, int l_a, double *out, void *stream);
/* Payload half of ContextStore.update_action_tokens (fp/context.py:166-175):
 * the newest context's payload re-published into another slot (the version
 * is released by auras_ring_commit). */
int auras_ring_copy_slot(double *payload, int elems, int src, int dst, void *stream);

/* -------------------------------------------------- causal transformer (AR)
 * fp64 pre-norm causal transformer with its KV cache in HBM
 * (fp/transformer.py:69-211): the model of the autoregressive merged prefill.
 * `params` packs, in order: tok_emb [vocab,d], pos_emb [max_len,d], per layer
 * {ln1_g, ln1_b [d], wq, wk, wv, wo [d,d], ln2_g, ln2_b [d], w1 [d,4d],
 * b1 [4d], w2 [4d,d], b2 [d]}, lnf_g, lnf_b [d]. */
int64_t auras_tf_param_count(int d_model, int n_heads, int n_layers, int vocab, int max_len);
/* Rows [start, start+n) of a sequence whose rows [0, start) are in `kv`
 * ([layers][2][max_len][d]): prefill (start 0; CausalTransformer.prefill /
 * prefill_embedded, :106-143), decode (n 1; :147-173) and the merged prefill
 * (:175-193).  Input rows are token ids (`token_ids`) or embeddings
 * (`embeddings` [n,d]); `resid`, `qbuf` are [n,d] scratch; `hidden` [n,d]
 * receives the final-LN hidden states. */
int auras_tf_forward(const double *params, int d_model, int n_heads, int n_layers, int vocab, int max_len,
                     const int *token_ids, const double *embeddings, int start, int n,
                     double *kv, double *resid, double *qbuf, double *hidden, void *stream);
/* logits = hidden @ tok_emb^T (:207-208) and the greedy token (:210-211);
 * either output may be NULL. */
int auras_tf_logits(const double *params, int d_model, int vocab, const double *hidden, int n,
                    double *logits, int *argmax, void *stream);

/* -------------------------------------------------- diffusion policy (DP)
 * Replaces PerceptionModel / GenerationModel arithmetic for the Diffusion
 * Policy CNN plugin.  The host builds a program of
 * conv ops once; every op is an implicit-GEMM convolution
 *    out[s, oy, ox, m] = sum_{ky,kx,c} W[m, ky, kx, c] * in[s, oy*st-ph+ky, ox*st-pw+kx, c]
 * followed by a fused epilogue (split-K reduce, bias, GroupNorm, activation,
 * FiLM, residual, optional zero-stuffed / pooled store). */

#define AURAS_DT_F32 0
#define AURAS_DT_BF16 1

#define AURAS_ACT_NONE 0
#define AURAS_ACT_RELU 1
#define AURAS_ACT_MISH 2
#define AURAS_ACT_GELU 3          /* exact erf GELU (ViT MLP)                                */

typedef struct auras_conv_op {
  /* operands (device pointers; element type = plan dtype) */
  const void *w;          /* [M][Kp], K index = (ky*kw + kx)*Cin + c, zero padded to Kp */
  const float *bias;      /* [M] or NULL                                            */
  const void *in;         /* NHWC view: elem(s,y,x,c) = in[((s*H + y)*W + x)*in_pitch + in_coff + c] */
  void *out;              /* NHWC view of the output                                 */
  const float *gn_gamma;  /* [M] or NULL (no GroupNorm)                              */
  const float *gn_beta;   /* [M]                                                     */
  const void *res;        /* residual tensor (same type/shape as out view) or NULL   */
  const float *res_f32;   /* residual as fp32 rows [S][Ho*Wo][M] or NULL             */
  float *out_f32;         /* if non-NULL: also store the pre-residual result fp32    */
  /* shapes */
  int32_t M, Cin, Kp;
  int32_t H, W, in_pitch, in_coff;
  int32_t kh, kw, stride, pad_h, pad_w;
  int32_t Ho, Wo, out_pitch, out_coff;
  int32_t res_pitch, res_coff;
  int32_t groups;         /* GroupNorm groups (ignored without gamma)                */
  int32_t act;            /* AURAS_ACT_*                                             */
  int32_t res_before_act; /* 1: act(gn(y) + res) (ResNet); 0: act(gn(y)) + res (UNet) */
  int32_t film_off;       /* >=0: FiLM scale at film_off, bias at film_off+M          */
  int32_t out_stuff;      /* 1: write out row 2*ox and a zero row 2*ox+1 (1-D only)  */
  int32_t pool_out;       /* 1: store mean over Ho*Wo as out[s][m] (fp32, out_f32)    */
  int32_t splits;         /* split-K factor chosen by the planner                    */
  int32_t cta_target;     /* gathered-im2col engine: CTAs to aim for (0 = 32)        */
  int32_t reserved[2];
} auras_conv_op;

/* Linear / GEMV: y[n][m] = sum_k W[m][k] * f(x[n][k]) + b[m], f = Mish or id. */
typedef struct auras_linear_op {
  const void *w;          /* [M][K] plan dtype */
  const float *bias;      /* [M] or NULL       */
  int32_t M, K;
  int32_t mish_in;        /* apply Mish to the input first */
  int32_t ldw;            /* weight row stride in elements (multiple of 8, >= K) */
} auras_linear_op;

/* Diffusion scheduler tables (DDPM / DDIM, computed on the host in fp64 and
 * uploaded once): per inference step i,
 *   timestep[i], c_x0[i], c_xt[i], c_eps[i] (DDIM), sigma[i] (DDPM),
 *   sqrt_ab[i], sqrt_1mab[i]. */
typedef struct auras_sched {
  const int32_t *timestep;
  const float *sqrt_ab, *sqrt_1mab, *c_x0, *c_xt, *c_eps, *sigma;
  int32_t n_steps;
  int32_t clip_sample;
  int32_t ddpm;           /* 1: add sigma_i * noise_i */
  int32_t reserved;
} auras_sched;

/* A compiled UNet program (opaque handle). */
typedef struct auras_unet_plan auras_unet_plan;

/* Build the plan: `ops` in execution order; `dtype` AURAS_DT_*; `s_max` the
 * largest batch of samples per step; scratch is allocated inside.  The FiLM
 * time table `film_tau` is [n_train][film_width] fp32; the FiLM row of
 * (agent a, ring slot k) is at ring_film + a*ring_agent_stride +
 * k*ring_slot_stride (floats).  `final_w`/`final_b` is the final 1x1 conv
 * (action_dim x C0).  `x_in_op` is the index of the op whose input is the
 * noisy action buffer. */
auras_unet_plan *auras_unet_plan_create(const auras_conv_op *ops, int n_ops, int dtype,
                                        int s_max, int horizon, int action_dim,
                                        const float *film_tau, const float *ring_film,
                                        int film_width, int64_t ring_slot_stride,
                                        int64_t ring_agent_stride,
                                        const void *final_w, const float *final_b,
                                        int final_cin, const auras_sched *sched,
                                        void *x_in_buffer, int x_in_pitch);
void auras_unet_plan_destroy(auras_unet_plan *plan);

/* The batched, staggered-timestep denoise chain for one frame
 * (fp/executor.py:318-349 + GenerationModel.step fp/policy.py:217-228):
 * sample s works on request lane lanes[s] of agent agents[s], starting at
 * inference step start[s] and running count[s] steps; `iters` = max(count).
 * Every sample reads FiLM rows from ring slot fetched[agents[s]*3] (written
 * by auras_ring_fetch).  x_lanes: [A][R][horizon][action_dim] fp32,
 * noise_lanes: [A][R][n_steps][horizon][action_dim] fp32 (DDPM) or NULL.
 * use_graph: capture the iteration chain into a CUDA graph (cached per
 * (S, iters)). */
int auras_unet_generate(auras_unet_plan *plan, int S, const int *lanes, const int *agents,
                        const int *start, const int *count, int iters, int lanes_per_agent,
                        float *x_lanes, const float *noise_lanes, const int64_t *fetched,
                        int use_graph, void *stream);

/* Kernel launches one denoise iteration issues (megakernel path: the
 * persistent step kernel + the iteration advance; layer path: prep, a GEMM and
 * an epilogue per conv op, final, advance).  Negative on error. */
/* Denoise-step engine used for batch size S: 0 layer-by-layer kernels,
 * 1 persistent megakernel with split-K through L2, 2 cluster megakernel
 * (DSMEM split-K + GroupNorm), -1 not chosen yet (picked by a timed dry run
 * of both persistent kernels on the first generate of that S). */
/* Health of the persistent denoise kernels (no reference counterpart: the
 * reference's deadlock guard is executor.py:311-313 on the host).  0 = fine,
 * 1 = a device-side dependency wait timed out (surfaced as DeadlockDetected),
 * < 0 = error.  Synchronous; reads and clears the error word. */
int auras_unet_check(auras_unet_plan *plan);
int auras_unet_kernel_for(const auras_unet_plan *plan, int S);

int auras_unet_launches_per_iter(const auras_unet_plan *plan);

/* Diagnostics: per-task globaltimer trace of the persistent denoise
 * megakernel for batch size S (trace: int64[n_tasks][8]; tasks_out:
 * int32[n_tasks][4] task table or NULL).  Returns n_tasks or < 0. */
int auras_unet_mega_trace(auras_unet_plan *plan, int S, long long *trace, int *tasks_out,
                          int max_tasks);

/* One conv op (standalone; used by the perception encoder and by tests). */
int auras_conv(const auras_conv_op *op, int dtype, int S, const float *film_rows,
               int film_stride, float *scratch, int64_t scratch_floats, void *stream);

/* auras_conv for a plain token-wise linear layer followed by LayerNorm
 * (out = act(W x + b) + res, ln_out = LayerNorm(out) with eps): the DP-T
 * decoder's residual adds fused with the next layer norm.  bf16, M <= 1024. */
int auras_conv_ln(const auras_conv_op *op, int dtype, int S, const float *ln_gamma, const float *ln_beta,
                  void *ln_out, int ln_pitch, float eps, float *scratch, int64_t scratch_floats, void *stream);

/* fp32 scratch floats auras_conv needs for this op at batch S (the engine
 * picks its own split-K factor). */
int64_t auras_conv_scratch_floats(const auras_conv_op *op, int dtype, int S);

/* Linear / GEMV for N input rows: y[n][m] (fp32, row stride ldy). */
int auras_linear(const auras_linear_op *op, int dtype, int N, const float *x, int ldx,
                 float *y, int ldy, void *stream);

/* Perception helpers (K1): uint8 CHW frames -> dtype NHWC in [-1, 1] padded
 * to `cpad` channels; 3x3/s2/p1 max pool on NHWC. */
int auras_image_to_nhwc(const uint8_t *img, int S, int C, int H, int W, void *out, int cpad,
                        int dtype, void *stream);
int auras_maxpool3s2(const void *in, int S, int H, int W, int C, void *out, int dtype,
                     void *stream);

/* ViT-B/16 perception (BASELINE configs[3]): the non-GEMM
 * parts of a pre-norm block.  Patch embedding and linear layers use auras_conv
 * (16x16/s16 and 1x1 kernels over the token axis).  Token rows are bf16
 * [S][N][C] (rows n_valid..N-1 of an image are zero padding); q|k|v rows
 * [S][N][3C] in timm's (3, heads, dh) order. */
int auras_vit_tokens(const void *patches, const float *cls, const float *pos, void *x, int S, int N, int n_valid,
                     int C, void *stream);
/* Per-row LayerNorm with fp32 statistics; out bf16 (out_f32 = 0) or fp32. */
int auras_layernorm(const void *in, int64_t ldi, void *out, int64_t ldo, int out_f32, const float *gamma,
                    const float *beta, int rows, int C, float eps, void *stream);
/* softmax(q k^T / sqrt(dh)) v for every (image, head) over the first n_valid
 * of N token rows (the rest are padding); dh <= 64. */
int auras_vit_attention(const void *qkv, void *out, int S, int N, int n_valid, int heads, int dh, void *stream);

/* DP-T denoiser (TransformerForDiffusion; BASELINE configs[3]): the pieces
 * around the conv-path GEMMs.  Samples are (agent, lane, inference step);
 * x lanes / noise lanes / scheduler tables as for the UNet plan. */
int auras_dpt_prep(const int *agents, const int *lanes, const int *steps, int S, const float *x_lanes,
                   int lanes_per_agent, int horizon, int adim, void *xin, const float *ring,
                   int64_t ring_agent_stride, int slot_floats, const int64_t *fetched, int tok_w, int n_obs,
                   void *gcbuf, int gpad, const float *temb, int E, void *c, const float *cond_pos, void *stream);
int auras_dpt_cond(const void *cobs, void *c, const float *cond_pos, int S, int n_obs, int E, void *stream);
/* kv2[s] = [kvt[steps[s]]; kvo[agents[s]][0..tc-2]]: rows of lw bf16 (the
 * cross-attention K|V of every layer), time row by inference step, observation
 * rows computed once per frame. */
int auras_dpt_kv_gather(void *kv2, const void *kvt, const void *kvo, const int *agents, const int *steps, int S,
                        int tc, int lw, void *stream);
/* softmax(q k^T / sqrt(dh) + mask) v, key j visible to query n iff
 * j <= n + mask_off; rows (s * Nq + n) * ld + head * dh; Nk <= 32. */
int auras_attention(const void *q, int ldq, const void *k, int ldk, const void *v, int ldv, void *out, int ldo,
                    int S, int Nq, int Nk, int heads, int dh, int mask_off, void *stream);
int auras_dpt_update(const float *eps, int eps_pitch, const int *agents, const int *lanes, const int *steps, int S,
                     float *x_lanes, const float *noise_lanes, int lanes_per_agent, int horizon, int adim,
                     const auras_sched *sched, void *stream);

/* Persistent DP-T iteration (csrc/dpt_persist.cu): one launch of one 8-CTA
 * cluster runs a whole denoise iteration of up to 128 action tokens (8 samples
 * x horizon 16) as a program of phases -- GEMM (tcgen05, CTA r owns columns
 * [r N/8, (r+1) N/8)), LayerNorm, attention, scheduler update -- separated by
 * cluster barriers.  Replaces the ~110 launches per iteration of the program
 * built from auras_conv / auras_layernorm / auras_attention / auras_dpt_update
 * (GenerationModel.step of the transformer policy, fp/policy.py:217-228).
 * Every pointer is device memory. */
typedef struct auras_dpt_gemm {
  const void *act;          /* A: [act_rows = 128][K] bf16 (tokens x channels) */
  int act_rows, K;          /* K % 64 == 0 */
  const void *w;            /* W: [N][K] bf16 */
  int N;                    /* N % 128 == 0 (8 CTAs x 16k columns) or N <= 16 (one CTA) */
  const float *bias;        /* [N] */
  const void *res;          /* optional bf16 residual [rows][ldr] (may alias out) */
  int ldr;
  void *out;                /* optional bf16 output [rows][ldo] */
  int ldo;
  float *out_f32;           /* optional fp32 output [rows][ldf] */
  int ldf;
  int act_fn;               /* AURAS_ACT_* applied before the residual */
  const void *ln_src;       /* optional: A = LayerNorm(ln_src [128][256] bf16; ln_g, ln_b), computed in the
                               GEMM phase itself (act is then ignored; K = 256) */
  const float *ln_g, *ln_b;
  int ksplit;               /* 1: K split over the cluster's two 8-CTA halves (CTA r: K half r / 8, columns
                               [(r % 8) N/8, +N/8)), the halves' partials summed over DSMEM -- each CTA
                               receives half the A operand (plain A, bf16 out, N / 8 % 16 == 0, K % 128 == 0) */
  int fuse_update;          /* 1 (the single-CTA action head, N = action dim <= 16, fp32 out): the DDPM / DDIM
                               update of every sample's request lane runs in this GEMM's epilogue (the
                               program then needs no type-3 op) */
  int a_from_lanes;         /* 1 (K = 64): A = every sample's action tokens bf16(x[t][a]) read straight from
                               its request lane into the UMMA tile (the program then needs no type-5 op) */
} auras_dpt_gemm;
typedef struct auras_dpt_op {
  int type;                 /* 0 GEMM, 1 LayerNorm (E = 256), 2 attention, 3 scheduler update, 4 no-op,
                               5 prep: the action tokens of every sample into out ([S T][64] bf16),
                               6 folded cross-attention block (auras_dpt_xfold tables): in = out = the
                               residual stream [rows][ldi] bf16, updated in place, h += ca_out(MHA(LN(h), mem));
                               k = the time-token table (float rows of ldk, row steps[s]), v = the
                               observation table (float rows of ldv, rows agents[s] * (nk - 1) + j - 1),
                               each pointing at the layer's block; nk <= 4 memory tokens, heads == 4;
                               without g: out == in; with g, b: the row is written back to in and its
                               LayerNorm(g, b) to out (bf16 [rows][ldo]), the A of a following plain GEMM */
  int gemm;                 /* GEMM: index into the gemm table */
  const void *in;           /* LN input rows / attention q */
  void *out;                /* LN output rows / attention output */
  const float *g, *b;       /* LN affine */
  const void *k, *v;        /* attention keys / values: rows (s * nk + j) */
  int ldi, ldo, ldk, ldv, nk, mask_off, heads, dh;
  int qrows, krows;         /* attention: rows of the q buffer / of the k, v buffers (TMA bounds) */
  const void *k2, *v2;      /* attention, gather = 1: k / v row 0 is row steps[s] of (k, v) (the time table),
                               rows 1 .. nk - 1 are rows agents[s] * (nk - 1) .. of (k2, v2) (observation rows) */
  int k2rows, gather;
} auras_dpt_op;
int auras_dpt_persist_build(const auras_dpt_gemm *gemms, int n_gemms, const auras_dpt_op *ops, int n_ops, int T,
                            void **plan);
int auras_dpt_persist_run(void *plan, int S, const float *eps, int eps_pitch, const int *agents, const int *lanes,
                          const int *steps, float *x_lanes, const float *noise_lanes, int lanes_per_agent,
                          int horizon, int adim, const auras_sched *sched, void *stream);
int auras_dpt_persist_trace(void *plan, long long *out, int n);   /* diagnostics (AURAS_DPT_TRACE) */
/* Cross-attention folded into per-memory-token vectors (the memory has only
 * 1 + n_obs tokens, so ca_in's query projection and ca_out fold into the keys
 * and values): for every kv row r (bf16, layer l's K at l*2E, V at l*2E + E),
 * layer l and head h, out[r][l] holds
 *   a'[h][e] = ln_g[e] * sum_d Wq[h dh + d][e] k[h dh + d] / sqrt(dh)   (H x E)
 *   U'[h][e] = sum_d Wo[e][h dh + d] v[h dh + d] + bo[e] / H             (H x E)
 *   c'[h]    = sum_e ln_b[e] a[h][e] + sum_d bq[h dh + d] k[h dh + d] / sqrt(dh)
 * (a block of xs >= 2 H E + H floats), so that with xhat the normalised
 * residual row, score[h][j] = xhat . a'[h][j] + c'[h][j] and
 * ca_out(attention) = sum_{h,j} p[h][j] U'[h][j].  wq: [L][E][E] (row = query
 * channel), woT: [L][E][E] transposed (row = attention channel), bq, bo, ln_g,
 * ln_b: [L][E]; all fp32.  Replaces the ca_in / cross-attention / ca_out
 * GEMMs of nn.TransformerDecoderLayer (Diffusion Policy's TransformerForDiffusion). */
int auras_dpt_xfold(const void *kv, int kv_ld, int rows, int L, int E, int H, const float *wq, const float *bq,
                    const float *woT, const float *bo, const float *ln_g, const float *ln_b, float *out, int xs,
                    void *stream);
void auras_dpt_persist_free(void *plan);

/* Assemble global_cond rows (the ContextStore.publish payload of the DP
 * plugin): for agent a, row = [feat_prev, pos_prev, feat, pos] (n_obs_steps
 * = 2) or [feat, pos] (1); feat_prev/pos_prev are the agent's previous
 * publish (the current one when `first`).  Row a is written at
 * gc_out + a * gc_row_stride (the agent's ring slot). */
int auras_dp_assemble_cond(const float *feat, const float *pos, float *prev_cache, int A,
                           int feat_dim, int pos_dim, int n_obs_steps, int first,
                           float *gc_out, int64_t gc_row_stride, void *stream);

/* Sinusoidal timestep embedding rows for timesteps t[0..n): out[n][dim]. */
int auras_sinusoidal(const int32_t *t, int n, int dim, float *out, void *stream);

/* Initialise request lane state: x_lanes[a][lane] <- x0 (device fp32 rows). */
int auras_dp_copy_rows(float *dst, const float *src, int64_t n_floats, void *stream);

/* GenerationModel.finish for DP: copy the denoised horizon of (agent, lane)
 * into out[agent][...] (fp32). */
int auras_dp_finish(const float *x_lanes, int A, const int *agents, const int *lanes, int n,
                    int lanes_per_agent, int row_floats, float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AURAS_B200_H */
