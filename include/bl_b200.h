/* bl_b200.h — C ABI of the B200-native batched joint CTC/attention decoder.
 *
 * Drop-in boundary for the reference decoding path (beamlattice,
 * /root/reference/proj). Plain pointers and sizes only; every entry point
 * names the reference interface it replaces. The C++ drop-in headers
 * (include/beamlattice/b200.hpp) and the Python mirror
 * (paper_2101_05600_b200/) are thin layers over these calls.
 *
 * Status codes map to the reference's exception types:
 *   BL_INVALID_ARGUMENT -> std::invalid_argument
 *   BL_RUNTIME_ERROR    -> std::runtime_error
 *   BL_LOGIC_ERROR      -> std::logic_error
 *   BL_CUDA_ERROR       -> (new) CUDA failure; no CPU fallback exists.
 * The message of the last failure on the calling thread is bl_last_error().
 */
#ifndef BL_B200_H
#define BL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BL_OK 0
#define BL_INVALID_ARGUMENT 1
#define BL_RUNTIME_ERROR 2
#define BL_LOGIC_ERROR 3
#define BL_CUDA_ERROR 4

/* kNoMargin (ctc_prefix.hpp:12) */
#define BL_NO_MARGIN (1 << 29)

/* EosMode / EosTrigger (beam_search.hpp:14-15) */
#define BL_EOS_BASELINE 0
#define BL_EOS_CTC 1
#define BL_EOS_BOTH 2
#define BL_TRIGGER_BASELINE 0
#define BL_TRIGGER_CTC 1
#define BL_TRIGGER_MAX_LEN 2

/* DecoderConfig (beam_search.hpp:21-33), same fields, same defaults via
 * bl_config_default. */
typedef struct bl_config {
  int beam_width;         /* B, default 3 */
  double ctc_weight;      /* lambda, default 0.3 */
  int eos_m;              /* default 3 */
  double eos_dend;        /* nats, default -10 */
  int eos_c;              /* default 2 */
  int margin_m1;          /* default 5 */
  int margin_m2;          /* default BL_NO_MARGIN */
  int eos_mode;           /* default BL_EOS_BOTH */
  double max_steps_ratio; /* default 1.0 */
} bl_config;

/* Utterance (grid.hpp:50-54) with its PosteriorGrid (grid.hpp:24-43):
 * num_frames x vocab float32 natural-log posteriors, row-major, blank last.
 * `logp` is a host pointer, or a device pointer when the decode call says so
 * (device grids must be 16-byte aligned). */
typedef struct bl_utt {
  const char* id;
  uint32_t num_frames;
  uint32_t vocab;
  uint32_t frame_shift_ms;
  const float* logp;
} bl_utt;

typedef struct bl_scorer bl_scorer;
typedef struct bl_decoder bl_decoder;
typedef struct bl_results bl_results;

/* Message of the last failing call on this thread ("" if none). */
const char* bl_last_error(void);

/* ---- configuration ------------------------------------------------------ */
void bl_config_default(bl_config* cfg);
/* DecoderConfig::validate (beam_search.cpp:36-46), same messages. */
int bl_config_validate(const bl_config* cfg);

/* ---- host-side path pieces (integer-exact, no GPU needed) ---------------- */
/* hard_segments (segmentation.hpp:64-65, segmentation.cpp:121-133):
 * writes up to `cap` half-open [start,end) pairs, *n_out = segment count. */
int bl_hard_segments(int num_frames, int min_len, int max_len, int* starts,
                     int* ends, int cap, int* n_out);
/* VAD segmentation, segmentation.hpp:49-60 composed (frame_llr ->
 * smooth_and_decide -> vad_segments): outputs [T][num_nodes] raw VAD model
 * values; speech/noise node sets; threshold (nats), smoothing window,
 * min_len/max_len in frames. Writes up to cap segments; *n_out = total. */
int bl_vad_segments(const float* outputs, int T, int num_nodes, const int* speech, int n_speech,
                    const int* noise, int n_noise, double threshold, int smooth_window,
                    int min_len, int max_len, int* starts, int* ends, int cap, int* n_out);
/* make_batches (batched.hpp:20-21, batched.cpp:12-30): stable ascending
 * sort by true_frames; order[n] receives the sorted input indices, batches
 * are consecutive chunks of batch_size. */
int bl_make_batches(int n, const uint32_t* true_frames, int batch_size,
                    int* order, int* n_batches);

/* ---- scorers: the "model load" hook (make_scorer, scorer.hpp:84) --------- */
/* spec: "uniform" | "table:PATH" | "loop:TOKEN:P" (scorer.cpp:117-135), and
 * "transformer:PATH[@DEVICE]" (a model file's decoder network, see
 * bl_model_save). */
int bl_scorer_create(const char* spec, int num_tokens, bl_scorer** out);
/* In-memory TableScorer (scorer.hpp:38-55): n_entries contexts of length
 * ctx_len[k] <= order-1 packed in ctx[k*max(order-1,1) ...], each with a
 * normalized (|C|+1)-vector logp[k*(num_tokens+1) ...] (checked like
 * TableScorer::add_entry, scorer.cpp:46-51). Later duplicates replace
 * earlier ones, as std::map assignment does. */
int bl_scorer_create_table(int num_tokens, int order, int n_entries,
                           const int* ctx_len, const int* ctx,
                           const double* logp, bl_scorer** out);
int bl_scorer_create_loop(int num_tokens, int loop_token, double p_loop,
                          bl_scorer** out);
int bl_scorer_num_tokens(const bl_scorer* s);
/* The attention vector the scorer returns for a prefix (Scorer::score,
 * scorer.hpp:20-21), computed host-side; out has num_tokens+1 entries. */
int bl_scorer_score(const bl_scorer* s, const int* prefix, int n, double* out);
void bl_scorer_destroy(bl_scorer* s);

/* ---- decoder: one handle per GPU, one CUDA stream per handle ------------ */
int bl_decoder_create(int device, const bl_config* cfg, const bl_scorer* scorer,
                      bl_decoder** out);
/* nbest: finished hypotheses kept per utterance in the results (>= 1).
 * exact: 1 = every candidate scored by the fp64 reference-order recursion
 *        (fp64-decision mode); 0 = fp32 factorised bulk with certified fp64
 *        refinement of every candidate near the top-B boundary (default).
 * slack: half-width multiplier of the certified interval (default 1.0). */
int bl_decoder_set_options(bl_decoder* d, int nbest, int exact, double slack);
/* Use an external CUDA stream (cudaStream_t as void*); NULL = own stream. */
int bl_decoder_set_stream(bl_decoder* d, void* stream);
/* Step-granular decoding: one kernel launch per decode step with the search
 * state saved in HBM between steps (what a network scorer needs); results are
 * identical to the default single-launch decode. */
int bl_decoder_set_step_mode(bl_decoder* d, int on);
void bl_decoder_destroy(bl_decoder* d);

/* batched_beam_search (batched.hpp:34-38): decodes the utterances of ONE
 * batch (or any number of batches back to back — results are independent
 * of grouping) and returns results in the given order. grids_on_device=1
 * means utts[i].logp are device pointers on the decoder's GPU; 0 means host
 * memory (copied through pinned staging inside the call). Blocks until the
 * results are in host memory. */
int bl_decode(bl_decoder* d, int n, const bl_utt* utts, int grids_on_device,
              bl_results** out);

/* ---- results (DecodeResult, beam_search.hpp:35-42) ---------------------- */
int bl_results_count(const bl_results* r);
int bl_results_get(const bl_results* r, int i, const char** id,
                   const int** tokens, int* n_tokens, double* joint_logp,
                   const int** label_times, int* steps, int* eos_trigger);
/* n-best (new): k-th best finished hypothesis of utterance i, best first;
 * returns BL_INVALID_ARGUMENT past the available count (bl_results_nbest_count). */
int bl_results_nbest_count(const bl_results* r, int i);
int bl_results_nbest(const bl_results* r, int i, int k, const int** tokens,
                     int* n_tokens, double* joint_logp, const int** label_times);
/* DecodeCounters (beam_search.hpp:68-79) summed over the call. */
int bl_results_counters(const bl_results* r, uint64_t* steps,
                        uint64_t* scorer_queries, uint64_t* ctc_frames_evaluated);
/* Instrumentation: device time of the decode kernel(s) on the decoder's
 * stream (CUDA events), algorithmic prefix-score bytes, kernel
 * launches, and the count of utterance-steps that took the exact fallback. */
int bl_results_stats(const bl_results* r, double* kernel_ms, uint64_t* k1_bytes,
                     int* launches, uint64_t* fallback_steps,
                     uint64_t* contenders);
/* Instrumentation: keys the on-chip filter kept during the prefix-score
 * bulk (large vocabularies), summed over utterance-steps. */
int bl_results_filter_keys(const bl_results* r, uint64_t* raw_keys);
/* Instrumentation: wide steps (beams of 13+), i.e. steps whose contender
 * count exceeded the chain slots (3B+16) while the theta0 list stayed
 * complete; they are decided from exact scores of the listed candidates in
 * the candidate order of batched.cpp:181-186, instead of the full fp64
 * fallback over all B x (|C|+1) candidates. */
int bl_results_wide_steps(const bl_results* r, uint64_t* wide_steps);
/* Bulk export (one call for all utterances): row i of tokens/label_times
 * (stride cap >= bl_results_max_tokens) holds n_tokens[i] entries. */
int bl_results_max_tokens(const bl_results* r);
int bl_results_export(const bl_results* r, int cap, int* n_tokens, int* steps,
                      int* trigger, double* joint, int* tokens, int* label_times);
/* Bytes moved host->device (grids) and device->host (result records). */
int bl_results_transfer(const bl_results* r, uint64_t* h2d, uint64_t* d2h);
/* Per-phase device cycle accounting, mean per utterance (16 slots), filled
 * only when the environment variable BL_PROFILE is set. */
int bl_results_profile(const bl_results* r, double* out16);
void bl_results_destroy(bl_results* r);

/* ---- decoder group: several GPUs of one process ---------
 * Replaces the reference's serial loop over batches with an OpenMP fan-out
 * inside each (tools/beamlattice.cpp:128-132, batched.cpp:146): segments are
 * sharded contiguously over the devices, each device decodes its block with
 * no per-step exchange, and the result records (1-best + n-best) are gathered
 * to the first device by one NCCL group (ncclSend/ncclRecv over NVLink),
 * then copied to the host once. One communicator from ncclCommInitAll over
 * the listed devices; NCCL is resolved at run time (libnccl.so.2). Uniform /
 * table / loop scorers (a transformer scorer is bound to one device). */
typedef struct bl_group bl_group;
int bl_group_create(int n_devices, const int* devices, const bl_config* cfg,
                    const bl_scorer* scorer, bl_group** out);
int bl_group_size(const bl_group* g);
/* bl_decoder_set_options on every member. */
int bl_group_set_options(bl_group* g, int nbest, int exact, double slack);
/* Host grids; results in input order, identical to one decoder's. Stats:
 * kernel_ms = the slowest device's decode, counters summed. */
int bl_group_decode(bl_group* g, int n, const bl_utt* utts, bl_results** out);
void bl_group_destroy(bl_group* g);

/* ------------------------------------------------------------------------
 * CTC encoder forward (SURVEY.md §8 a'1, the producer of the PosteriorGrid).
 * The reference takes grids from files (`read_grid`, grid.cpp:108-127); this
 * encoder writes them straight into device memory for bl_decode
 * (grids_on_device = 1). ESPnet-style Transformer encoder, eval mode:
 * Conv2dSubsampling(1->d->d, 3x3 stride 2, ReLU), linear(d*F2 -> d),
 * x*sqrt(d) + sinusoidal PE, `layers` x pre-LN [MHA, FFN(ReLU)] with
 * residuals, final LayerNorm (eps 1e-12), CTC linear(d -> vocab),
 * log_softmax. bf16 tensor-core GEMMs (tcgen05) with fp32 accumulation.
 *
 * Weights: one flat fp32 array in torch layouts, in this order:
 *   conv1.w[d][1][3][3] conv1.b[d] conv2.w[d][d][3][3] conv2.b[d]
 *   out.w[d][d*F2] out.b[d]        (F2 = frames_out(idim), input index c*F2+f)
 *   per layer: ln1.g[d] ln1.b[d] wq[d][d] bq[d] wk[d][d] bk[d] wv[d][d] bv[d]
 *              wo[d][d] bo[d] ln2.g[d] ln2.b[d] w1[dff][d] b1[dff]
 *              w2[d][dff] b2[d]
 *   after_norm.g[d] after_norm.b[d] ctc.w[vocab][d] ctc.b[vocab]
 * ---------------------------------------------------------------------- */
typedef struct bl_encoder_spec {
  int idim;    /* fbank features per frame (80) */
  int d_model; /* multiple of 64, <= 1024 */
  int heads;   /* d_model / 64 */
  int d_ff;
  int layers;
  int vocab;   /* CTC width |C|+1, multiple of 4 */
} bl_encoder_spec;
typedef struct bl_encoder bl_encoder;

/* Encoder frames for `frames_in` fbank frames (1000 -> 249); 0 if < 7. */
int bl_encoder_frames_out(int frames_in);
size_t bl_encoder_num_weights(const bl_encoder_spec* spec);
int bl_encoder_create(int device, const bl_encoder_spec* spec, const float* weights,
                      size_t n_weights, bl_encoder** out);
/* Stream used verbatim (NULL = the legacy default stream); the encoder starts
 * on a private non-blocking stream. */
int bl_encoder_set_stream(bl_encoder* e, void* stream);
/* Segments processed per internal chunk (default 148: 148 x 249 rows is two waves of
 * 128-row GEMM tiles on 148 SMs; workspace ~ chunk x 50 MB at d=512). */
int bl_encoder_set_chunk(bl_encoder* e, int segments);
/* n equal-length segments, fbank [n][frames_in][idim] fp32 (host or device),
 * grid [n][frames_out][vocab] fp32 DEVICE memory. Enqueued on the encoder's
 * stream; returns after enqueue unless `sync` is non-zero. */
int bl_encoder_forward(bl_encoder* e, int n, int frames_in, const float* fbank,
                       int fbank_on_device, float* grid, int sync);
/* Same, also writing the encoder output (final LayerNorm, the decoder's
 * memory) as bf16 DEVICE memory [n][frames_out][d_model] when memory != NULL. */
int bl_encoder_forward_mem(bl_encoder* e, int n, int frames_in, const float* fbank,
                           int fbank_on_device, float* grid, void* memory, int sync);
/* Kernels launched by the last forward. */
int bl_encoder_launches(const bl_encoder* e);
void bl_encoder_destroy(bl_encoder* e);

/* Tensor-core GEMM used by the encoder, exported for tests/benchmarks:
 * C[M,N] = A[M,K] . B[N,K]^T, A/B bf16 device pointers (K-major, strides in
 * elements, multiples of 8); epilogue mode 0 plain, 1 ReLU, 2 residual
 * (out_f32 += ...), 3 scale + positional table (scale, pe[pe_rows][N]).
 * Exactly one of out_f32 / out_bf16 (modes 2 and 3: out_f32); output row
 * stride ldo a multiple of 16 bytes. */
int bl_gemm_bf16(int M, int N, int K, const void* A, int lda, const void* B, int ldb,
                 int mode, const float* bias, float* out_f32, void* out_bf16, int ldo,
                 float scale, const float* pe, int pe_rows, void* stream);

/* ------------------------------------------------------------------------
 * Transformer attention-decoder scorer (SURVEY.md §8 a'2): the paper's
 * network behind the reference's Scorer contract (scorer.hpp:11-22), run on
 * device for every hypothesis of every utterance once per decode step
 * (the decoder switches to step-granular decoding). ESPnet
 * TransformerDecoder, eval mode: Embedding*sqrt(d)+PE, `layers` x pre-LN
 * [causal self-attention (ancestor-indexed KV cache), source attention over
 * the encoder memory, FFN(ReLU)], final LayerNorm, output linear,
 * log_softmax with an fp64 normaliser. sos = eos = vocab-1.
 *
 * Weights: flat fp32, torch layouts, in this order:
 *   embed.w[vocab][d]
 *   per layer: ln1.g ln1.b wq bq wk bk wv bv wo bo        (self-attention)
 *              ln2.g ln2.b wq2 bq2 wk2 bk2 wv2 bv2 wo2 bo2 (source attention)
 *              ln3.g ln3.b w1[dff][d] b1[dff] w2[d][dff] b2[d]
 *   after_norm.g after_norm.b out.w[vocab][d] out.b[vocab]
 * ---------------------------------------------------------------------- */
typedef struct bl_transformer_spec {
  int d_model; /* multiple of 64, <= 1024 */
  int heads;   /* d_model / 64 */
  int d_ff;
  int layers;
  int vocab;   /* |C|+1, eos = sos = vocab-1 */
} bl_transformer_spec;

size_t bl_transformer_num_weights(const bl_transformer_spec* spec);
int bl_scorer_create_transformer(int device, const bl_transformer_spec* spec,
                                 const float* weights, size_t n_weights, bl_scorer** out);
/* bl_decode with a transformer scorer: `memory` is the encoder output, bf16
 * DEVICE memory [n][mem_frames][d_model] (bl_encoder_forward_mem), utterance
 * i's rows at memory + i*mem_frames*d_model. */
int bl_decode_memory(bl_decoder* d, int n, const bl_utt* utts, int grids_on_device,
                     const void* memory, int mem_frames, bl_results** out);
/* Bulk form for large batches: decodes like bl_decode / bl_decode_memory
 * (memory may be NULL) and writes the 1-best results straight into caller
 * arrays — n_tokens/steps/trigger/joint [n], tokens/label_times [n][cap] —
 * without per-utterance result objects. *stats receives a bl_results holding
 * only the counters/stats/transfer figures (count 0); destroy it as usual.
 * When tokens and label_times are page-locked (bl_host_alloc) and cap >= the
 * step cap, those rows are copied device -> caller directly (no host pass). */
int bl_decode_into(bl_decoder* d, int n, const bl_utt* utts, int grids_on_device,
                   const void* memory, int mem_frames, int cap, int* n_tokens, int* steps,
                   int* trigger, double* joint, int* tokens, int* label_times,
                   bl_results** stats);
/* Page-locked host memory for bl_decode_into's outputs (cudaMallocHost). */
int bl_host_alloc(size_t bytes, void** out);
void bl_host_free(void* p);
/* Record mode (parity tests): keep every scorer row the network produced for
 * a live hypothesis, with the utterance index and the token prefix, so a
 * host replay scorer can drive the reference decoder with identical rows. */
int bl_decoder_set_record(bl_decoder* d, int on);
int bl_decoder_record_count(const bl_decoder* d);
int bl_decoder_record_get(const bl_decoder* d, int i, int* utt, int* len, const int** prefix,
                          const double** row);

/* ---- model files and the long-recording chain --------------------------- */
/* Model file (new; the reference's model-load hook is make_scorer,
 * scorer.hpp:84): "BLM1", u32 version 1, u32 sections, each {u32 kind
 * (1 encoder, 2 decoder), u32 spec[6], u64 count, float32[count]} with the
 * flat weight layouts of bl_encoder_create / bl_scorer_create_transformer.
 * Either part may be NULL. bl_scorer_create("transformer:PATH[@DEVICE]", |C|)
 * loads the decoder section (vocabulary checked like table:PATH). */
int bl_model_save(const char* path, const bl_encoder_spec* enc, const float* enc_w,
                  size_t n_enc, const bl_transformer_spec* dec, const float* dec_w,
                  size_t n_dec);
int bl_encoder_create_from_file(int device, const char* path, bl_encoder** out);

/* One long recording end to end (the chain the reference CLI does by hand,
 * tools/beamlattice.cpp:234-273 then :117-146): fbank [T][idim] float32 host
 * -> hard_segments(T, min_len, max_len) -> per segment length one encoder
 * call (grids and, for a transformer scorer, the memory stay in HBM) -> one
 * decode call -> results in segment order, ids "<recording_id>:<start>-<end>"
 * (fbank frames). Encoder and decoder on the same device. */
int bl_recognize(bl_encoder* e, bl_decoder* d, const float* fbank, int T, int idim,
                 const char* recording_id, int min_len, int max_len, bl_results** out);

#ifdef __cplusplus
}
#endif

#endif
