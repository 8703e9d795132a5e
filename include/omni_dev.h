/*
 * omni_dev.h — C ABI of the B200 stage-execution backend (libomni_dev.so).
 *
 * This is the drop-in boundary under the reference's C++ stage engines
 * (/root/reference/proj/include/omniserve). The reference runs every model
 * hook per sequence on the host:
 *   - StageModel::{prefill,on_prompt_consumed,decode,pack_chunk}
 *       registry.hpp:79-89, called from ArEngine::run_batch ar_engine.hpp:308-337
 *       and ArEngine::send_chunk ar_engine.hpp:367-374
 *   - denoise(const DiffusionJob&)  diffusion_engine.hpp:28-43, called per job
 *       from DiffusionEngine::begin_iteration diffusion_engine.hpp:84-112
 *   - Connector::stream_send / stash / materialize  connector.hpp:213-321 with
 *       the payload wire codec payload.hpp:142-166
 * Here each of those becomes ONE batched, asynchronous device call per engine
 * iteration. Plain C: no C++ or torch types cross this line; all host pointers
 * are ordinary memory owned by the caller, device pointers are uint64_t.
 *
 * Threading: a stage handle is used from one host thread at a time (the
 * reference runs all hooks on the orchestrator loop thread,
 * orchestrator.hpp:220,355). Work is enqueued on the stage's own CUDA stream.
 * Errors: every call returns omni_status; omni_last_error() gives the
 * thread-local message. Status codes mirror the reference's error tree
 * (errors.hpp:8-84): E_OOM ~ RegionFull/RejectedTooLarge, E_BADARG ~
 * BadDtype/ConfigInvalid, E_FORWARD ~ ForwardError, E_TRANSPORT ~
 * TransportDown/ProtocolViolation. There is no CPU fallback: without a usable
 * sm_100 device every compute entry point fails with OMNI_E_NOGPU.
 */
#ifndef OMNI_DEV_H
#define OMNI_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum omni_status {
  OMNI_OK = 0,
  OMNI_EAGAIN = 1,       /* asynchronous work not finished yet */
  OMNI_E_OOM = 2,        /* device pool / arena exhausted */
  OMNI_E_BADARG = 3,     /* malformed batch, shape or dtype */
  OMNI_E_FORWARD = 4,    /* model step failed */
  OMNI_E_TRANSPORT = 5,  /* connector ring / peer access failure */
  OMNI_E_CUDA = 6,       /* CUDA runtime error */
  OMNI_E_NOGPU = 7       /* no sm_100 device visible */
} omni_status;

#define OMNI_ABI_VERSION 1

int omni_abi_version(void);
const char* omni_last_error(void);

/* Selects the devices this process drives and enables peer access between
 * every pair (NVLink 5 / NVSwitch). n_dev == 0 means "device 0 only". */
omni_status omni_init(int32_t n_dev, const int32_t* dev_ids);
omni_status omni_device_count(int32_t* n);

/* ------------------------------------------------------------------------ */
/* Models. The reference's mock recurrences (reference_pipeline.hpp:20-45)  */
/* are replaced by random-init bf16 transformers whose weights are a pure   */
/* function of (weight_seed, tensor id, index) — see DESIGN.md §Models.     */
/* ------------------------------------------------------------------------ */
typedef enum omni_model_kind {
  OMNI_MODEL_THINKER = 0, /* text AR LM, emits (token, hidden row)          */
  OMNI_MODEL_TALKER = 1,  /* codec AR LM conditioned on thinker hidden rows */
  OMNI_MODEL_DIT = 2      /* token-local DiT denoiser (Code2Wav / image)    */
} omni_model_kind;

typedef struct omni_model_desc {
  int32_t kind;
  int32_t d_model;
  int32_t n_layers;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t d_ff;
  int32_t vocab;        /* AR: output vocabulary; DiT: conditioning token vocabulary */
  int32_t cond_dim;     /* talker: width of the upstream hidden rows */
  int32_t dit_channels; /* DiT latent channels per sample */
  int32_t dit_samples;  /* DiT samples per token (S) */
  int32_t dit_steps;    /* DiT Euler steps (T) */
} omni_model_desc;

typedef struct omni_stage_limits {
  int32_t max_batch_tokens; /* EngineConfig::max_batch_tokens (registry.hpp:22) */
  int32_t max_resident;     /* EngineConfig::max_resident_requests */
  int32_t max_seq_len;      /* longest context (prompt + emitted) per sequence */
  int32_t kv_pages;         /* paged-KV pool size in 16-token pages (0 = auto) */
  int32_t dit_max_tokens;   /* DiT: max codec tokens per batch */
} omni_stage_limits;

typedef struct omni_stage omni_stage;

omni_status omni_model_default(int32_t kind, omni_model_desc* out);
omni_status omni_stage_create(const omni_model_desc* model, const omni_stage_limits* limits,
                              int32_t dev, uint64_t weight_seed, omni_stage** out);
omni_status omni_stage_destroy(omni_stage* st);
omni_status omni_stage_weight_bytes(const omni_stage* st, uint64_t* bytes);
/* Raw device address of a named weight tensor (tests / oracle checks).
 * Row-major [rows, cols] bf16, except names ending in ".tiled" (the AR
 * stages' gate-up / down weights, "L<l>.wgu.tiled", "L<l>.wd.tiled"): those
 * hold [rows/128][cols/64] blocks of 16 KB, each the SWIZZLE_128B shared-
 * memory image of its 128 x 64 tile (gemm_tc.cu block_weight_kernel). */
omni_status omni_stage_tensor(const omni_stage* st, const char* name, uint64_t* dev_ptr,
                              int64_t* rows, int64_t* cols);

/* ------------------------------------------------------------------------ */
/* AR step: replaces the per-entry loop of ArEngine::run_batch              */
/* (ar_engine.hpp:308-337) with one batched forward over every entry of     */
/* the IterationBatch, in entry order (decoders by request id, then         */
/* prefills — ar_engine.hpp:149-192).                                       */
/* ------------------------------------------------------------------------ */
enum { OMNI_PHASE_PREFILL = 0, OMNI_PHASE_DECODE = 1 };

typedef struct omni_ar_batch {
  int32_t n_entries;
  const uint64_t* seq_id;    /* [n_entries] request id = KV sequence handle */
  const int32_t* phase;      /* [n_entries] OMNI_PHASE_* */
  const int32_t* span;       /* [n_entries] tokens fed (decode: 1) */
  const int32_t* pos0;       /* [n_entries] first KV position written */
  const int32_t* out_index;  /* [n_entries] decode: emitted index k (hidden-ring row); else -1 */
  const int32_t* tokens;     /* [sum span] input ids (prefill: prompt span; decode k: emitted[k-1], k=0 -> start id) */
  const uint64_t* cond_src;  /* talker: [sum span] device address of the bf16 hidden row feeding
                                each prefill token (0 for decode tokens); NULL otherwise */
  const int32_t* cond_row;   /* talker: [sum span] conditioning row j (prefill: prompt index,
                                decode step m: m/4); NULL otherwise */
} omni_ar_batch;

/* Enqueues the step on the stage stream and returns immediately. Results for
 * DECODE entries (greedy token id, top-2 logit margin) are copied to
 * token_out/margin_out (host, [n_entries]) by omni_stage_wait / a successful
 * omni_stage_query. PREFILL entries emit nothing (ar_engine.hpp:313-324). */
omni_status omni_ar_step(omni_stage* st, const omni_ar_batch* batch, int32_t* token_out,
                         float* margin_out);
/* Sampling of DECODE rows: top_k <= 1 = greedy argmax (default; the
 * reference's token_of is greedy, reference_pipeline.hpp:34), 2..32 = top-k
 * sampling at temperature 1 with a draw keyed by (seed, request id, emitted
 * index) -- deterministic and batch-invariant, so recompute preemption
 * (ar_engine.hpp:229-257) replays the same tokens. The margin output stays
 * the top-2 logit margin. */
omni_status omni_stage_set_sampling(omni_stage* st, int32_t top_k, uint64_t seed);

/* Prefix cache of a Thinker stage (on by default): full
 * 16-token prompt pages are keyed by a chained hash of their token prefix and
 * shared read-only between sequences; a prefill span whose pages are cached
 * runs only its uncached suffix on the device (prefill emits nothing, so the
 * caller sees no difference: outputs are bit-identical). Toggle only with no
 * resident sequence. Stats: prompt tokens served from the cache, pages held,
 * pages evicted (when the KV pool runs out). */
omni_status omni_stage_set_prefix_cache(omni_stage* st, int32_t enable);
omni_status omni_stage_prefix_stats(const omni_stage* st, uint64_t* hit_tokens, uint64_t* cached_pages,
                                    uint64_t* evicted_pages);
/* SM share of a DiT stage: its denoise iteration is one persistent kernel that
 * holds whole SMs (192 KB shared memory, all of TMEM) for the iteration, so
 * beside AR stages on the same GPU it must leave them SMs. sms <= 0 = all SMs
 * of the device (the DiT has its GPU to itself). No effect on results. */
omni_status omni_stage_set_sm_share(omni_stage* st, int32_t sms);

/* Admits a sequence's KV pages for positions [0, upto_tokens) ahead of a
 * step, so a sequence that does not fit fails alone (OMNI_E_OOM) instead of
 * failing the whole batched step (the reference fails per entry,
 * ar_engine.hpp:332-334). omni_ar_step reserves implicitly. */
omni_status omni_seq_reserve(omni_stage* st, uint64_t seq_id, int32_t upto_tokens);
/* The same for a PREFILL span [pos0, pos0 + span) with its prompt token ids:
 * a Thinker stage first maps the span's cached prompt pages (prefix cache),
 * so reserving ahead of the step does not pre-empt the cache. */
omni_status omni_seq_reserve_prompt(omni_stage* st, uint64_t seq_id, int32_t pos0, int32_t span,
                                    const int32_t* tokens);

/* Frees the KV pages / hidden ring / conditioning rows of a sequence
 * (finish, recompute-preemption ar_engine.hpp:233-257, or failure). */
omni_status omni_seq_release(omni_stage* st, uint64_t seq_id);

/* Device address of hidden-ring row `index` of a thinker sequence (bf16[d]). */
omni_status omni_seq_hidden_row(omni_stage* st, uint64_t seq_id, int32_t index,
                                uint64_t* dev_ptr);

/* ------------------------------------------------------------------------ */
/* DiT step: replaces per-job denoise() (diffusion_engine.hpp:28-43, 98)    */
/* with one batched T-step Euler denoise over every codec token of every    */
/* job. Noise is keyed by (request id, global token position, sample), so   */
/* output is independent of chunking and batching (diffusion_engine.hpp:25- */
/* 27, test_diffusion.cpp:50-65).                                           */
/* ------------------------------------------------------------------------ */
typedef struct omni_dit_batch {
  int32_t n_jobs;
  const uint64_t* request_id;  /* [n_jobs] */
  const int32_t* token_offset; /* [n_jobs] global codec position of the job's first token */
  const int32_t* n_tokens;     /* [n_jobs] */
  const int32_t* tokens;       /* [sum n_tokens] conditioning ids */
} omni_dit_batch;

/* samples_out: host [sum n_tokens * dit_samples] int32, filled at completion. */
omni_status omni_dit_step(omni_stage* st, const omni_dit_batch* batch, int32_t* samples_out);

/* Completion of the last enqueued step (and pack) of a stage. */
omni_status omni_stage_query(omni_stage* st); /* OMNI_OK | OMNI_EAGAIN */
omni_status omni_stage_wait(omni_stage* st);
/* Device time of the last completed step in microseconds (CUDA events). */
omni_status omni_stage_last_step_us(omni_stage* st, float* us);

/* ------------------------------------------------------------------------ */
/* Connector data plane: replaces pack_chunk (reference_pipeline.hpp:113-   */
/* 123) + encode_payload (payload.hpp:142-151) + stash (connector.hpp:214-  */
/* 236) for the hidden-state edge. Each chunk is written in the reference   */
/* wire layout  [dtype u8=FIX16(2)][rank u8=2][n u32 LE][1+d u32 LE]        */
/* [n x (1+d) little-endian u16: col 0 = token id, cols 1..d = bf16 bits]   */
/* into a device arena (local or peer GPU).                                  */
/* ------------------------------------------------------------------------ */
typedef struct omni_arena omni_arena;
omni_status omni_arena_create(int32_t dev, uint64_t bytes, omni_arena** out);
omni_status omni_arena_destroy(omni_arena* a);
omni_status omni_arena_base(const omni_arena* a, uint64_t* dev_ptr, uint64_t* bytes);

/* Blob size of one packed chunk of `rows` hidden rows of width d. */
uint64_t omni_pack_bytes(int32_t rows, int32_t d);

/* Packs rows [begin[c], end[c]) of seq_id[c]'s hidden ring, with token ids
 * tokens[sum of previous row counts ...], into dst_base + dst_offset[c] for
 * every chunk c, in one launch on the source stage's stream. Destinations may
 * lie on a peer GPU (remote stores over NVLink; omni_init enables peer
 * access) and may differ per chunk (dst_base = 0, absolute dst_offset). */
omni_status omni_pack_hidden(omni_stage* src, int32_t n_chunks, const uint64_t* seq_id,
                             const int32_t* begin, const int32_t* end, const int32_t* tokens,
                             uint64_t dst_base, const uint64_t* dst_offset);
/* Make `dst`'s next step wait (on-device) for everything `src` enqueued so far. */
omni_status omni_stage_after(omni_stage* dst, omni_stage* src);
/* Make `dst`'s next step wait (on-device, across GPUs) for `src`'s most recent
 * omni_pack_hidden only -- not for steps `src` enqueued after the pack. This
 * is the connector's consumer-side ordering: the Talker reads rows the
 * Thinker packed into its arena without serialising behind the Thinker's next
 * step. No-op before the first pack. */
omni_status omni_stage_after_pack(omni_stage* dst, omni_stage* src);

/* ------------------------------------------------------------------------ */
/* Multi-process placement (the reference's SHM / TCP        */
/* transports, connector.hpp:23-30, 77-90, shm_region.hpp). A consumer      */
/* process exports its connector arena; the producer process imports it     */
/* and packs straight into it (omni_pack_hidden with absolute destinations  */
/* inside the imported arena), then records an interprocess event that the  */
/* consumer's stage waits on. The control frames (DEVICE locators, arena-   */
/* relative offsets) travel over the serve library's IPC channel.           */
/* ------------------------------------------------------------------------ */
typedef struct omni_ipc_handle {
  uint8_t handle[64]; /* cudaIpcMemHandle_t */
  uint64_t bytes;
  int32_t dev;
  int32_t reserved;
} omni_ipc_handle;
typedef struct omni_ipc_event_handle {
  uint8_t handle[64]; /* cudaIpcEventHandle_t */
} omni_ipc_event_handle;
typedef struct omni_ipc_event omni_ipc_event;
omni_status omni_arena_export(const omni_arena* a, omni_ipc_handle* out);
/* Maps another process's exported arena; omni_arena_destroy unmaps it. */
omni_status omni_arena_import(const omni_ipc_handle* h, omni_arena** out);
omni_status omni_ipc_event_create(int32_t dev, omni_ipc_event** out, omni_ipc_event_handle* handle);
omni_status omni_ipc_event_open(int32_t dev, const omni_ipc_event_handle* handle, omni_ipc_event** out);
omni_status omni_ipc_event_destroy(omni_ipc_event* e);
/* Records `e` on src's stream (call right after omni_pack_hidden). */
omni_status omni_stage_record_pack(omni_stage* src, omni_ipc_event* e);
/* dst's next step waits (on-device) for the last record of `e`, which may
 * have been made by another process. */
omni_status omni_stage_wait_event(omni_stage* dst, omni_ipc_event* e);
omni_status omni_ipc_event_sync(omni_ipc_event* e);
/* Plumbing for tests / bench (no compute): device memory and copies. */
omni_status omni_mem_alloc(int32_t dev, uint64_t bytes, uint64_t* dev_ptr);
omni_status omni_mem_free(uint64_t dev_ptr);
omni_status omni_mem_h2d(uint64_t dst_dev, const void* src, uint64_t bytes);
omni_status omni_mem_d2h(void* dst, uint64_t src_dev, uint64_t bytes);
omni_status omni_mem_set(uint64_t dst_dev, int32_t byte, uint64_t bytes);
omni_status omni_device_sync(void);
/* Process-wide counters: kernels launched by libomni_dev, bytes copied
 * host->device / device->host by the step / pack entry points. */
omni_status omni_dev_counters(uint64_t* launches, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* Step-graph cache: graphs captured (first use of a launch geometry) and replayed. */
omni_status omni_dev_graph_counters(uint64_t* captures, uint64_t* replays);

/* ------------------------------------------------------------------------ */
/* Kernel-level entry points (parity tests / microbenchmarks). All pointers */
/* are device addresses; run on the current device's default stream.        */
/* ------------------------------------------------------------------------ */
/* Y[M,N] = X[M,K] * W[N,K]^T with epilogue `epi` (0 bf16, 1 f32, 2 f32 +=,
 * 3 gated f32 +=, 4 swiglu bf16, 5 gelu bf16). Returns the split-K factor
 * used via *splits (may be NULL). */
omni_status omni_k_gemm(uint64_t W, int32_t N, int32_t K, uint64_t X, int32_t M, int32_t epi,
                        uint64_t out, int32_t ldo, uint64_t gate, int32_t ldg, int32_t gate_off,
                        int32_t rows_per_group, int32_t max_splits, int32_t* splits);
/* Fills dst[n] (bf16) with the counter-based weight stream of (seed, tensor_id). */
omni_status omni_k_fill_weights(uint64_t dst, int64_t n, uint64_t seed, uint32_t tensor_id,
                                float scale);
/* Times `iters` back-to-back launches of omni_k_gemm (device ms per launch). */
omni_status omni_k_gemm_time(uint64_t W, int32_t N, int32_t K, uint64_t X, int32_t M,
                             int32_t epi, uint64_t out, int32_t ldo, int32_t max_splits,
                             int32_t iters, float* ms);

/* CUDA-event time per launch of a graph of `iters` GEMMs cycling over n_w
 * distinct weight copies (footprint > L2 => every launch streams HBM). */
omni_status omni_k_gemm_time_multi(const uint64_t* Ws, int32_t n_w, int32_t N, int32_t K, uint64_t X,
                                   int32_t M, int32_t epi, uint64_t out, int32_t ldo, int32_t max_splits,
                                   int32_t iters, float* ms);

/* Phase trace of the last of n_w chained launches (tools/gemm_trace.py):
 * trace_dev holds 8 u64 per CTA (globaltimer entry/exit + clock64 phase
 * offsets); *grid_ctas = CTAs of the launch. */
omni_status omni_k_gemm_trace(const uint64_t* Ws, int32_t n_w, int32_t N, int32_t K, uint64_t X, int32_t M,
                              int32_t epi, uint64_t out, int32_t ldo, int32_t max_splits, uint64_t trace_dev,
                              int32_t* grid_ctas);

/* Debug phase traces (tools/attn_trace.py); 0 disables. attn_trace: 8 u64
 * globaltimer stamps per attention CTA, indexed (layer, kv_head, block);
 * gemm_marks: 3 u64 atomic-max marks (last QKV CTA exit, last O-projection
 * producer past its PDL wait, last O-projection CTA exit). */
omni_status omni_k_debug_traces(uint64_t attn_trace, uint64_t gemm_marks);

#ifdef __cplusplus
}
#endif
#endif /* OMNI_DEV_H */
