/*
 * seqpipe_b200.h — the C-ABI drop-in boundary of the B200-native Seq1F1B engine.
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, never
 * throws, and returns an int status (SP_OK == 0). On failure the message is
 * available from sp_last_error() (thread-local). The C++ wrapper in
 * include/seqpipe/ (C++ headers) re-throws the reference's exception types from these
 * codes, so code written against the reference `seqpipe::` API keeps working.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   sp_scenario / sp_scenario_validate      core/include/seqpipe/scenario.hpp:25-50, core/src/scenario.cpp:22-41
 *   sp_preset_scenario                      core/include/seqpipe/scenario.hpp:83, core/src/scenario.cpp:172-189
 *   sp_apply_override / sp_parse_scenario   core/include/seqpipe/scenario.hpp:76-80, core/src/scenario.cpp:76-139
 *   sp_segment_flops                        core/include/seqpipe/cost.hpp:22-23, core/src/cost.cpp:20-26
 *   sp_forward_cost / sp_task_cost          core/include/seqpipe/cost.hpp:29-33, core/src/cost.cpp:28-55
 *   sp_partition / sp_make_partition        core/include/seqpipe/partition.hpp:31-52, core/src/partition.cpp:60-281
 *   sp_balance_report                       core/include/seqpipe/partition.hpp:59, core/src/partition.cpp:283-303
 *   sp_warmup                               core/include/seqpipe/schedule.hpp:57-63, core/src/schedule.cpp:38-58
 *   sp_schedule_ops                         core/include/seqpipe/schedule.hpp:80, core/src/schedule.cpp:313-349
 *   sp_dependencies                         core/include/seqpipe/sim.hpp:27, core/src/sim.cpp:14-44
 *   sp_simulate                             core/include/seqpipe/sim.hpp:80, core/src/sim.cpp:121-317
 *   sp_check_schedule / sp_check_warmup     core/include/seqpipe/validate.hpp:34,42, core/src/validate.cpp:85-325
 *   sp_schedule_to_json / _from_json        core/include/seqpipe/json_io.hpp:19-20, core/src/json_io.cpp:59-97
 *   sp_report_to_json                       core/include/seqpipe/json_io.hpp:25-26, core/src/json_io.cpp:99-159
 *   sp_render_gantt / sp_engine_render_gantt  core/include/seqpipe/render.hpp:15-21, core/src/render.cpp:46-124
 *   sp_compare_csv                          core/include/seqpipe/sim.hpp:82-99, core/src/sim.cpp:319-367
 *   sp_device_partition / sp_device_schedule_ops   GPU-resident launcher core (no reference counterpart;
 *                                           bit-exact with cwp_partition/generate)
 *   sp_engine_*                             replaces the modeled execution of simulate() (sim.cpp:121-317)
 *                                           with real sm_100a execution of the same op tables
 */
#ifndef SEQPIPE_B200_H_
#define SEQPIPE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped 1:1 onto the reference's exception types) ---- */
enum {
  SP_OK = 0,
  SP_ERR_INVALID_ARGUMENT = 1,   /* std::invalid_argument                 */
  SP_ERR_UNSUPPORTED = 2,        /* seqpipe::UnsupportedScheduleError      */
  SP_ERR_OUT_OF_RANGE = 3,       /* std::out_of_range                      */
  SP_ERR_DOMAIN = 4,             /* std::domain_error                      */
  SP_ERR_OVERFLOW = 5,           /* std::overflow_error                    */
  SP_ERR_DEADLOCK = 6,           /* seqpipe::DeadlockError                 */
  SP_ERR_MISSING_DEPENDENCY = 7, /* seqpipe::MissingDependencyError        */
  SP_ERR_LOGIC = 8,              /* std::logic_error                       */
  SP_ERR_RUNTIME = 9,            /* std::runtime_error (other)             */
  SP_ERR_CUDA = 10,              /* CUDA runtime / driver failure          */
  SP_ERR_NCCL = 11,              /* NCCL failure                           */
  SP_ERR_BUFFER_TOO_SMALL = 12   /* caller buffer too small; size reported */
};

const char* sp_last_error(void);
const char* sp_version(void);

/* ---- exact rationals (int64 num/den, reduced, den > 0) ---- */
typedef struct sp_rational {
  int64_t num;
  int64_t den;
} sp_rational;

/* ---- enums (same order as the reference enums) ---- */
enum { SP_COST_FLOPS = 0, SP_COST_UNIFORM = 1 };                       /* CostModel     */
enum { SP_PART_EVEN = 0, SP_PART_CWP = 1, SP_PART_ORACLE = 2 };       /* PartitionMode */
enum { SP_TASK_F = 0, SP_TASK_B = 1, SP_TASK_I = 2, SP_TASK_W = 3 };  /* TaskKind      */
enum {                                                                 /* ScheduleKind  */
  SP_SCHED_GPIPE = 0,
  SP_SCHED_1F1B = 1,
  SP_SCHED_1F1B_I = 2,
  SP_SCHED_SEQ1F1B = 3,
  SP_SCHED_SEQ1F1B_I = 4,
  SP_SCHED_ZB1P = 5,
  SP_SCHED_SEQZB1P = 6
};

/* ScenarioConfig (scenario.hpp:25-50), field for field. */
typedef struct sp_scenario {
  int32_t pipeline_size;
  int32_t stages_per_device;
  int32_t micro_batches;
  int32_t segments;
  int64_t seq_len;
  int32_t layers;
  int32_t cost_model;
  int64_t hidden_dim;
  int64_t param_count;
  sp_rational backward_ratio;
  sp_rational bw_input_ratio;
  sp_rational bw_weight_ratio;
  sp_rational comm_latency;
  sp_rational activation_cost_per_token;
  sp_rational time_per_flop;
  sp_rational uniform_forward;
} sp_scenario;

/* Task (task.hpp:35-43): all indices 1-based. */
typedef struct sp_task {
  int32_t kind;
  int32_t micro_batch;
  int32_t segment;
  int32_t stage;
  int32_t device;
} sp_task;

typedef struct sp_task_timing {
  sp_task task;
  sp_rational start;
  sp_rational end;
} sp_task_timing;

/* DeviceReport (sim.hpp:35-48) without the memory series (queried separately). */
typedef struct sp_device_report {
  int32_t device;
  int32_t warmup_forward_tasks;
  int64_t peak_allocations;
  sp_rational first_start;
  sp_rational last_end;
  sp_rational busy;
  sp_rational idle;
  sp_rational bubble_ratio;
  sp_rational idle_in_makespan;
  sp_rational bubble_ratio_in_makespan;
  sp_rational peak_memory;
  int64_t memory_series_len;
} sp_device_report;

typedef struct sp_sim_summary {
  sp_rational makespan;
  sp_rational aggregate_bubble_ratio;
  sp_rational aggregate_bubble_ratio_in_makespan;
  sp_rational max_peak_memory;
  sp_rational modeled_throughput;
} sp_sim_summary;

/* ---- scenario ---- */
void sp_scenario_default(sp_scenario* out);
int sp_scenario_validate(const sp_scenario* cfg);
int sp_preset_scenario(const char* name, sp_scenario* out);
int sp_apply_override(sp_scenario* cfg, const char* key, const char* value);
int sp_parse_scenario_text(const char* text, sp_scenario* out);
/* Writes the flat key = value text (scenario_to_text); *len in/out. */
int sp_scenario_to_text(const sp_scenario* cfg, char* buf, size_t* len);

/* ---- cost model (Eq. 8) ---- */
/* 128-bit exact result split into hi (signed) / lo (unsigned) words. */
int sp_segment_flops(const sp_scenario* cfg, int64_t prefix_before, int64_t length, int64_t* hi,
                     uint64_t* lo);
int sp_forward_cost(const sp_scenario* cfg, const int64_t* lengths, int32_t k, int32_t segment,
                    sp_rational* out);
int sp_task_cost(const sp_scenario* cfg, const int64_t* lengths, int32_t k, const sp_task* task,
                 sp_rational* out);

/* ---- partition ---- */
/* lengths_out must hold cfg->segments entries. */
int sp_partition(const sp_scenario* cfg, int32_t mode, int64_t* lengths_out, sp_rational* imbalance_out);
int sp_even_partition(int64_t n, int32_t k, const sp_scenario* cfg, int64_t* lengths_out,
                      sp_rational* imbalance_out);
int sp_make_partition(const sp_scenario* cfg, const int64_t* lengths, int32_t k, sp_rational* imbalance_out);
/* segment_costs must hold k entries. */
int sp_balance_report(const sp_scenario* cfg, const int64_t* lengths, int32_t k,
                      sp_rational* segment_costs, sp_rational* imbalance_out);

/* ---- schedule ---- */
/* kind: 0 = 1f1b, 1 = seq1f1b, 2 = 1f1b-i, 3 = seq1f1b-i; a = micro_batches (kinds 0,1) or
 * stages_per_device (kinds 2,3). */
int sp_warmup(int32_t formula, int32_t pipeline_size, int32_t a, int32_t segments, int32_t device,
              int32_t* out);
/* Size query: ops == NULL fills counts[P] and returns SP_OK. Fill: ops holds sum(counts)
 * entries laid out device after device. */
int sp_schedule_ops(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, sp_task* ops,
                    int64_t* counts);
int sp_dependencies(const sp_task* task, const sp_scenario* cfg, sp_task* out, int32_t* n_out);

/* ---- simulate ---- */
/* timings (optional) aligned with ops; devices (optional) holds P entries. */
int sp_simulate(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                const int64_t* counts, sp_task_timing* timings, sp_device_report* devices,
                sp_sim_summary* summary);
/* Memory series of one device (1-based): pairs (time, level); *len in/out. */
int sp_simulate_memory_series(const sp_scenario* cfg, int32_t kind, const int64_t* lengths,
                              const sp_task* ops, const int64_t* counts, int32_t device,
                              sp_rational* series, int64_t* len);

/* ---- JSON wire formats (core/include/seqpipe/json_io.hpp:19-26, core/src/json_io.cpp:59-159) ----
 * seqpipe.schedule.v1 of an op table / seqpipe.simreport.v1 of its simulation, canonical bytes
 * (sorted keys, exact rationals, `indent` spaces per level, trailing newline). Text out via
 * (buf, len): buf == NULL returns the needed size (incl. NUL) in *len. sp_schedule_from_json:
 * ops == NULL fills cfg_out / kind_out / counts[P] only (P <= max_devices). */
int sp_schedule_to_json(const sp_scenario* cfg, int32_t kind, const sp_task* ops, const int64_t* counts,
                        int32_t indent, char* buf, size_t* len);
int sp_schedule_from_json(const char* text, sp_scenario* cfg_out, int32_t* kind_out, sp_task* ops,
                          int64_t* counts, int32_t max_devices);
int sp_report_to_json(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                      const int64_t* counts, int32_t indent, int64_t memory_downsample, char* buf,
                      size_t* len);

/* ---- Timeline rendering and comparison (core/include/seqpipe/render.hpp:15-21, core/src/render.cpp:46-124;
 * core/include/seqpipe/sim.hpp:82-99, core/src/sim.cpp:319-367) ----
 * sp_render_gantt: simulate(schedule, partition) drawn as text (SP_RENDER_ASCII, `width` cells per row)
 * or SVG (SP_RENDER_SVG); sp_engine_render_gantt draws the engine's last MEASURED step (ns times,
 * needs SP_FLAG_TIMELINE). sp_compare_csv: compare() of the simulations of n >= 2 op tables, as CSV
 * (ComparisonTable::to_csv); reports must share seq_len / micro_batches unless allow_mixed.
 * Text out via (buf, len) as above. */
enum { SP_RENDER_ASCII = 0, SP_RENDER_SVG = 1 };
int sp_render_gantt(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                    const int64_t* counts, int32_t format, int32_t width, char* buf, size_t* len);
int sp_compare_csv(int32_t n, const sp_scenario* cfgs, const int32_t* kinds, const int64_t* const* lengths,
                   const sp_task* const* ops, const int64_t* const* counts, int32_t allow_mixed, char* buf,
                   size_t* len);

/* ---- validate ---- */
/* Violations as lines "code\tdevice\tdetail\n"; *n_violations set; *len in/out. */
int sp_check_schedule(const sp_scenario* cfg, int32_t kind, const sp_task* ops, const int64_t* counts,
                      char* buf, size_t* len, int32_t* n_violations);
int sp_check_warmup_formulas(const sp_scenario* cfg, int32_t kind, const sp_task* ops,
                             const int64_t* counts, char* buf, size_t* len, int32_t* n_violations);

/* ---- GPU-resident launcher core (sm_100a) ---- */
/* cwp / even partition computed by a device kernel (IEEE double, no contraction). */
int sp_device_partition(const sp_scenario* cfg, int32_t mode, int32_t cuda_device, int64_t* lengths_out);
/* Op tables of the non-interleaved kinds (gpipe, 1f1b, seq1f1b) generated on the device in
 * closed form, copied back into ops/counts (same layout as sp_schedule_ops). */
int sp_device_schedule_ops(const sp_scenario* cfg, int32_t kind, int32_t cuda_device, sp_task* ops,
                           int64_t* counts);

/* ---- pipeline P2P plan (what the multi-process engine sends / receives) ---- */
enum { SP_COMM_SEND = 0, SP_COMM_RECV = 1 };
typedef struct sp_comm_op {
  int32_t op_index;   /* position in the device order                               */
  int32_t when;       /* 0: before the op (receive), 1: after the op (send)           */
  int32_t dir;        /* SP_COMM_SEND / SP_COMM_RECV                                  */
  int32_t peer;       /* peer rank (device - 1)                                       */
  int32_t channel;    /* pipeline edge (v, v+1): 2(v-1) activations, 2(v-1)+1 gradients */
  int32_t kind;       /* task kind of the op                                          */
  int32_t micro_batch, segment, stage;
  int32_t reserved;
  int64_t elems;      /* segment_tokens * hidden                                      */
} sp_comm_op;
/* Size query with out == NULL. device is 1-based. */
int sp_comm_plan(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths, int32_t device,
                 int64_t hidden, sp_comm_op* out, int64_t* n);

/* ---- execution engine ---- */
enum { SP_MODEL_GPT = 0, SP_MODEL_LLAMA = 1 };
enum { SP_DTYPE_F32 = 0, SP_DTYPE_BF16 = 1 };

/* Transformer shape + numerics. Engine-only keys live here, separate from sp_scenario so the
 * scenario file stays byte-compatible with the reference parser. */
typedef struct sp_model {
  int32_t family;     /* SP_MODEL_GPT: LayerNorm, GeLU(tanh), learned positions; SP_MODEL_LLAMA:
                         RMSNorm, SwiGLU, RoPE */
  int32_t dtype;      /* SP_DTYPE_F32 validation mode, SP_DTYPE_BF16 production mode */
  int32_t vocab;
  int32_t hidden;
  int32_t layers;     /* total layers, split evenly over the pipeline stages */
  int32_t heads;
  int32_t head_dim;
  int32_t ffn;
  int64_t max_seq;    /* learned position table size (GPT) */
  uint64_t seed;      /* weight init seed */
  float init_std;     /* N(0, init_std); out/down projections scaled by 1/sqrt(2L) */
  float norm_eps;
  float rope_theta;
  float lr;           /* AdamW step applied at the end of every step (0 disables) */
  float beta1, beta2, adam_eps, weight_decay;
  int32_t flags;      /* SP_FLAG_* */
  int32_t reserved;
} sp_model;

enum {
  SP_FLAG_NO_TCGEN05 = 1,   /* bf16 mode: force the SIMT GEMM (debug / A-B testing)   */
  SP_FLAG_NO_TC_ATTN = 2,   /* bf16 mode: force the SIMT attention                    */
  SP_FLAG_TIMELINE = 4,     /* record per-op CUDA events for the measured report      */
  SP_FLAG_KPROBE = 8,       /* CUDA events around every GEMM / attention launch        */
  SP_FLAG_RECOMPUTE_MLP = 16 /* do not keep the MLP up-projection output u in the (m,s) record;
                                recompute it in B (one extra [n,h]x[h,Fup] GEMM per layer).
                                Fixed at engine creation (it sizes the activation records). */
};

typedef struct sp_engine sp_engine;

/* Measured counterpart of SimReport for one executed step on one stage (device). */
typedef struct sp_step_report {
  double step_ms;             /* CUDA-event time of the whole step on this device           */
  double busy_ms;             /* sum of op durations                                        */
  double first_start_ms;      /* relative to the step start event                           */
  double last_end_ms;
  double bubble_ratio;        /* idle / (last_end - first_start), as sim.cpp:252-254        */
  double loss;                /* mean token loss (last stage; 0 elsewhere)                  */
  double peak_activation_bytes;  /* activation arena high-water mark (KV prefix included)   */
  double arena_bytes;         /* bytes reserved for the activation arena                    */
  double weight_bytes;        /* params + grads + optimizer state                           */
  int64_t ops_executed;
  int64_t kernel_launches;
  double dominant_kernel_ms;  /* summed duration of the dominant kernel class (KPROBE)      */
  int64_t dominant_kernel_launches;
  double dominant_kernel_flops;  /* algorithmic FLOPs of those launches (all issued FLOPs when
                                    KPROBE is off)                                          */
  int32_t dominant_kernel_class; /* 0 tcgen05/SIMT GEMM, 1 attention fwd, 2 attention bwd   */
  int32_t reserved0;
  double class_ms[3];         /* per class: GEMM, attention fwd, attention bwd (KPROBE)      */
  double class_flops[3];
  int64_t class_launches[3];
} sp_step_report;

/* One engine = one device (all stages this device owns). world_size == pipeline_size for the
 * multi-process NCCL path; world_size == 1 runs every stage in this process on one GPU, with
 * stage hand-offs as device copies (the single-GPU validation configuration). */
int sp_engine_create(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths,
                     const sp_model* model, int32_t rank, int32_t world_size, int32_t cuda_device,
                     sp_engine** out);
int sp_engine_destroy(sp_engine* eng);
/* Analytical activation footprint of one stage under a schedule (host-only replay of the
 * engine's arena plan; no device memory): live high-water mark, arena size, and the fp32
 * dK/dV accumulator. Used to report configurations that would not fit (e.g. 1F1B at 128K). */
int sp_plan_memory(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths, const sp_model* model,
                   int32_t stage, double* live_peak_bytes, double* arena_bytes, double* dkv_bytes);
/* Multi-rank data plane (world_size == pipeline_size). One channel per pipeline edge and direction
 * (sp_comm_op.channel); sp_engine_comm_channels gives their number.
 * NCCL (one process per GPU): rank 0 calls sp_nccl_unique_id once per channel, the id bytes travel by
 * any side channel, every rank calls sp_engine_comm_init with all of them (one communicator each).
 * In-process (several engines in one process, one host thread each, e.g. P ranks on one GPU):
 * sp_local_hub_create once, sp_engine_attach_local on every engine; a receive that does not pair up
 * within watchdog_seconds fails with SP_ERR_DEADLOCK instead of hanging. */
typedef struct sp_local_hub sp_local_hub;
int sp_engine_comm_channels(sp_engine* eng, int32_t* n);
int sp_nccl_unique_id(uint8_t* out, size_t len);
int sp_engine_comm_init(sp_engine* eng, const uint8_t* const* ids, int32_t n_ids);
/* Peer-memory data plane instead of NCCL (one process per GPU, CUDA IPC): every rank calls
 * sp_engine_ipc_export (size query with out == NULL, then the copy; it allocates the rank's
 * receive rings and flag words once), the blobs travel over any side channel, then every rank
 * calls sp_engine_ipc_connect with all of them in rank order. A message is one device-to-device
 * copy into the receiver's ring plus two flag words, written and awaited by the streams
 * themselves (cuStreamWriteValue64 / cuStreamWaitValue64: no SM spins). A transfer that never
 * pairs up: sp_engine_step returns SP_ERR_DEADLOCK after the watchdog time (SP_P2P_WATCHDOG_S);
 * the engine is then unusable (later steps fail the same way) and sp_engine_destroy releases it
 * without waiting on the parked streams, so the process can exit. */
int sp_engine_ipc_export(sp_engine* eng, uint8_t* out, size_t* len);
int sp_engine_ipc_connect(sp_engine* eng, const uint8_t* const* blobs, const size_t* lens, int32_t n);
int sp_local_hub_create(int32_t world_size, double watchdog_seconds, sp_local_hub** out);
int sp_local_hub_destroy(sp_local_hub* hub);
int sp_engine_attach_local(sp_engine* eng, sp_local_hub* hub);
/* Single-rank engines: capture the step body (every op of the op table + the optimizer) into a
 * CUDA graph on the next step and replay it from then on (on != 0); 0 returns to eager launches.
 * Steps with SP_FLAG_KPROBE run eagerly. */
int sp_engine_enable_graph(sp_engine* eng, int32_t on);
/* Replace the engine's SP_FLAG_* set (e.g. turn kernel probes on for a timed region). */
int sp_engine_set_flags(sp_engine* eng, int32_t flags);
/* tokens: micro_batches x (seq_len + 1) int32 (inputs are [:, :T], labels [:, 1:]).
 * tokens_on_device != 0 means `tokens` is a device pointer. */
int sp_engine_step(sp_engine* eng, const int32_t* tokens, int32_t tokens_on_device,
                   sp_step_report* report);
/* Executed op log of the last step for this engine (same layout as sp_schedule_ops). */
int sp_engine_op_log(sp_engine* eng, sp_task* ops, int64_t* counts);
/* The last step as a seqpipe.simreport.v1 document with MEASURED values (requires
 * SP_FLAG_TIMELINE): task start/end in integer ns from the step start, per-device busy / idle /
 * bubble ratios (sim.cpp:234-274 definitions), memory in bytes of activation records and
 * KV-prefix slabs (+ at F end, - at B end). Text out via (buf, len) as sp_schedule_to_json. */
int sp_engine_report_json(sp_engine* eng, int32_t indent, int64_t memory_downsample, char* buf, size_t* len);
int sp_engine_render_gantt(sp_engine* eng, int32_t format, int32_t width, char* buf, size_t* len);
/* Per-op measured timeline of the last step (requires SP_FLAG_TIMELINE): start/end in ms. */
int sp_engine_timeline(sp_engine* eng, double* start_ms, double* end_ms, int64_t* n);
/* Parameter / gradient access in fp32. Names: "embed", "pos", "final_norm", "lm_head",
 * "layer<i>.<norm1|wqkv|wo|norm2|w1|w2>" with i the global layer index. */
int sp_engine_param_count(sp_engine* eng, int64_t* n);
int sp_engine_param_info(sp_engine* eng, int64_t idx, char* name, size_t name_len, int64_t* numel,
                         int32_t* rows, int32_t* cols);
int sp_engine_read_param(sp_engine* eng, const char* name, float* out, int64_t numel);
int sp_engine_read_grad(sp_engine* eng, const char* name, float* out, int64_t numel);
int sp_engine_write_param(sp_engine* eng, const char* name, const float* in, int64_t numel);
/* Synchronise and report device memory in use by the engine. */
int sp_engine_memory(sp_engine* eng, double* allocated_bytes, double* device_free_bytes);

/* ---- kernel-level entry points (tests + microbenchmarks) ---- */
/* C[M,N] = A · B with A [M,K] (a_kmajor) or [K,M], B [N,K] (b_kmajor) or [K,N], all device
 * pointers; dtype SP_DTYPE_BF16 inputs with fp32 output when c_f32 != 0, else bf16 output.
 * accumulate != 0: C += A·B (fp32 C only). impl: 0 auto, 1 SIMT, 2 tcgen05. */
int sp_gemm(int32_t dtype, int32_t impl, const void* A, int32_t a_kmajor, const void* B,
            int32_t b_kmajor, void* C, int32_t c_f32, int32_t accumulate, int64_t M, int64_t N,
            int64_t K, void* stream);
/* Causal attention of a query block at global offset q_off over a KV prefix of kv_len rows.
 * q [n, H*hd], kv [kv_len, 2*H*hd] (K then V per row), o [n, H*hd], lse [H, n] fp32. */
int sp_attention_fwd(int32_t dtype, int32_t impl, const void* q, const void* kv, void* o, float* lse,
                     int64_t n, int64_t q_off, int64_t kv_len, int32_t heads, int32_t head_dim,
                     void* stream);
/* dq [n, H*hd] (dtype), dkv_acc [kv_len, 2*H*hd] fp32 accumulated (+=). */
int sp_attention_bwd(int32_t dtype, int32_t impl, const void* q, const void* kv, const void* o,
                     const void* dout, const float* lse, void* dq, float* dkv_acc, int64_t n,
                     int64_t q_off, int64_t kv_len, int32_t heads, int32_t head_dim, void* stream);
/* Row norm of x [n, h] (LayerNorm, or RMSNorm when rms != 0) with gain g [h] fp32; saves
 * mean (LayerNorm only) and rstd [n] fp32. Backward: dx = d(norm)/dx^T dy (+ dres when
 * non-null), dg [h] fp32 accumulated (+=). */
int sp_norm_fwd(int32_t dtype, int32_t rms, const void* x, const float* g, void* y, float* mean,
                float* rstd, int64_t n, int32_t h, float eps, void* stream);
int sp_norm_bwd(int32_t dtype, int32_t rms, const void* dy, const void* x, const float* g,
                const float* mean, const float* rstd, const void* dres, void* dx, float* dg,
                int64_t n, int32_t h, void* stream);
/* MLP activation: family SP_MODEL_GPT = GeLU(tanh) of u [n, F]; SP_MODEL_LLAMA = SwiGLU of
 * u [n, 2F] = [gate | up] -> [n, F]. Backward writes du (same shape as u). */
int sp_act_fwd(int32_t dtype, int32_t family, const void* u, void* out, int64_t n, int32_t F,
               void* stream);
int sp_act_bwd(int32_t dtype, int32_t family, const void* u, const void* dout, void* du, int64_t n,
               int32_t F, void* stream);
int sp_device_synchronize(int32_t cuda_device);
int sp_cuda_device_count(int32_t* n);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* SEQPIPE_B200_H_ */
