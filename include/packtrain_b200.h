/*
 * packtrain_b200.h — C-ABI of the B200-native pack primitive.
 *
 * K static MLPs ("members") are trained as one packed network on one B200,
 * fed by shared input streams.  This ABI is the boundary a host binding
 * (ctypes here; cgo/JNI would bind the same symbols) calls in place of the
 * reference's numpy engine.  Every entry point names the reference function
 * it replaces (paths relative to /root/reference/pkg/src/packtrain/).
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch / CUDA types in signatures
 *     (a stream is passed as `void*` holding a cudaStream_t).
 *   - Host buffers are borrowed for the duration of a call only.
 *   - Every function returns a PK_* status; details via pk_ctx_last_error().
 *   - Parameters cross the boundary as float64 in the reference's layout:
 *     per affine layer l = 0..n_layers-1, W_l row-major [dims[l], dims[l+1]]
 *     (x @ W, engine.py:201) then b_l [dims[l+1]].  Optimizer slots follow
 *     the same flat layout, one block per slot in the order
 *     momentum:{velocity} adagrad:{accum} adam:{m, v} (engine.py:307-317).
 *   - Device precision is chosen per context (PK_F32 default, PK_F64);
 *     f64 -> f32 conversion is IEEE round-to-nearest, so get(set(x)) ==
 *     float32(x) bit-exactly.
 *   - Not thread-safe per context: one host thread drives one context
 *     (the reference's packed_step is not reentrant).
 */
#ifndef PACKTRAIN_B200_H
#define PACKTRAIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_ABI_VERSION 1
#define PK_MAX_LAYERS 8 /* affine layers per member (hidden <= 7) */

/* status codes */
#define PK_OK 0
#define PK_ERR_ARG 1            /* bad argument / shape (ShapeMismatch, PackError) */
#define PK_ERR_NONFINITE_VALUE 2 /* forward node non-finite: EngineError, engine.py:233-235 */
#define PK_ERR_NONFINITE_GRAD 3  /* NonFiniteGradient, engine.py:297-299 */
#define PK_ERR_OOM 4            /* device allocation failed */
#define PK_ERR_CUDA 5           /* CUDA runtime error */
#define PK_ERR_STATE 6          /* API misuse (e.g. pending async step) */
#define PK_SKIPPED 7            /* step status: skipped, an earlier in-flight step failed */

/* enums follow the reference tuples' order (engine.py:21-22) */
#define PK_ACT_SIGMOID 0
#define PK_ACT_LEAKY_RELU 1
#define PK_ACT_TANH 2
#define PK_ACT_RELU 3
#define PK_OPT_SGD 0
#define PK_OPT_MOMENTUM 1
#define PK_OPT_ADAM 2
#define PK_OPT_ADAGRAD 3
#define PK_F32 0
#define PK_F64 1

typedef struct pk_ctx pk_ctx;
typedef struct pk_dataset pk_dataset;
typedef struct pk_order pk_order;
typedef struct pk_member pk_member;
typedef struct pk_pack pk_pack;

/* Static description of one member (replaces MLPArch + make_optimizer,
 * packing.py:32-38 / engine.py:99-105). */
typedef struct {
  int32_t n_layers;                   /* affine layers = len(hidden) + 1 */
  int32_t dims[PK_MAX_LAYERS + 1];    /* input_dim, hidden..., classes */
  int32_t activation;                 /* PK_ACT_* (hidden layers) */
  int32_t optimizer;                  /* PK_OPT_* */
  double learning_rate;               /* > 0 */
  double weight_decay;                /* coupled L2 extension; 0 = reference */
  int32_t max_rows;                   /* batch_size: rows per step <= this */
  int32_t reserved;
} pk_member_desc;

/* One member's input for one packed step (replaces _next_batch + pad/mask,
 * packing.py:161-172, :213-239).  Row r of the batch is dataset row
 * order[pos + r] (or pos + r when order is NULL), r < take.  take == 0
 * marks the member inactive for this step (finished / parked). */
typedef struct {
  const pk_dataset* data;
  const pk_order* order;
  int64_t pos;
  int32_t take;
  int32_t group; /* input-group id (members with equal ids share rows) */
} pk_feed;

/* Outcome of one packed step (reference exception semantics,
 * packing.py:246-253): on PK_ERR_NONFINITE_VALUE nothing commits; on
 * PK_ERR_NONFINITE_GRAD the members before `member` (pack order) commit. */
typedef struct {
  int32_t code;      /* PK_OK / PK_ERR_NONFINITE_VALUE / PK_ERR_NONFINITE_GRAD */
  int32_t member;    /* offending member index in the pack, else -1 */
  int32_t index;     /* value error: node index (0=in, 2l+1=aff l, 2l+2=act l,
                        2n=loss); grad error: position in the grads order
                        W_{n-1}, b_{n-1}, ..., W_0, b_0 (engine.py:270-271) */
  int32_t committed; /* members whose update committed */
} pk_status;

/* ---- kernel plan (MLP pack path) ----------------------------------------
   Which kernel family trains which member is decided when a pack is created,
   from the member shapes and these process-wide options.  The defaults are the
   production plan; the other values exist for A/B measurements and for tests
   that pin a family.  pk_pack_kernel_plan() reports what a pack actually got. */
typedef struct pk_plan_options {
  int32_t fwd;          /* tensor-path forward: 0 auto (k_m1c_fwd when its clusters fit one
                           wave, k_m1s_fwd past two waves, else k_m1t_fwd), 1 split-K clusters
                           k_m1t_fwd only, 2 streaming k_m1s_fwd whenever it fits */
  int32_t fwd_cluster;  /* cap on the k_m1c_fwd cluster size (0 = none) */
  int32_t tcgen05;      /* 1: tensor path for eligible fp32 one-hidden-layer members */
  int32_t mlp1;         /* 1: fused FFMA one-hidden-layer kernels where eligible */
  int32_t m1x;          /* 1: one-launch FFMA cluster step k_m1x_step (experimental; slower) */
  int32_t fwd_split;    /* 1: k_phase FWD input ranges */
  int32_t wgrad_narrow; /* 1: 64x16 WGRAD tiles for layers with <= 16 outputs */
  int32_t inline_desc;  /* 1: step descriptors inline in the graph's kernel parameters */
  int32_t run_batch;    /* steps per graph launch in pk_pack_run (0 = 8) */
  int32_t trace;        /* 1: %globaltimer stage stamps (pk_pack_trace) */
  int32_t conv_cluster; /* conv path, read when a program is created: 1 (default) FPROP /
                           DGRAD GEMMs with TMA-fed operands and K >= 512 run on CTA pairs
                           that multicast the weight tile (k_conv_gemm_pc); 2 = CTA-pair
                           M=256 tcgen05.mma.cta_group::2 (k_conv_gemm_p2, bit-identical,
                           no measured gain); 0 = one CTA per tile */
  int32_t conv_halo;    /* conv path: 1 (default) 3x3 stride-1 FPROP / DGRAD with C % 64 == 0,
                           >= 14-wide outputs and 256-wide N tiles stage one halo box per
                           channel block and run the nine taps on shifted operand
                           descriptors (k_conv_gemm_halo); 0 = TMA im2col per tap */
  int32_t reserved[4];
} pk_plan_options;
int pk_plan_options_get(pk_plan_options* out);
int pk_plan_options_set(const pk_plan_options* in); /* NULL restores the defaults */

/* ---- context ------------------------------------------------------------ */
int pk_abi_version(void);
int pk_ctx_create(int32_t device, int32_t dtype, pk_ctx** out);
int pk_ctx_destroy(pk_ctx* ctx);
const char* pk_ctx_last_error(const pk_ctx* ctx);
int pk_ctx_set_stream(pk_ctx* ctx, void* cuda_stream); /* NULL = own stream */
int pk_ctx_synchronize(pk_ctx* ctx);
int pk_ctx_mem_info(pk_ctx* ctx, uint64_t* free_bytes, uint64_t* total_bytes,
                    uint64_t* ctx_bytes);

/* ---- data (replaces Dataset / epoch_permutation / batch_at storage,
 *      data.py:18-39, :124-136): device-resident copies ------------------- */
int pk_dataset_create(pk_ctx* ctx, int64_t n, int32_t dim, pk_dataset** out);
/* write rows [row0, row0+rows) from host f64 features / int64 labels */
int pk_dataset_write(pk_dataset* ds, int64_t row0, int64_t rows,
                     const double* features, const int64_t* labels);
/* streamed inputs: rows [row0, row0+rows) already in the context's device
 * precision (float32 / float64) and int32 labels, copied asynchronously on
 * the context stream (the host buffers must stay valid until the next sync;
 * pinned memory makes the copy a true DMA).  Replaces the per-step batch of
 * _next_batch (packing.py:161-172) when datasets live on the host. */
int pk_dataset_write_rows(pk_dataset* ds, int64_t row0, int64_t rows, const void* features,
                          const int32_t* labels);
/* Streamed inputs in one call: gather host rows idx[0..rows) (device
 * precision, row stride src_ld elements; labels int32) into the pinned
 * staging buffers, then enqueue the same H2D as pk_dataset_write_rows into
 * rows [0, rows).  Replaces the reference's per-step batch gather
 * (reference data.py:131-136) on the host-resident input path. */
int pk_dataset_gather_rows(pk_dataset* ds, int64_t rows, const void* src_features, int64_t src_ld,
                           const int32_t* src_labels, const int64_t* idx, void* stage_features,
                           int32_t* stage_labels);

/* Page-lock a host buffer and map it into the device address space
 * (cudaHostRegister, mapped); *dev receives the device view.  Streamed inputs
 * whose rows the GPU gathers itself over PCIe (pk_pack_run) avoid the host-side
 * memcpy + copy calls of pk_dataset_gather_rows.  pk_host_unmap undoes it. */
int pk_host_map(pk_ctx* ctx, void* host, int64_t bytes, void** dev);
int pk_host_unmap(pk_ctx* ctx, void* host);
int pk_dataset_destroy(pk_dataset* ds);
int pk_order_create(pk_ctx* ctx, const int64_t* perm, int64_t n, pk_order** out);
int pk_order_destroy(pk_order* order);

/* ---- members (replaces ModelHandle params + OptimizerState,
 *      packing.py:52-81, engine.py:85-96) -------------------------------- */
int pk_member_create(pk_ctx* ctx, const pk_member_desc* desc, pk_member** out);
int pk_member_destroy(pk_member* m);
int64_t pk_member_param_count(const pk_member* m);
int32_t pk_member_slot_count(const pk_member* m);
int64_t pk_member_device_bytes(const pk_member* m);
int pk_member_set_lr(pk_member* m, double learning_rate);
/* upload params (and slots when non-NULL, else zeros) + step counter */
int pk_member_set_state(pk_member* m, const double* params, const double* slots,
                        int64_t step_counter);
/* download committed params / slots (either may be NULL) + step counter */
int pk_member_get_state(pk_member* m, double* params, double* slots,
                        int64_t* step_counter);
/* testing hook (fault injection): the member's next step sees a NaN in the
 * gradient tensor at `grad_position` (grads order, see pk_status.index);
 * -1 clears.  Exercises the NonFiniteGradient commit rules. */
int pk_member_inject_fault(pk_member* m, int32_t grad_position);

/* ---- packs (replaces pack_models / packed_step / standalone_step,
 *      packing.py:136-142, :185-282) ------------------------------------- */
int pk_pack_create(pk_ctx* ctx, pk_member* const* members, int32_t k, pk_pack** out);
int pk_pack_destroy(pk_pack* p);
/* one synchronous packed step: losses[k] (float64) for active members */
int pk_pack_step(pk_pack* p, const pk_feed* feeds, double* losses, pk_status* st);
/* asynchronous form for pipelined drivers: enqueue, then wait by ticket */
int pk_pack_step_async(pk_pack* p, const pk_feed* feeds, int64_t* ticket);
int pk_pack_step_wait(pk_pack* p, int64_t ticket, double* losses, pk_status* st);

/* ---- native multi-step driver (reference packing.py:185-264, looped) ------
 * Up to `max_steps` packed steps with up to `depth` (<= 32) in flight,
 * planned and applied in C: active members, epoch rolls, input groups sorted
 * by (dataset, epoch, pos, batch), rows perm[pos : pos + take], label bound
 * checks, per-step feeds (device-resident order or streamed rows gathered
 * into pinned slots), and at result time the cursor updates
 * (steps_done, pos, samples_used[idx] += 1) with the reference's commit rules.
 * `mem` (K entries, pack order) is updated in place.  Outputs per completed
 * step i: losses[i*K + k], active[i*K + k] (1 = member k stepped and
 * committed), stats[3*i .. 3*i+2] = (groups, physical inputs, driver batch).
 * The loop stops before a step it cannot plan alone (*stop, PK_RUN_*); a
 * failed step is reported in *st (not counted in *done). */
typedef struct {
  int32_t dataset;        /* index into the run's datasets */
  int32_t batch;          /* batch size */
  int64_t epoch, pos, steps_done, target_steps; /* cursor (in/out) */
  int64_t* samples_used;  /* [n] use counts of the current epoch (in/out), or NULL */
} pk_run_member;

typedef struct {
  int64_t n;
  int32_t dim;
  int32_t max_label;
  const void* host_x;     /* streamed inputs: host rows in device precision, or NULL */
  int64_t host_ld;        /* row stride of host_x (elements) */
  const int32_t* host_y;  /* host labels (always; label bound checks) */
  const pk_dataset* device;     /* device-resident inputs (host_x == NULL) */
  int64_t epoch0;               /* permutations / orders given for epochs */
  int32_t n_epochs;             /*   epoch0 .. epoch0 + n_epochs - 1 */
  const int64_t* const* perm;   /* host permutations */
  const pk_order* const* order; /* device orders (device-resident inputs; streamed inputs
                                   with mapped_x use them for the on-device gather) */
  const void* mapped_x;         /* streamed inputs: device view of host_x (pk_host_map), or NULL */
  const int32_t* mapped_y;      /* device view of host_y */
} pk_run_dataset;

#define PK_RUN_MAX_STEPS 0    /* ran max_steps */
#define PK_RUN_NO_MEMBER 1    /* every member reached target_steps */
#define PK_RUN_NEED_PERM 2    /* the next step needs a permutation not given */
#define PK_RUN_LABEL_BOUNDS 3 /* the next step's labels exceed a member's classes */
#define PK_RUN_FAILED 4       /* a step failed (non-finite); see *st */

int pk_pack_run(pk_pack* p, pk_run_member* mem, const pk_run_dataset* ds, int32_t n_ds,
                int32_t share_inputs, int64_t max_steps, int32_t depth, double* losses,
                uint8_t* active, int32_t* stats, int64_t* done, pk_status* st, int32_t* stop);
/* forward-only mean softmax-xent of every member on `rows` rows of one
 * dataset (order NULL = rows 0..rows-1); replaces EngineExecutor._val_loss
 * (tuner.py:460-464).  Nothing is updated. */
int pk_pack_eval(pk_pack* p, const pk_dataset* data, const pk_order* order,
                 int64_t pos, int64_t rows, double* losses, pk_status* st);
/* profiling: run one real step un-graphed with CUDA events around every
 * phase (state advances as for pk_pack_step).  Arrays hold
 * pk_pack_launches_per_step(p) entries: device ms, kind (a k_phase tile kind
 * 0..4, or 16 + id for the fused kernels: 17 k_mlp1_fwd, 18 k_mlp1_bwd,
 * 19 k_m1t_fwd, 20 k_m1t_bwd, 21 k_m1s_fwd, 22 k_m1c_fwd), layer index, and
 * tile (CTA) count. */
int pk_pack_profile_step(pk_pack* p, const pk_feed* feeds, float* phase_ms,
                         int32_t* phase_kind, int32_t* phase_layer,
                         int32_t* phase_ctas, double* losses, pk_status* st);
/* profiling: with PK_TRACE=1 in the environment at pack creation, every CTA
 * of every train phase stamps %globaltimer (ns) at 8 stage boundaries
 * (entry, operands ready, GEMM done, epilogue 1, epilogue 2, tile done,
 * finalize start, finalize end) of the most recent step.  Layout:
 * [phase][cta][8].  Returns the element count (-1 when tracing is off). */
int64_t pk_pack_trace(pk_pack* p, uint64_t* out, int64_t cap);
/* number of kernel launches one pk_pack_step enqueues */
int32_t pk_pack_launches_per_step(const pk_pack* p);

/* ======================================================================
 * Conv pack path (BASELINE configs 1-4: LeNet / MobileNetV2 / ResNet /
 * DenseNet members).  The reference engine has no conv layers
 * (SPEC.md:15, :90); these entry points extend its pack primitive
 * (packing.py:185-264 packed_step semantics: shared input groups, per-member
 * valid rows, one optimizer step per member) to conv members.  Activations
 * are NHWC bf16, GEMMs run on tcgen05 (bf16 operands, fp32 accumulate),
 * master weights and optimizer slots are fp32.
 * ====================================================================== */
typedef struct pk_conv_geom {
  int32_t n, h, w, c;            /* input NHWC (c a multiple of 8) */
  int32_t k, r, s, stride, pad;  /* output channels, filter, stride (1|2), pad */
  int32_t p, q;                  /* output spatial dims */
} pk_conv_geom;

/* One implicit-GEMM conv on caller-owned device buffers (unit-test and
 * microbenchmark hook of the kernel every conv layer uses).
 *   mode 0 FPROP: out bf16 [n*p*q][k]  = conv(x bf16 [n,h,w,c], w bf16 [k][kpad]),
 *                 kpad = roundup(r*s*c, 64), w[k][(r*s_+s)*c + ci]
 *   mode 1 DGRAD: out bf16 [n*h*w][c]  from dy bf16 [n*p*q][k] and the transposed
 *                 weights w = wt bf16 [c][roundup(r*s*k, 64)], wt[ci][(r*s_+s)*k + co]
 *   mode 2 WGRAD: out f32 [splits][k][kpad] partial sums over pixel splits
 * ntile: GEMM N tile (16..256, multiple of 16; of 64 for WGRAD); stages 2..6. */
int pk_conv_gemm_test(int32_t mode, const pk_conv_geom* g, const void* x, const void* w,
                      const void* dy, void* out, int32_t ntile, int32_t splits,
                      int32_t stages, void* stream);

/* ----------------------------------------------------------------------
 * Conv pack program.  A packed conv train step is a fixed sequence of
 * grouped kernel launches ("ops"); each op covers one layer of every member
 * of the pack (nprob problems, one per member / input group), so a K-member
 * pack of identical nets costs the launches of one net.  The host planner
 * (paper_2002_02885_b200/cnn.py) owns the device buffers (HBM layout in
 * DESIGN.md §3b) and describes every launch with the structs below; the
 * program copies the descriptors to the device once and replays them
 * (optionally as one CUDA graph) every step.  All tensors are NHWC with a
 * pixel-row stride (ld*) in elements; channel counts are multiples of 8.
 * Activations / GEMM operands are bf16, master weights, optimizer slots,
 * BN statistics and gradients fp32.
 * ---------------------------------------------------------------------- */
#define PK_CNN_CONV_FPROP 0     /* implicit-GEMM conv forward (tcgen05)          */
#define PK_CNN_CONV_DGRAD 1     /* implicit-GEMM conv data gradient (tcgen05)    */
#define PK_CNN_CONV_WGRAD 2     /* implicit-GEMM conv weight gradient (tcgen05)  */
#define PK_CNN_BN_STATS 3       /* batch mean / rstd over valid rows             */
#define PK_CNN_BN_APPLY 4       /* y -> act(bn(y) [+ residual])                  */
#define PK_CNN_BN_BWD_REDUCE 5  /* dgamma, dbeta, Σg / Σg·xhat                   */
#define PK_CNN_BN_BWD_APPLY 6   /* dx (and the residual gradient)                */
#define PK_CNN_DW_FPROP 7       /* depthwise conv forward                        */
#define PK_CNN_DW_DGRAD 8
#define PK_CNN_DW_WGRAD 9
#define PK_CNN_MAXPOOL_FWD 10
#define PK_CNN_MAXPOOL_BWD 11
#define PK_CNN_AVGPOOL_FWD 12
#define PK_CNN_AVGPOOL_BWD 13
#define PK_CNN_XENT 14          /* softmax cross-entropy head (+ last bias grad) */
#define PK_CNN_BIAS_ACT_BWD 15  /* g = dy·act'(out), dbias = Σ_rows g            */
#define PK_CNN_SPLIT_REDUCE 16  /* dW = Σ_split partials (fixed order)           */
#define PK_CNN_OPT 17           /* fused multi-member optimizer + bf16 publish   */
#define PK_CNN_PUBLISH_T 18     /* transposed bf16 weights for DGRAD             */
#define PK_CNN_COMMIT 19        /* per-member step counter / non-finite verdict  */
#define PK_CNN_GATHER 20        /* batch rows src[idx[i]] -> dst[i] (e.g. over PCIe) */
#define PK_CNN_IM2COL 21        /* dense im2col rows of a narrow input (first conv)  */
#define PK_CNN_NUM_KINDS 22

#define PK_CNN_ACT_NONE 0
#define PK_CNN_ACT_RELU 1
#define PK_CNN_ACT_RELU6 2

/* conv geometry of the forward conv: x [n,h,w,c] * W [k][r][s][c] -> y [n,p,q,k] */
typedef struct pk_cnn_conv {
  const void* src;        /* FPROP/WGRAD: x (pixel stride ldx); DGRAD: dy (stride ldy) */
  const void* dy;         /* WGRAD: dy (stride ldy) */
  const void* wt;         /* FPROP: W16 bf16 [k][kpad]; DGRAD: Wt16 bf16 [c][kpadt] */
  void* dst;              /* FPROP: y (bf16, or fp32 if out_f32), stride ldo;
                             DGRAD: dx bf16 stride ldo; WGRAD: fp32 [splits][k][kpad] */
  const int64_t* idx;     /* FPROP/WGRAD: batch image i reads source image idx[i] */
  const float* bias;      /* FPROP: per output channel (NULL = none) */
  int32_t* flag;          /* WGRAD (splits == 1): member's non-finite flag */
  int64_t dseg;           /* FPROP concat-N: elements between member segments of dst;
                             WGRAD concat-N: elements between the members' dy buffers */
  int32_t n, h, w, c, k, r, s, stride, pad, p, q;
  int32_t ldx, ldy, ldo;
  int32_t act;            /* FPROP: PK_CNN_ACT_* after bias */
  int32_t out_f32;        /* FPROP: dst fp32 */
  int32_t accumulate;     /* DGRAD: dst += result */
  int32_t splits;         /* WGRAD: pixel splits */
  int32_t nseg;           /* FPROP concat-N: output channels per member segment (0 = one);
                             WGRAD concat-N (k = members x 64, nseg = 64, splits >= 2): one
                             GEMM over the shared input for all members, member j's fp32
                             partials [splits][64][kpad] at dst + j*splits*64*kpad */
} pk_cnn_conv;

/* batch norm over the `rows` valid rows of one member (BN_* kinds) */
typedef struct pk_cnn_bn {
  const void* x;          /* pre-norm y (bf16, stride ldx) */
  const void* res;        /* APPLY: residual added before act (bf16, stride ldr) or NULL */
  void* out;              /* APPLY: act(bn(x) + res) (bf16, stride ldo) */
  const void* dout;       /* BWD: dL/d out (bf16, stride ldd) */
  const void* fout;       /* BWD: forward out, for act' (bf16, stride ldo) */
  void* dx;               /* BWD_APPLY: dL/dx (bf16, stride ldx2) */
  void* dres;             /* BWD_APPLY: dL/d res = g (bf16, stride ldr) or NULL */
  const float* gamma;
  const float* beta;
  float* dgamma;          /* BWD_REDUCE: gradient slab entries */
  float* dbeta;
  float* stats;           /* [4][c]: mean, rstd, mean(g), mean(g·xhat) */
  float* run_mean;        /* STATS: running statistics (torch momentum rule) or NULL */
  float* run_var;
  float* ws;              /* partials workspace (see rpb) */
  int32_t* counter;       /* int32[17], zero-initialised; the kernels reset it */
  int32_t* flag;          /* member's non-finite flag */
  int32_t rows, c, ldx, ldo, ldr, ldd, ldx2;
  int32_t act;            /* PK_CNN_ACT_* */
  int32_t accumulate;     /* BWD_APPLY: dx += */
  int32_t res_accumulate; /* BWD_APPLY: dres += */
  int32_t use_running;    /* APPLY: normalise with running stats (eval) */
  float eps, momentum;
  int32_t rpb;            /* STATS / BWD_REDUCE: rows per partial block (multiple of 32),
                             ceil(rows/rpb) <= 256; ws >= nblk*2c floats + (ceil(nblk/16)
                             + 1)*2c doubles (+1 float of alignment) */
  int32_t pad0;
} pk_cnn_bn;

/* depthwise r x s conv (groups = c), weights bf16 [r*s][c] / gradient fp32 [r*s][c] */
typedef struct pk_cnn_dw {
  const void* x;          /* FPROP/WGRAD input (stride ldx) */
  const void* wt;         /* FPROP/DGRAD: W16 bf16 [r*s][c] */
  const void* dy;         /* DGRAD/WGRAD (stride ldy) */
  void* y;                /* FPROP output (stride ldy) / DGRAD dx (stride ldx) */
  float* dw;              /* WGRAD gradient [r*s][c] */
  float* ws;              /* WGRAD partials */
  int32_t* counter;
  int32_t* flag;
  int32_t n, h, w, c, r, s, stride, pad, p, q, ldx, ldy;
  int32_t ppb;            /* WGRAD: output pixels per partial block (<= 256 blocks);
                             ws as pk_cnn_bn with r*s*c outputs; counter int32[17] */
  int32_t pad0;
} pk_cnn_dw;

/* pooling: max (window r x s, stride, pad; argmax kept as uint8) or average */
typedef struct pk_cnn_pool {
  const void* x;          /* FWD input (stride ldx) */
  void* y;                /* FWD output (stride ldy) */
  const void* dy;         /* BWD (stride ldy) */
  void* dx;               /* BWD (stride ldx) */
  uint8_t* arg;           /* MAXPOOL: argmax tap per output element [n*p*q][c] */
  int32_t n, h, w, c, r, s, stride, pad, p, q, ldx, ldy;
  int32_t accumulate;     /* BWD: dx += */
} pk_cnn_pool;

/* softmax cross-entropy over the member's `rows` rows (mean), reference
 * engine.py:211-230 / :252-264 */
typedef struct pk_cnn_head {
  const float* logits;    /* fp32 [rows][ldl] (bias already added) */
  const int64_t* labels;  /* dataset labels */
  const int64_t* idx;     /* batch row i has label labels[idx[i]] */
  void* dlogits;          /* bf16 [rows][ldl] (NULL = loss only, eval) */
  float* dbias;           /* last-layer bias gradient [classes] or NULL */
  float* loss;            /* member's loss (mean over rows) */
  int32_t* flag;
  int32_t rows, classes, ldl;
} pk_cnn_head;

/* g = dy · act'(fout), written bf16; dbias = Σ_rows g */
typedef struct pk_cnn_bias {
  const void* dy;         /* stride ld */
  const void* fout;       /* stride ld */
  void* g;                /* stride ld (may alias dy) */
  float* dbias;
  float* ws;
  int32_t* counter;
  int32_t* flag;
  int32_t rows, c, ld, act;
  int32_t rpb;            /* rows per partial block; ws as pk_cnn_bn */
  int32_t pad0;
} pk_cnn_bias;

/* dst[i] = Σ_{j<splits} src[j*len + i] (j in order) */
typedef struct pk_cnn_reduce {
  const float* src;
  float* dst;
  int32_t* flag;
  int64_t len;
  int32_t splits, pad0;
} pk_cnn_reduce;

/* one contiguous parameter segment of one member for the fused optimizer */
typedef struct pk_cnn_opt_seg {
  float* w;               /* fp32 master */
  const float* g;         /* gradient */
  float* s1;              /* slot 1 (velocity / accum / adam m) or NULL */
  float* s2;              /* slot 2 (adam v) or NULL */
  void* w16;              /* bf16 mirror (GEMM operand) or NULL */
  const int32_t* step;    /* member step counter (t-1) */
  const int32_t* flag;    /* member's commit verdict (COMMIT mode 0): skip if set */
  int64_t len;
  int32_t kind;           /* PK_OPT_* */
  float lr, wd;
} pk_cnn_opt_seg;

/* Wt16[ci][(r*s_+s)*kp + co] = W16[co][(r*s_+s)*cp + ci] */
typedef struct pk_cnn_tpose {
  const void* src;
  void* dst;
  int32_t k, c, taps, kpad, kpadt, pad0;
} pk_cnn_tpose;

/* per-member commit (op cfg0 = mode).  mode 0, before PK_CNN_OPT: verdict =
 * OR of the flags of this and every earlier problem (the reference's update
 * loop stops at the first non-finite member, packing.py:250-253); mode 1,
 * after it: if (!verdict) ++step; verdict |= (flag != 0) << 1; flag = 0. */
typedef struct pk_cnn_commit {
  int32_t* step;
  int32_t* flag;
  int32_t* verdict;
} pk_cnn_commit;

/* dst row i = src row idx[i] (row_bytes a multiple of 16); src may be
 * page-locked host memory (read by the GPU over PCIe) */
typedef struct pk_cnn_gather {
  const void* src;
  void* dst;
  const int64_t* idx;
  int64_t row_bytes;
  int32_t rows, pad0;
} pk_cnn_gather;

/* Dense im2col of a narrow network input for the first conv: dst row m =
 * (n, oy, ox) holds the r*s*c real input values of its window, (tap, channel)
 * order, zero past the plane, zero-padded to ldo (a multiple of 8) columns.
 * The first conv then runs as a 1x1 GEMM over these rows with K = ldo instead
 * of r*s*cp (cp = the input's padded channel pitch, 16): a 7x7x3 stem reads
 * 152 columns instead of 784. */
typedef struct pk_cnn_im2col {
  const void* src; /* bf16 [n][h][w][cp], c <= 8 real channels */
  void* dst;       /* bf16 [n*p*q][ldo]  */
  int32_t n, h, w, cp, c, r, s, stride, pad, p, q, ldo;
} pk_cnn_im2col;

typedef struct pk_cnn_op {
  int32_t kind;           /* PK_CNN_* */
  int32_t nprob;
  int32_t cfg0;           /* CONV: GEMM N tile */
  int32_t cfg1;           /* CONV: pipeline stages */
  int32_t lane;           /* 0: the program's stream.  L > 0: an independent chain (the
                             members of one architecture in a heterogeneous pack) that
                             forks from lane 0 after the last lane-0 op before it and
                             joins lane 0 before the next lane-0 op, so different lanes'
                             launches overlap on the GPU.  16 + a (a = 1..8): async lane
                             a — the op waits for everything its parent stream (lane a
                             while that lane is open, else the program stream) issued
                             before it, and lane 0 joins it only before the next COMMIT /
                             OPT op (weight gradients overlap the rest of the backward) */
  int32_t pad0;
  const void* probs;      /* nprob structs of the kind's type (host, copied) */
} pk_cnn_op;

typedef struct pk_cnn_prog pk_cnn_prog;

/* Build a program on `device` from nops op descriptors (host memory, copied). */
int pk_cnn_prog_create(const pk_cnn_op* ops, int32_t nops, int32_t device, pk_cnn_prog** out);
void pk_cnn_prog_destroy(pk_cnn_prog* p);
/* Enqueue the whole program on `stream`; use_graph != 0 captures it once into
 * a CUDA graph and replays that graph on later calls. */
int pk_cnn_prog_run(pk_cnn_prog* p, void* stream, int32_t use_graph);
/* Run op by op, bracketing each op with CUDA events; op_ms[i] = duration. */
int pk_cnn_prog_profile(pk_cnn_prog* p, void* stream, float* op_ms);
/* kernel launches one run enqueues */
int32_t pk_cnn_prog_launches(const pk_cnn_prog* p);
/* last error of the conv pack path on this thread */
const char* pk_cnn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PACKTRAIN_B200_H */
