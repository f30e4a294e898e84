/*
 * sdp.h — C ABI of libsdp.so, the B200 (sm_100a) hot path of Subnetwork Data
 * Parallelism (arXiv 2507.09029).
 *
 * The reference (`/root/reference/pkg/src/subnetdp`) has no FFI: its boundary
 * is a set of Python functions over numpy arrays.  These entry points are what
 * those functions bind to in this framework (see INTEGRATION.md for the ctypes
 * stub a maintainer adds, and paper_2507_09029_b200/_native.py for ours).
 *
 *   reference function (file:line)                     replaced by
 *   -------------------------------------------------  -----------------------------
 *   masking.assign_units / assign_grouped_units        sdp_assign_units
 *     (masking.py:69-117) + slot_windows (:56-66)
 *   induce_channel_param_mask / induce_block_param_    sdp_build_masks
 *     mask (:120-170), _governor_counts (:288-302),
 *     MaskAssignment.__post_init__ coverage/divisor
 *     (:203-205), validate's active counts (:442)
 *   MaskAssignment.worker_view param_mask (:238-243)   sdp_worker_mask
 *   engine.aggregate (engine.py:60-79)                 sdp_plan_tiles + sdp_owner_sync
 *   models.masked_forward  theta * mask (models.py:355) sdp_masked_extract
 *   width-wise slice extraction (models.py:355-362)    sdp_gather_slices
 *   models.flat_gradient write-back (models.py:369-382) sdp_scatter_slices
 *   optim.SgdNesterov.update (optim.py:78-84)          sdp_nesterov_update / fused in
 *                                                      sdp_owner_sync (SDP_SYNC_NESTEROV)
 *
 * Conventions
 *   - Every function returns an int status: SDP_OK (0) or one of the SDP_ERR_*
 *     codes below, which the Python layer maps 1:1 onto the reference's
 *     exception classes (errors.py:8-45).  sdp_last_error() returns the message
 *     of the last failure on the calling thread.
 *   - All array pointers are DEVICE pointers owned by the caller unless marked
 *     "host".  libsdp never allocates device memory.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it.  Calls do not synchronise the device, except where noted.
 *   - No torch types appear here; the library links only the CUDA runtime.
 */
#ifndef SDP_H_
#define SDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDP_ABI_VERSION 2

/* status codes (errors.py:8-45) */
#define SDP_OK 0
#define SDP_ERR_CONFIG 1      /* ConfigError      */
#define SDP_ERR_TOPOLOGY 2    /* TopologyError    */
#define SDP_ERR_VALIDATION 3  /* ValidationError  */
#define SDP_ERR_PROTOCOL 4    /* ProtocolError    */
#define SDP_ERR_NUMERICAL 5   /* NumericalError   */
#define SDP_ERR_USAGE 6       /* UsageError       */
#define SDP_ERR_CUDA 7        /* CUDA runtime failure (no reference analogue) */

#define SDP_MAX_WORKERS 64

int sdp_abi_version(void);
const char* sdp_last_error(void);
/* Number of SMs of the current device (grid sizing helper). */
int sdp_device_sm_count(int* out);

/* *out = 1 iff ptr is page-locked host memory the current device reads and
 * writes through the SAME address (unified addressing): the zero-copy form of
 * engine.aggregate's host-buffer path (engine.py:60-79 on numpy inputs) hands
 * such pointers to sdp_owner_sync directly. */
int sdp_host_ptr_on_device(const void* ptr, int* out);

/* ------------------------------------------------------------------------ */
/* Mask builder                                                              */
/* ------------------------------------------------------------------------ */

/* One assignment group: units [first_unit, first_unit + size) drawn with one
 * permutation (masking.py:110-116).  Block strategy = a single group. */
typedef struct {
  int32_t first_unit;
  int32_t size;
} sdp_group_desc;

/* One parameter tensor of the flat vector (topology.py:16-23). */
typedef struct {
  int64_t offset;      /* flat offset of element 0 */
  int64_t size;        /* elements */
  int32_t rule_begin;  /* rules [rule_begin, rule_begin + rule_count) govern it */
  int32_t rule_count;
} sdp_param_desc;

/* Element e (0-based within its parameter) is governed by unit
 *   unit_base + (e / inner) % dim
 * -- an own/consumer slice along one axis (masking.py:140-149; inner is the
 * product of the trailing dims, dim the axis length) or, with inner = dim = 1,
 * a whole block (masking.py:167-169). */
typedef struct {
  int32_t inner;
  int32_t dim;
  int32_t unit_base;
  uint32_t inner_mul, inner_shr; /* q = umulhi(e, mul) >> shr == e / inner (e < 2^31) */
  uint32_t dim_mul, dim_shr;     /* same for / dim; mul = 0 encodes a divisor of 1 */
  int32_t pad_;
} sdp_rule_desc;

/* Seeded cyclic assignment (masking.py:56-117) on the device, bit-exact with
 * numpy's default_rng(seed).permutation (SeedSequence + PCG64).
 *   seed_words (host): the non-negative seed as little-endian uint32 words.
 *   groups (device):   n_groups descriptors, drawn in order from ONE generator.
 *   unit_bits (device, out): uint64 owner mask per unit; units outside every
 *                      group get all N bits (they are never masked).
 *   scratch (device):  >= 8 x n_units + 1 int32 (the parallel shuffle's
 *                      arrays: step targets, slots, buckets, chains).
 * Errors: SDP_ERR_CONFIG unless 1 <= P <= N <= 64 and groups are non-empty. */
int sdp_assign_units(const uint32_t* seed_words, int n_seed_words,
                     const sdp_group_desc* groups, int n_groups, int max_group,
                     int n_units, int n_workers, int replication,
                     uint64_t* unit_bits, int32_t* scratch, void* stream);

/* Same permutation as a standalone primitive: out[k] = default_rng(seed)
 * .permutation(n)[k] after `skip` earlier permutations of sizes skip_sizes
 * (host) were drawn from the same generator.  Used by tests. */
int sdp_permutation(const uint32_t* seed_words, int n_seed_words,
                    const int32_t* skip_sizes, int n_skip, int n,
                    int32_t* out, void* stream);

/* Expand unit ownership to every element of the flat vector.
 * Outputs (all device, each may be NULL):
 *   owner_mask   [d] elements of mask_bytes (1,2,4,8) bytes: bit w = worker w
 *   param_masks  [N, d] bool (reference layout, masking.py:131,160)
 *   coverage     [d] int64     (masking.py:204)
 *   divisor      [d] float64   max(coverage, 1) (masking.py:205)
 *   governors    [d] int64     number of governing rules (masking.py:288-302)
 *   active_counts [N] int64    params held per worker (masking.py:442); must be
 *                              zeroed by the caller, accumulated atomically. */
int sdp_build_masks(const sdp_param_desc* params, int n_params,
                    const sdp_rule_desc* rules, int n_rules,
                    const uint64_t* unit_bits, int n_workers, int64_t total,
                    void* owner_mask, int mask_bytes, uint8_t* param_masks,
                    int64_t* coverage, double* divisor, int64_t* governors,
                    int64_t* active_counts, void* stream);

/* Per-worker mask view (masking.py:238-243): for worker w,
 *   mask_f64[j] = bit w of owner_mask[j] ? 1.0 : 0.0   (nullable)
 *   mask_u8[j]  = bit w ? 1 : 0                         (nullable) */
int sdp_worker_mask(const void* owner_mask, int mask_bytes, int64_t total,
                    int worker, double* mask_f64, uint8_t* mask_u8, void* stream);

/* ------------------------------------------------------------------------ */
/* Owner-subset sync (engine.aggregate, engine.py:60-79)                     */
/* ------------------------------------------------------------------------ */

/* A tile is `tile` consecutive elements starting at tile_index * tile.
 * uniform tiles carry their owner set; mixed tiles read owner_mask. */
typedef struct {
  uint64_t owner_bits; /* uniform: the owner set; mixed: union of owner sets */
  uint32_t tile_index;
  uint32_t len_flags;  /* bits 0..23: length in elements; bit 31: uniform */
} sdp_tile_desc;

#define SDP_TILE_UNIFORM 0x80000000u
#define SDP_TILE_LEN_MASK 0x00FFFFFFu

/* Classify every tile of the flat vector (warp-shuffle AND/OR reduction).
 * tiles (device, out): ceil(total / tile) descriptors in tile order.
 * owned (device, out, nullable): per tile, sum over its elements of |O_j|
 * (the coverage sum, masking.py:203, without a [d] coverage table).
 * tile must be a multiple of 1024 and <= 1<<20. */
int sdp_plan_tiles(const void* owner_mask, int mask_bytes, int64_t total,
                   int tile, sdp_tile_desc* tiles, int64_t* owned, void* stream);

#define SDP_DTYPE_F32 0
#define SDP_DTYPE_F64 1

/* flags */
#define SDP_SYNC_WRITEBACK 0x1       /* write the mean into every owner's replica */
#define SDP_SYNC_CHECK_UNCOVERED 0x2 /* engine.py:75-78 leak check -> status */
#define SDP_SYNC_CHECK_FINITE 0x4    /* optim.py:79-80 isfinite(gbar) -> status */
#define SDP_SYNC_NESTEROV 0x8        /* fused optim.py:81-84 update on theta/vel */
#define SDP_SYNC_ADAM 0x10           /* fused optim.py:101-109 update on theta/m/v */
#define SDP_SYNC_LOCAL_UPDATE 0x20   /* NESTEROV / ADAM run as a third phase on the
                                        rank's local workers' (compact) state, after
                                        the exit barrier, instead of in the leader's
                                        epilogue on one flat theta */
#define SDP_SYNC_DIRECT 0x40         /* world 1, flat replicas, N <= 8 (small buffers;
                                        width-wise plans whose owners hold most of
                                        the vector):
                                        no tile table -- every thread loads its
                                        elements' owner masks and ALL N replicas at
                                        once (one DRAM round trip instead of the
                                        descriptor -> mask -> owners chain) and adds
                                        exactly each element's owners, ascending */
#define SDP_SYNC_STREAM 0x80         /* with SDP_SYNC_DIRECT: grid-stride over resident
                                        CTAs, replica loads only for the workers a
                                        warp's lanes own, the next vector's masks
                                        prefetched (owned-line traffic, one round
                                        trip per vector); a launch with no
                                        WRITEBACK / NESTEROV / ADAM runs the
                                        mean-only instantiation (whole-vector
                                        stores of the means, no epilogue) */

/* status word bits written (atomicOr) by the kernel */
#define SDP_STATUS_UNCOVERED_LEAK 0x1
#define SDP_STATUS_NONFINITE 0x2
#define SDP_STATUS_BARRIER_TIMEOUT 0x4

typedef struct {
  int32_t dtype;        /* SDP_DTYPE_F32 / SDP_DTYPE_F64: replicas, out, theta */
  int32_t n_workers;    /* N <= 64 */
  int32_t mask_bytes;   /* element size of owner_mask */
  int32_t tile;         /* elements per tile (the plan's tile) */
  int64_t total;        /* d */
  const void* owner_mask;          /* [d]; needed when any tile is mixed */
  const sdp_tile_desc* tiles;      /* CTA-major: CTA b runs tiles[b*tiles_per_cta ..] */
  int32_t n_tiles;
  int32_t tiles_per_cta;
  int32_t grid;                    /* CTAs; 0 = ceil(n_tiles / tiles_per_cta) */
  int32_t flags;
  void* replicas[SDP_MAX_WORKERS];     /* worker gradient buffers [d] (local or peer) */
  void* shadow_bf16[SDP_MAX_WORKERS];  /* per-worker bf16 copy of the mean, or NULL */
  void* out;            /* [d] mean (dtype), or NULL */
  void* out_bf16;       /* [d] bf16 mean, or NULL */
  /* fused Nesterov (SDP_SYNC_NESTEROV): theta/velocity [d] dtype, bf16 weights */
  void* theta;
  void* velocity;
  void* theta_bf16;
  double lr;
  double momentum;
  uint32_t* status;     /* device word, OR-ed with SDP_STATUS_* (may be NULL) */
  /* cross-GPU barrier (multi-process); world == 1 disables it */
  int32_t rank;
  int32_t world;
  uint32_t* signal_pads[8];  /* per-rank pad (peer-mapped), >= grid*8 words */
  uint32_t epoch;            /* increments every launch */
  uint32_t pad_;
  int64_t timeout_cycles;    /* spin limit per barrier */
  /* fused Adam (SDP_SYNC_ADAM, optim.py:90-109): `velocity` holds m, this v;
   * the host passes 1 - beta (as the reference computes it in float64) and
   * the bias corrections bias1 = 1 - beta1^t, bias2 = 1 - beta2^t. */
  void* second_moment;
  double beta1, beta2, one_minus_beta1, one_minus_beta2, bias1, bias2, eps;
  /* multi-GPU, optional: device-resident barrier epochs, one uint32 per CTA
   * (zeroed once).  When set, each CTA takes epoch = counter + 1 and stores
   * it back after its exit barrier, so the launch can be replayed from a
   * CUDA graph; `epoch` above is then ignored. */
  uint32_t* epoch_counters;
  /* compact owned-block storage, optional (SURVEY §7 hard part 7): worker w
   * keeps only the tiles whose owner union contains w; its replica / bf16
   * shadow of tile t starts at element slots[w * slot_stride + t] * tile of
   * its (compact) buffer, -1 = not stored.  NULL = every replica is the flat
   * [d] layout (tile t at t * tile).  These are the per-owner offsets of the
   * block descriptors: one int32 per (worker, tile). */
  const int32_t* slots;
  int64_t slot_stride;
  /* SDP_SYNC_LOCAL_UPDATE: CTA b applies the optimizer to
   * updates[b * updates_per_cta ...] (len 0 = hole) after its exit barrier --
   * exactly the tiles whose leader ran in CTA b on some rank, so the pairwise
   * per-CTA barrier already orders their write-back before the update. */
  const struct sdp_update_desc* updates;
  int32_t updates_per_cta;
  int32_t pad2_;
  const struct sdp_worker_state* states;  /* device array indexed by sdp_update_desc.state */
  /* fused Adam, optional: device-resident step (graph replay).  When
   * adam_step is set, the kernel reads t = *adam_step and takes the bias
   * corrections from adam_bias_table[2 * min(t, adam_table_len - 1) + {0, 1}]
   * (the host fills the table with 1 - beta^t exactly as the reference
   * computes it; past the last entry both are exactly 1.0), ignoring
   * bias1 / bias2 above. */
  const int32_t* adam_step;
  const double* adam_bias_table;
  int32_t adam_table_len;
  int32_t pad3_;
} sdp_sync_args;

/* One local worker's optimizer state, all in its compact storage layout. */
typedef struct sdp_worker_state {
  void* theta;          /* dtype, compact */
  void* velocity;       /* Nesterov v / Adam m */
  void* second_moment;  /* Adam v (NULL for Nesterov) */
  void* theta_bf16;     /* bf16 training copy, or NULL */
  const void* grad;     /* the worker's replica: holds the mean after the sync */
} sdp_worker_state;

/* One stored tile of one local worker: elements [slot*tile, slot*tile+len). */
typedef struct sdp_update_desc {
  uint32_t state;
  uint32_t slot;
  uint32_t len;
  uint32_t pad_;
} sdp_update_desc;

/* Launch the owner-subset sync.  For every element j with owner set O_j:
 *   acc = +0; for w in O_j ascending: acc += replicas[w][j];
 *   mean = acc / max(|O_j|, 1)            (IEEE division, no reciprocal)
 * then writes mean to out/out_bf16 and, with SDP_SYNC_WRITEBACK, to every
 * owner's replica and bf16 shadow.  Non-owner replica entries are never read
 * (except with CHECK_UNCOVERED at zero-coverage elements). */
int sdp_owner_sync(const sdp_sync_args* args /* host */, void* stream);

/* Fused-optimizer standalone (optim.py:78-84): v = mu v + g; th -= lr (g + mu v). */
int sdp_nesterov_update(int dtype, int64_t total, void* theta, void* velocity,
                        const void* grad, double lr, double momentum,
                        void* theta_bf16, uint32_t* status, void* stream);

/* Standalone optim.Adam.update (optim.py:101-109) on a flat vector, after the
 * caller's step counter was incremented to `step` (>= 1):
 *   m = b1 m + (1-b1) g;  v = b2 v + ((1-b2) g) g;
 *   th -= (lr (m / (1 - b1^step))) / (sqrt(v / (1 - b2^step)) + eps)
 * in numpy's evaluation order (f64: bit-identical); theta_bf16 optional. */
int sdp_adam_update(int dtype, int64_t total, void* theta, void* m, void* v, const void* grad,
                    double lr, double beta1, double beta2, double eps, int step,
                    void* theta_bf16, void* stream);

/* Finite check that runs BEFORE an optimizer update (optim.py:78-80 raises
 * NumericalError before touching theta): ORs SDP_STATUS_NONFINITE into
 * *status if any of x[0..total) is Inf or NaN. */
int sdp_check_finite(int dtype, int64_t total, const void* x, uint32_t* status, void* stream);

/* ------------------------------------------------------------------------ */
/* Extraction / write-back (models.py:333-382)                               */
/* ------------------------------------------------------------------------ */

/* out[j] = theta[j] * (bit w of owner_mask[j])  — models.py:355, bit-exact
 * (keeps -0.0 and NaN propagation of the multiply). */
int sdp_masked_extract(int dtype, const void* theta, const void* owner_mask,
                       int mask_bytes, int64_t total, int worker, void* out,
                       void* stream);

/* One parameter tensor of a width-wise subnetwork in canonical 3-D form: the
 * full tensor is viewed as [rows, cols, inner] (inner = the contiguous
 * trailing dims no slice governs), its compact sub-tensor as
 * [crows, ccols, inner]; rows and/or cols are selected through index maps
 * (masking.py:140-149 own slices = rows, consumer slices = cols):
 *   fwd_maps[row_map + r] = full row of compact row r          (gather)
 *   inv_maps[row_map + f] = compact row of full row f, or -1   (scatter)
 * and the same for columns; a map offset of -1 is the identity.  crows = 0
 * marks a tensor the worker does not hold (a dropped block).
 * inner_mul / inner_shr: fast division by inner, q = umulhi(n, mul) >> shr
 * (valid for n < 2^31; mul = 0, shr = 0 when inner == 1). */
typedef struct {
  int64_t full_offset;
  int64_t compact_offset;
  int32_t rows, cols, inner;
  int32_t crows, ccols;
  int32_t row_map, col_map;
  uint32_t inner_mul;
  uint32_t inner_shr;
  uint32_t rowlen_mul;  /* fast division by the row length the kernel walks: */
  uint32_t rowlen_shr;  /* ccols*inner (gather table), cols*inner (scatter) */
  int32_t col_tab;      /* offset in the map buffer of the expanded column table
                         * (one int32 per element of a walked row: the element's
                         * offset in the other side's row, -1 = not held), or -1
                         * for the identity; required when col_map >= 0 and the
                         * walked row has >= 256 elements */
} sdp_slice_desc;

/* A unit of work of the gather/scatter kernels: rows [row_begin, row_end) of
 * descriptor `desc` (compact rows for gather, full rows for scatter), and
 * within each of those rows the elements [elem_begin, elem_end).  Rows of
 * fewer than 256 elements must be whole (elem_begin = 0, elem_end = row length). */
typedef struct {
  int32_t desc;
  int32_t row_begin, row_end;
  int32_t elem_begin, elem_end;
  int32_t seg;      /* segment (worker) of a *_multi launch; ignored (0) otherwise */
  int32_t pad_[2];
} sdp_slice_task;

/* compact[...] = full[...] over every task (persistent CTAs walk the task list;
 * a tensor holds fewer than 2^31 elements).
 * flags & SDP_GATHER_REVERSE: full[...] = compact[...] through the same
 * forward maps (only mapped full elements are written) -- the inverse of a
 * gather whose descriptors tile the full tensor, e.g. leaving the
 * window-class-major sync layout.  dtype SDP_DTYPE_U8 moves owner masks,
 * SDP_DTYPE_U16 bf16 training copies (gathers are typeless copies). */
#define SDP_GATHER_REVERSE 0x1
#define SDP_DTYPE_U8 2
#define SDP_DTYPE_U16 3  /* 2-byte elements moved as bits (bf16 training copies) */
int sdp_gather_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                      int n_tasks, const int32_t* fwd_maps, const void* full,
                      void* compact, int flags, void* stream);

/* Several workers' slices in ONE launch: task `seg` selects the segment's
 * (full, compact) base pointers from this host-side table (copied into the
 * kernel's parameters).  The descriptor / task / map tables are the
 * per-worker tables concatenated (models.SliceBatch).  A compact pointer may
 * be NULL in a scatter segment only if that segment has no tasks. */
typedef struct {
  const void* full[SDP_MAX_WORKERS];
  const void* compact[SDP_MAX_WORKERS];
  int32_t n;
} sdp_slice_segs;
int sdp_gather_slices_multi(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                            int n_tasks, const int32_t* fwd_maps, const sdp_slice_segs* segs,
                            int flags, void* stream);

#define SDP_SCATTER_ZERO_FILL 0x1  /* full[j] = 0 where no compact element maps */
#define SDP_SCATTER_ACCUMULATE 0x2 /* full[j] += compact[...] instead of = */

/* Write compact grads back into the flat layout (models.py:376-381): tasks
 * cover FULL rows (coalesced stores, every covered full element written once
 * in ZERO_FILL mode; in ACCUMULATE mode only mapped elements are touched). */
int sdp_scatter_slices(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                       int n_tasks, const int32_t* inv_maps, const void* compact, void* full,
                       int flags, void* stream);
int sdp_scatter_slices_multi(int dtype, const sdp_slice_desc* descs, const sdp_slice_task* tasks,
                             int n_tasks, const int32_t* inv_maps, const sdp_slice_segs* segs,
                             int flags, void* stream);

/* out[j] = acc[j] / divisor[j] in dtype (the engine.py:74 divide after an
 * owner-ordered scatter-accumulate).  divisor is float64 [d]. */
int sdp_divide(int dtype, const void* acc, const double* divisor, int64_t total,
               void* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Channels-last GroupNorm (+ReLU) over contiguous ragged channel groups      */
/* (the active-channel GroupNorm of compact subnetworks, ops.py:140-204)      */
/* ------------------------------------------------------------------------ */

#define SDP_GN_RELU 0x1             /* y = relu(groupnorm(x)) */
#define SDP_GN_GROUPS_ALIGNED8 0x2  /* every group start is a multiple of 8: 16-B vectors */
#define SDP_GN_AFFINE_BF16 0x4      /* gamma / beta are bf16 (else fp32) */

/* x, y: bf16 [batch, hw, channels] (channels_last); group g = channels
 * [group_starts[g], group_starts[g+1]) (device int32 [groups + 1]); gamma,
 * beta fp32 [channels]; mean / rstd fp32 [batch * groups] (out).
 * y = relu?((x - mean) * rstd * gamma + beta), statistics in fp32.
 * flags: SDP_GN_RELU | SDP_GN_GROUPS_ALIGNED8 (the caller's promise about
 * group_starts; the library checks channels and pointer alignment). */
int sdp_group_norm_fwd(const void* x_bf16, int batch, int hw, int channels, const int32_t* group_starts,
                       int groups, int max_group_channels, const void* gamma, const void* beta, float eps,
                       int flags, void* y_bf16, float* mean, float* rstd, void* stream);

/* Backward of sdp_group_norm_fwd: dx (bf16, same layout) and dgamma / dbeta
 * [channels] WRITTEN in the affine dtype (SDP_GN_AFFINE_BF16: bf16, else
 * fp32).  Deterministic: every CTA writes one partial row of fp32 dgamma /
 * dbeta sums into `scratch` (no zeroing needed) and a second launch folds the
 * rows in a fixed order -- no floating-point atomics, so repeated calls are
 * bit-identical.  `scratch` holds at least sdp_group_norm_bwd_scratch(...)
 * floats; calls sharing a scratch must be ordered (one stream).  batch > 0. */
int sdp_group_norm_bwd_scratch(int batch, int hw, int channels, int max_group_channels, long long* floats);
int sdp_group_norm_bwd(const void* x_bf16, const void* y_bf16, const void* dy_bf16, int batch, int hw,
                       int channels, const int32_t* group_starts, int groups, int max_group_channels,
                       const void* gamma, const float* mean, const float* rstd, int flags, void* dx_bf16,
                       void* dgamma, void* dbeta, float* scratch, long long scratch_floats, void* stream);

/* Row LayerNorm on bf16 [rows, cols] activations, cols a multiple of 256 (up
 * to 2048 forward, 1024 backward): the GPT-2 blocks of the C4 training step
 * (train._layer_norm).  Forward saves fp32 mean / rstd per row.  Backward
 * writes dx and the bf16 dgamma / dbeta; `scratch` holds 2 x cols x parts
 * floats, parts = sdp_layer_norm_bwd_parts(rows, cols) (per-CTA partial sums folded
 * in CTA order: deterministic). */
int sdp_layer_norm_fwd(const void* x_bf16, int64_t rows, int cols, const void* gamma_bf16,
                       const void* beta_bf16, float eps, void* y_bf16, float* mean, float* rstd, void* stream);
int sdp_layer_norm_bwd_parts(int64_t rows, int cols);
int sdp_layer_norm_bwd(const void* dy_bf16, const void* x_bf16, int64_t rows, int cols, const void* gamma_bf16,
                       const float* mean, const float* rstd, void* dx_bf16, void* dgamma_bf16, void* dbeta_bf16,
                       float* scratch, int parts, void* stream);
/* Residual-fused forms (GPT-2 blocks): the forward normalises
 * sum = bf16(a + b) and also writes `sum` (the residual stream); the
 * backward adds the residual branch's gradient `dres` into dx. */
int sdp_add_layer_norm_fwd(const void* a_bf16, const void* b_bf16, int64_t rows, int cols, const void* gamma_bf16,
                           const void* beta_bf16, float eps, void* sum_bf16, void* y_bf16, float* mean, float* rstd,
                           void* stream);
int sdp_layer_norm_bwd_res(const void* dy_bf16, const void* x_bf16, const void* dres_bf16, int64_t rows, int cols,
                           const void* gamma_bf16, const float* mean, const float* rstd, void* dx_bf16,
                           void* dgamma_bf16, void* dbeta_bf16, float* scratch, int parts, void* stream);

/* Attention-head gradient merge (train._SplitHeads backward): dq, dk, dv
 * [batch, heads, seq, head_dim] with element strides (stride_batch,
 * stride_head, stride_seq) shared by the three and contiguous head rows ->
 * out [batch, seq, 3, heads, head_dim], the fused qkv projection's gradient.
 * elem_bytes 2 or 4. */
int sdp_merge_heads(const void* dq, const void* dk, const void* dv, int64_t batch, int64_t seq, int heads,
                    int head_dim, int elem_bytes, int64_t stride_batch, int64_t stride_head, int64_t stride_seq,
                    void* out, void* stream);

/* Convolution-weight gradients, channels-last bf16 -> reference-layout fp32
 * (train.SubnetTrainer._store_grads): for each descriptor, the weight at
 * element `offset` of both buffers is [out, kernel_elems, in] (OHWI) in
 * `src_bf16` and is written [out, in, kernel_elems] (OIHW) into `dst`.
 * in_channels * kernel_elems <= sdp_conv_grad_max_block(). */
typedef struct {
  int64_t offset;
  int32_t out_channels;
  int32_t in_channels;
  int32_t kernel_elems;
  int32_t pad_;
} sdp_conv_grad_desc;

int sdp_conv_grads_to_oihw(const sdp_conv_grad_desc* descs, int n_desc, int max_out_channels, const void* src_bf16,
                           float* dst, void* stream);
int sdp_conv_grad_max_block(void);
/* The reverse direction for the training copy: bf16 OIHW -> bf16 OHWI
 * (channels-last) for every descriptor, same table layout. */
int sdp_conv_weights_to_ohwi(const sdp_conv_grad_desc* descs, int n_desc, int max_out_channels, const void* src_bf16,
                             void* dst_bf16, void* stream);

/* Column sums of a bf16 [rows, cols] matrix into bf16 [cols] with fp32
 * accumulation (GPT-2 projection bias gradients, train._Linear); cols a
 * multiple of 8, x 16-B aligned; `scratch` holds cols x sdp_col_sum_parts()
 * floats; deterministic (parts folded in order). */
int sdp_col_sum_parts(void);
int sdp_col_sum_bf16(const void* x_bf16, int64_t rows, int cols, void* out_bf16, float* scratch, void* stream);

/* ------------------------------------------------------------------------ */
/* Fused LM-head cross-entropy rows (C4 training step, train.lm_loss)        */
/* ------------------------------------------------------------------------ */

/* For each row r of a bf16 [rows, pitch] logits chunk (columns >= vocab are
 * padding and ignored):
 *   lse[r] = log sum_{j<vocab} exp(logit[r, j]),  loss_rows[r] = lse[r] - logit[r, targets[r]]
 * (fp32 accumulation, one pass). */
int sdp_ce_rows_fwd(const void* logits_bf16, int64_t rows, int vocab, int64_t pitch, const int64_t* targets,
                    float* lse, float* loss_rows, void* stream);

/* dlogits = bf16((exp(logit - lse[r]) - [j == targets[r]]) * grad_out[0] * inv_n)
 * for j < vocab and 0 in the padding columns: the gradient of mean
 * cross-entropy w.r.t. the chunk's logits; grad_out is a device scalar (no
 * host sync, CUDA-graph capturable).  16-B aligned buffers. */
int sdp_ce_rows_bwd(const void* logits_bf16, int64_t rows, int vocab, int64_t pitch, const int64_t* targets,
                    const float* lse, const float* grad_out, float inv_n, void* dlogits_bf16,
                    void* stream);

/* ------------------------------------------------------------------------ */
/* Gradient-alignment diagnostic (diagnostics.py:33-78)                      */
/* ------------------------------------------------------------------------ */

/* A chunk [offset, offset + length) of segment `segment` (one layer's slice). */
typedef struct {
  int64_t offset;
  int64_t length;
  int32_t segment;
  int32_t pad_;
} sdp_reduce_task;

/* Per segment s: out[4s..4s+3] = (sum a*b, sum a*a, sum b*b, count) over the
 * elements with support[j] != 0 (support = NULL: all), accumulated in float64.
 * partials: [n_tasks * 4] float64 scratch.  Deterministic (fixed-order
 * second pass, no float atomics).  The restricted cosine is
 * ab / (sqrt(aa) * sqrt(bb)) (diagnostics.py:43-47). */
int sdp_restricted_dots(int dtype, const void* a, const void* b, const uint8_t* support,
                        const sdp_reduce_task* tasks, int n_tasks, int n_segments,
                        double* partials, double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Cross-process peer mapping (multi-GPU owner sync)                         */
/* ------------------------------------------------------------------------ */

#define SDP_IPC_HANDLE_BYTES 64

/* Export `ptr` (inside any cudaMalloc allocation): handle + byte offset of
 * ptr from the allocation base. */
int sdp_ipc_export(const void* ptr, uint8_t* handle_out /* host, 64 B */,
                   uint64_t* offset_out /* host */);
/* Map a peer's export into this process; *ptr_out = base + offset. */
int sdp_ipc_import(const uint8_t* handle /* host */, uint64_t offset,
                   void** ptr_out /* host */);
int sdp_ipc_close(void* ptr);
/* Enable direct peer access from the current device to `peer` (idempotent). */
int sdp_enable_peer(int peer);

/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault) on `stream`: the peer
 * copy probe bench.py runs at start-up for the measured NVLink peak (SURVEY
 * §8d), with dst a peer-mapped (sdp_ipc_import) address. */
int sdp_copy_async(void* dst, const void* src, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SDP_H_ */
