/*
 * mpo.h -- C ABI of the residual-compensated 16-bit optimizer step (arXiv 2309.12381,
 * "16-bit-only mixed precision"), B200 / sm_100a.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n (the section is named alongside),
 * "R<k>" = a reading of a paper-silent point, listed in DESIGN.md section 3.
 *
 * What the library computes (sec. "16bits only Mixed-Precision"): every parameter is
 * held as a 16-bit value (fp16 or bf16; "the 16bits value used in the computations")
 * plus a 16-bit residual ("storing only the difference between the two formats").  An
 * operation reconstructs the fp32 weight from value + residual, "performs the operation in
 * full precision using the extra bits saved separately and outputs both the updated 16 bits
 * float and its extra bits".  The operations are the "classic optimizers (Adam and
 * SGD)", applied either to all parameters "as one only stream of values" (the
 * fused / multi-tensor form), or per parameter from inside backward, or (not in the
 * paper; BASELINE.json north_star (c)) to one shard of a flat parameter buffer per GPU.
 *
 * Representation (readings R1-R5):
 *   value    = IEEE-754 round-to-nearest-even of the fp32 weight x to fp16 / bf16 (R2);
 *              NaN -> 0x7FFF (R4); overflow -> +-Inf (IEEE).
 *   residual = int16, sat16( bits32(x) - bits32(widen(value)) ), the signed difference of the
 *              two binary32 bit patterns (R1), saturated to [-32768, 32767] (R3); 0 for NaN/Inf.
 *   reconstruct(value, residual) = f32( bits32(widen(value)) + residual ); NaN -> 0x7FFFFFFF.
 *   This is lossless for bf16 except on the 32 640 RNE upper-tie patterns (1 ulp32 low, R3),
 *   and for fp16 on 2^-16 <= |x| < 65520 (R5).
 *
 * Conventions shared by every entry point:
 *   * All array arguments are DEVICE pointers to caller-owned memory (e.g. torch tensors).
 *     The library keeps no reference after return and allocates nothing persistent.
 *   * Every array base pointer must be 16-byte aligned (MPO_EALIGN otherwise); lengths are
 *     arbitrary (ragged tails are handled element by element).  Arrays must not alias.
 *   * Calls are ASYNCHRONOUS: they validate, enqueue kernels (and NCCL collectives) on
 *     `stream` and return.  Asynchronous device faults surface at the caller's next sync.
 *   * In place on value / residual / optimizer state; gradients are read-only, except that
 *     mpo_sharded_step reduce-scatters into its grad_flat argument.
 *   * Hyper-parameters arrive as doubles.  The library derives every kernel scalar on the host
 *     in double and rounds it ONCE to float (R7); the device never calls pow().
 *   * Errors are status codes; nothing aborts or throws across the ABI.  mpo_last_error()
 *     returns a thread-local message describing the last non-OK status (validation errors in
 *     a tensor table name the offending table index).  NaN/Inf in gradients is NOT an error:
 *     it propagates into the weights (training-divergence signal left to the caller).
 *
 * Two builds of the same sources are shipped: libmpo_exact.so (-fmad=false, bit-exact to the
 * CPU oracle for every entry point; the build the Python binding, the optimizers and bench.py use by
 * default) and libmpo.so (FMA contraction; within DESIGN.md R12's tolerance, 0.5-1 % faster).
 */
#ifndef MPO_H
#define MPO_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The stream is a cudaStream_t; declared opaque so this header needs no CUDA include. */
typedef void* mpo_stream;

typedef enum {
    MPO_OK = 0,
    MPO_EINVAL = 1,   /* bad enum, negative size, non-finite hyper-parameter, bad sharding */
    MPO_EALIGN = 2,   /* an array base pointer is not 16-byte aligned                      */
    MPO_EDTYPE = 3,   /* value dtype not FP16/BF16, or unsupported grad dtype              */
    MPO_ECUDA = 4,    /* kernel launch failed (cudaGetLastError)                            */
    MPO_ENCCL = 5     /* an NCCL call failed (message from ncclGetErrorString)              */
} mpo_status;

/* Value storage formats and gradient dtypes.  A storage format names the 16-bit value dtype and
 * the scheme of its residual (code = base | scheme << 4):
 *   MPO_FP16, MPO_BF16       RNE value + int16 signed difference (R1-R5; the default)
 *   MPO_FP16_RTZ, _BF16_RTZ  round-to-zero value + uint16 extra bits ("saving only the first
 *                            part of the 32bit significand is equivalent to applying a
 *                            round-to-zero"); bf16 is lossless on every finite fp32 value
 *   MPO_FP16_SR              stochastic rounding + int16 signed difference whose sign is the
 *                            paper's "un-round" bit ("fp16 + 13 stochastic"); draws
 *                            from the counter-based generator keyed by (seed, sr_stream, index/2),
 *                            upper 32 bits for even, lower for odd elements (R14)
 *   MPO_FP16_X8, _BF16_X8    RNE value + 8 extra bits: int8 residual ("keeping only part of
 *                            those bits"; P:134 fp16+8), reading R14
 *   MPO_FP16_X8Z, _BF16_X8Z  the paper's own fp16+8 / bf16+8: round-to-zero value + the next 8
 *                            significand bits, truncated: uint8 residual, R20
 * Gradients: MPO_FP16, MPO_BF16 or MPO_FP32 (variant formats: their base dtype or MPO_FP32). */
typedef enum {
    MPO_FP16 = 0, MPO_BF16 = 1, MPO_FP32 = 2,
    MPO_FP16_RTZ = 16, MPO_BF16_RTZ = 17, MPO_FP16_SR = 32, MPO_FP16_X8 = 48, MPO_BF16_X8 = 49,
    MPO_FP16_X8Z = 64, MPO_BF16_X8Z = 65
} mpo_dtype;
typedef enum { MPO_SGD = 0, MPO_ADAM = 1 } mpo_optim;

/* One parameter tensor of a multi-tensor table ("one only stream of values").
 *   value     : n 16-bit values (storage format vdt), updated in place
 *   resid     : n residuals, updated in place: int16 (MPO_FP16/BF16, FP16_SR), uint16 bit
 *               patterns (the RTZ formats), int8 (the X8 formats) or uint8 (X8Z)
 *   grad      : n gradients (dtype gdt: FP16, BF16 or FP32), read-only
 *   m         : n fp32 -- SGD momentum buffer, or Adam first moment (NULL for SGD w/o momentum)
 *   v         : n fp32 -- Adam second moment (ignored by SGD)
 *   n         : element count (>= 0)
 *   hp        : index into the hyper-parameter group array of the call
 *   sr_stream : stream id of the stochastic-rounding draws of this tensor (0 <= id < 2^27;
 *               ignored by deterministic formats)                                          */
typedef struct {
    void* value;
    void* resid;
    const void* grad;
    float* m;
    float* v;
    int64_t n;
    int32_t hp;
    int32_t sr_stream;
} mpo_tensor;

/* torch.optim.SGD semantics (R6; "classic optimizers"; P:19 drop-in hyper-parameters).
 * grad_scale multiplies the incoming gradient first (loss-scale unscale, 1/N data-parallel
 * mean; "every operations on the gradient (eg. clipping or scaling) has to be done
 * through the optimizer").  first_step != 0: the momentum buffer is initialised to the
 * gradient (torch's clone on the first step) and is not read. */
typedef struct {
    double lr, momentum, dampening, weight_decay, grad_scale;
    int32_t nesterov, first_step;
    uint64_t seed;   /* stochastic-rounding draws of this step (MPO_FP16_SR); else ignored */
    double clip_value;       /* > 0: clamp the scaled gradient to [-c, c] (see below); 0: off */
    int32_t skip_nonfinite;  /* != 0: skip the update when a scaled gradient is Inf/NaN (below) */
    int32_t norm_ready;      /* != 0: norm_ws[0] already holds S of the whole step (below) */
} mpo_sgd_hp;

/* torch.optim.Adam / AdamW semantics (R6).  step is 1-based (bias correction).  adamw != 0:
 * decoupled decay w *= (1 - lr*weight_decay); else L2 (g += weight_decay*w).
 * max_grad_norm > 0 enables global-norm clipping (R9; multi-tensor and sharded modes only,
 * P:93 "prohibits any operation that would require every gradients of the model at the same
 * time"); the same value must then be given to every group of the call. */
typedef struct {
    double lr, beta1, beta2, eps, weight_decay, grad_scale, max_grad_norm;
    int32_t adamw, _pad;
    int64_t step;
    uint64_t seed;   /* stochastic-rounding draws of this step (MPO_FP16_SR); else ignored */
    double clip_value;       /* > 0: clamp the scaled gradient to [-c, c] (see below); 0: off */
    int32_t skip_nonfinite;  /* != 0: skip the update when a scaled gradient is Inf/NaN (below) */
    int32_t norm_ready;      /* != 0: norm_ws[0] already holds S of the whole step (below) */
} mpo_adam_hp;

/* Gradient surgery inside the optimizer ("every operations on the gradient (eg. clipping or
 * scaling) has to be done through the optimizer"; "perform the clipping through a
 * parameter hook ... The same applies to loss scaling"):
 *   grad_scale      multiplies first (loss-scale unscale; 1/N data-parallel mean);
 *   clip_value      then clamps to [-c, c] like torch.clamp (NaN stays NaN), in every mode;
 *                   exclusive with max_grad_norm;
 *   skip_nonfinite  loss-scaling "found inf": the fp64 sum of squares S of the scaled grads is
 *                   computed first (needs norm_ws) and the update is skipped -- nothing written --
 *                   when S is not finite.  Multi-tensor and sharded modes skip the whole call
 *                   (sharded: S all-reduced, all ranks agree); the hook mode can only skip the
 *                   one parameter (earlier parameters of the same backward were already stepped,
 *                   P:93) and accumulates S into norm_ws[mpo_norm_ws_doubles() - 1] so the
 *                   caller learns at the end of backward whether any gradient was non-finite.
 * Must be the same for every group of a call. */

/* norm_ready (multi-tensor entry points only): a step whose parameters span several tables (e.g.
 * tensors of different gradient dtypes, one mpo_adam_step call each) needs ONE S over all of them
 * for global-norm clipping (R9: "the norm of all gradients") and for an all-or-nothing
 * found-inf skip.  The caller then fills norm_ws[0] with mpo_grad_sumsq over every table first
 * (accumulate = 0 for the first, 1 for the rest) and sets norm_ready in every group of every step
 * call: the calls do no pre-pass and read S from norm_ws[0].  Rejected (MPO_EINVAL) by the hook and
 * sharded entry points, which compute their own S. */

/* Largest number of hyper-parameter groups one call may carry. */
#define MPO_MAX_HP_GROUPS 16

/* Split fp32 weights into (16-bit value, residual) (readings R1-R5, R14).
 *   vdt   : a storage format (see mpo_dtype)
 *   w     : n fp32 (device, read-only);  value: n 16-bit (device, written);
 *   resid : n residuals of the format's type (device, written)
 *   seed, sr_stream : key of the stochastic-rounding draws (MPO_FP16_SR; ignored otherwise) */
mpo_status mpo_split(mpo_dtype vdt, const float* w, void* value, void* resid, int64_t n,
                     uint64_t seed, int32_t sr_stream, mpo_stream stream);

/* Reconstruct the fp32 weights from value + residual ("performs the operation in full
 * precision using the extra bits saved separately").  value/resid read-only, w written. */
mpo_status mpo_reconstruct(mpo_dtype vdt, const void* value, const void* resid, float* w,
                           int64_t n, mpo_stream stream);

/* Residual-compensated SGD(-momentum) step over a table of nt tensors, one fused launch per
 * table slice.  hp: nhp groups (1 <= nhp <= MPO_MAX_HP_GROUPS) in HOST memory;
 * t: nt entries in HOST memory (copied into the launch; not retained). */
mpo_status mpo_sgd_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt,
                        const mpo_sgd_hp* hp, int32_t nhp, double* norm_ws, mpo_stream stream);

/* Residual-compensated Adam/AdamW step over a table of nt tensors.
 * norm_ws: DEVICE scratch of at least mpo_norm_ws_doubles() doubles, required iff
 * max_grad_norm > 0 (global-norm clipping: fp64 sum of squares of the scaled gradients over
 * the whole table, coef = min(1, max_norm / (sqrt(S) + 1e-6)), R9) or skip_nonfinite.  On
 * return (stream order) norm_ws[0] holds S.  mpo_sgd_step takes the same workspace (needed iff
 * skip_nonfinite). */
mpo_status mpo_adam_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt,
                         const mpo_adam_hp* hp, int32_t nhp, double* norm_ws,
                         mpo_stream stream);

/* Doubles of device scratch the norm pre-pass needs (clipping, skip_nonfinite): [0] = S of the
 * call, then per-block partials, last = S accumulated by hook-mode calls (zeroed by the caller). */
int64_t mpo_norm_ws_doubles(void);

/* Sum of squares of the scaled gradients of a table: S = sum_i (double)(f32(grad_i) * gs)^2 with
 * gs = (float)grad_scale[t.hp] (R9; the pre-pass of clipping and of the found-inf skip, exposed so a
 * step spanning several tables shares one S -- see norm_ready).  Only the grad, n and hp fields of
 * the table entries are read (grad 16-B aligned; value/resid/m/v ignored).
 *   gdt        : MPO_FP16 | MPO_BF16 | MPO_FP32
 *   grad_scale : nhp doubles (HOST), 1 <= nhp <= MPO_MAX_HP_GROUPS, finite
 *   norm_ws    : DEVICE scratch of mpo_norm_ws_doubles() doubles; accumulate == 0: norm_ws[0] = S,
 *                else norm_ws[0] += S (stream order).  The partials in norm_ws[1..] are clobbered. */
mpo_status mpo_grad_sumsq(mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const double* grad_scale,
                          int32_t nhp, double* norm_ws, int32_t accumulate, mpo_stream stream);

/* A step that can be captured ONCE in a CUDA graph and replayed every step (whole-iteration graph
 * capture, "CUDA graphs instead of a tracing compiler"): the per-step derived hyper-parameters --
 * bias corrections (step), lr, betas, eps, weight decay, SGD's first step, the stochastic-rounding
 * seed -- are not kernel arguments but a block that the call copies from host_block to dev_block
 * in stream order before the kernels read it.  A graph that captured the call repeats that copy at
 * every replay, reading host_block's CURRENT contents, so the caller refills host_block with
 * mpo_hp_block_fill (a host function, no CUDA call) before each replay.
 *   kind, vdt, gdt, t, nt, norm_ws : as mpo_sgd_step / mpo_adam_step (the table -- pointers, sizes,
 *               groups -- is fixed at capture)
 *   hp, nhp   : HOST hyper-parameters used for validation and the step's static parts: the kernel
 *               choice, max_grad_norm, skip_nonfinite and the norm pre-pass's grad scales
 *   host_block: mpo_hp_block_bytes(kind) bytes of PAGE-LOCKED host memory (cudaHostAlloc / torch
 *               pin_memory), filled by mpo_hp_block_fill
 *   dev_block : mpo_hp_block_bytes(kind) bytes of device memory, 16-B aligned (owned by the caller)
 *   ack       : NULL, or a page-locked host word the device writes the block's sequence number to
 *               right after the copy: a caller that reads back the sequence number it wrote may
 *               refill host_block for the next replay without racing this one's copy
 * Bit-identical to the corresponding mpo_sgd_step / mpo_adam_step with the same hp. */
int64_t mpo_hp_block_bytes(mpo_optim kind);
/* Derive the kernel's per-group scalars from nhp hyper-parameter groups (host memory, R7: in double,
 * rounded once to float) into host_block (mpo_hp_block_bytes(kind) bytes) and tag it with `seq`.
 * No CUDA call. */
mpo_status mpo_hp_block_fill(mpo_optim kind, const void* hp, int32_t nhp, uint64_t seq, void* host_block);
mpo_status mpo_step_graphed(mpo_optim kind, mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt,
                            const void* hp, int32_t nhp, const void* host_block, void* dev_block,
                            unsigned long long* ack, double* norm_ws, mpo_stream stream);

/* Fused backward + optimizer step for ONE parameter, called from its post-accumulate-grad hook
 * ("operate the optimization step as soon as the gradient is computed").
 *   kind : MPO_SGD (hp -> mpo_sgd_hp) | MPO_ADAM (hp -> mpo_adam_hp), hp in HOST memory
 *   one  : the parameter's table entry (its hp field is ignored)
 *   norm_ws : device workspace, required iff skip_nonfinite (see "Gradient surgery")
 * Global operations are impossible here: MPO_EINVAL if max_grad_norm > 0.
 * The caller frees the gradient right after the call; stream order makes that safe. */
mpo_status mpo_fused_backward_hook_step(mpo_optim kind, mpo_dtype vdt, mpo_dtype gdt,
                                        const mpo_tensor* one, const void* hp, double* norm_ws,
                                        mpo_stream stream);

/* Data-parallel sharded step (not in the paper, which lists distribution as future work,
 * P:196; BASELINE.json north_star (c)).  Collective: every rank calls it with the same
 * arguments except rank and its own buffers.
 *   nccl_comm   : an ncclComm_t (borrowed, e.g. from torch's ProcessGroupNCCL; never freed)
 *   value_flat  : n_total 16-bit values, replicated on every rank (all-gathered on return)
 *   grad_flat   : n_total 16-bit gradients of THIS rank (the value format's base dtype);
 *                 overwritten:
 *                 shard `rank` becomes the reduced (summed) gradient
 *   resid_shard, m_shard, v_shard : n_total/world entries of this rank's shard (v ignored,
 *                 m may be NULL, for SGD without momentum)
 *   n_total     : multiple of 8*world
 *   hp          : mpo_sgd_hp* | mpo_adam_hp* (HOST); grad_scale should be 1/world for a mean
 *   norm_ws     : as for mpo_adam_step (clipping: the shard sums are all-reduced in fp64)
 * Sequence on `stream`: ncclReduceScatter(sum) -> [sumsq + ncclAllReduce] -> step on the shard
 * -> ncclAllGather of the 16-bit values only (in place; at world 1 NCCL's single-rank path makes
 * them no-ops, but they are still issued).  The shard's stochastic-rounding stream is its rank. */
mpo_status mpo_sharded_step(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world,
                            mpo_dtype vdt, void* value_flat, void* grad_flat,
                            void* resid_shard, float* m_shard, float* v_shard,
                            int64_t n_total, const void* hp, double* norm_ws,
                            mpo_stream stream);

/* One piece of a rank's shard for mpo_sharded_step_grouped: the elements [start, next start) of the
 * shard (the last piece runs to the shard's end) use hyper-parameter group `hp` and draw their
 * stochastic-rounding numbers from stream `sr_stream` (0 <= id < 2^27), indexed from the piece's
 * first element. */
typedef struct {
    int64_t start;
    int32_t hp;
    int32_t sr_stream;
} mpo_segment;

/* mpo_sharded_step with per-parameter hyper-parameter groups ("does not necessitate any
 * alterations to the hyperparameters": e.g. GPT/LLaMA recipes that exempt 1-D tensors from weight
 * decay).  Same collective sequence and arguments as mpo_sharded_step, plus:
 *   seg, nseg : HOST array partitioning THIS rank's shard [0, n_total/world) into pieces (seg[0].start
 *               == 0, starts strictly increasing and < the shard length; every start a multiple of 8
 *               elements, 16 for the 8-bit-residual formats (X8, X8Z), so each piece's arrays stay 16-B aligned); ranks
 *               pass their own tables
 *   hp, nhp   : nhp groups (mpo_sgd_hp* | mpo_adam_hp*, HOST), 1 <= nhp <= MPO_MAX_HP_GROUPS;
 *               grad_scale, max_grad_norm, clip_value and skip_nonfinite as for a multi-tensor call
 * mpo_sharded_step(..) == this call with one segment {0, 0, rank} and one group. */
mpo_status mpo_sharded_step_grouped(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world,
                                    mpo_dtype vdt, void* value_flat, void* grad_flat,
                                    void* resid_shard, float* m_shard, float* v_shard,
                                    int64_t n_total, const mpo_segment* seg, int32_t nseg,
                                    const void* hp, int32_t nhp, double* norm_ws, mpo_stream stream);

/* Polls an NCCL communicator for an asynchronous error (ncclCommGetAsyncError): MPO_OK while it is
 * healthy or still initialising, MPO_ENCCL (message: ncclGetErrorString + ncclGetLastError) once a
 * collective on it failed -- e.g. a peer died or the network reported an error.  The sharded entry
 * points check it before issuing collectives, so a failed communicator is reported instead of
 * hanging; a training loop can poll it between steps.  Never blocks. */
mpo_status mpo_comm_check(uintptr_t nccl_comm);

/* The sharded step fused with its collectives over NVLink SHARP: one kernel
 * per rank reads the SUM over all ranks of its shard's 16-bit gradients with multimem.ld_reduce
 * (fp32 accumulation in the switch, one rounding to 16 bits), updates value/residual/state like
 * mpo_sharded_step, and multicasts the new 16-bit values to every rank's replica with
 * multimem.st -- no reduce-scatter / all-gather launches and no reduced-gradient buffer.
 *   value_mc, grad_mc : multicast addresses of the replicated n_total-element value buffer and
 *                       of the per-rank gradient buffers (a multicast object every rank bound)
 *   value_uc          : this rank's unicast address of its value replica (read)
 *   resid_shard, m_shard, v_shard : this rank's shard state (n_total/world entries)
 *   vdt               : any storage format (mpo_dtype); grads of its base 16-bit dtype;
 *                       stochastic-rounding draws: stream = rank, index inside the shard
 *   hp                : mpo_sgd_hp* | mpo_adam_hp*; grad_scale 1/world for a mean; no global-norm
 *                       clipping and no skip_nonfinite (no pre-pass); clip_value allowed
 * The caller orders the call after every rank finished writing its gradients and before any
 * rank reads the values again (cross-rank barriers); the kernel ends with fence.proxy.alias +
 * fence.acq_rel.sys. */
mpo_status mpo_nvls_sharded_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt,
                                 void* value_mc, const void* value_uc, const void* grad_mc,
                                 void* resid_shard, float* m_shard, float* v_shard,
                                 int64_t n_total, const void* hp, mpo_stream stream);

/* Validation entry point of the NVLS kernel on a box without a multicast object (one GPU):
 * the SAME kernel as mpo_nvls_sharded_step (indexing, state streams, update, re-split, fences),
 * with its two multicast operations performed over ordinary peer pointers instead --
 *   multimem.ld_reduce.add.acc::f32  ->  the ranks' 8 gradients summed in fp32 in rank order
 *                                         and rounded once to the 16-bit format (RNE; NaN ->
 *                                         0x7FFF), equal to the switch's result whenever the
 *                                         fp32 sum is order-independent (exact-sum inputs);
 *   multimem.st                      ->  a store into every rank's replica.
 * Arguments as mpo_p2p_sharded_step (value_peers / grad_peers: HOST arrays of `world` device
 * pointers, value_peers[rank] is the replica read), constraints as mpo_nvls_sharded_step
 * (any storage format, grads of its base dtype, no pre-pass); 1 <= world <= 8.
 * Not a product path: the multi-GPU path is mpo_nvls_sharded_step on a real multicast object. */
mpo_status mpo_nvls_emulated_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt,
                                  void* const* value_peers, const void* const* grad_peers,
                                  void* resid_shard, float* m_shard, float* v_shard,
                                  int64_t n_total, const void* hp, mpo_stream stream);

/* The sharded step fused with its collectives over NVLink peer memory (the
 * P2P form; needs no multicast object): one kernel per rank that, for each 8-element unit of its
 * shard [rank*S, (rank+1)*S), S = n_total/world,
 *   1. loads the 16-bit gradients of EVERY rank from grad_peers[k] (NVLink P2P loads) and sums
 *      them in fp32 in rank order, ((g_0 + g_1) + g_2) + ... (deterministic; R15),
 *   2. reconstructs, updates and re-splits exactly like mpo_sharded_step's shard update, the
 *      sum entering as an fp32 gradient (times grad_scale: 1/world for a mean),
 *   3. stores the new 16-bit values into EVERY rank's replica value_peers[k] (P2P stores);
 *      residual / m / v stay local.
 * It replaces reduce-scatter + update + all-gather by one launch with no reduced-gradient
 * buffer; the NVLink traffic per rank equals RS + AG (2 B * S * (world-1) each way).
 *   value_peers, grad_peers : HOST arrays of `world` device pointers (16-B aligned) to every
 *                 rank's n_total-element value replica and 16-bit gradient buffer, mapped into
 *                 this process (CUDA IPC, torch symmetric memory, or, for tests, buffers of the
 *                 same device); value_peers[rank] / grad_peers[rank] are this rank's own
 *   resid_shard, m_shard, v_shard : this rank's shard state (S entries; m NULL for SGD without
 *                 momentum; v ignored for SGD)
 *   vdt         : any storage format; gradients are its base 16-bit dtype
 *   world       : 1 .. 8;  n_total : multiple of 8*world
 *   hp          : mpo_sgd_hp* | mpo_adam_hp* (HOST); no global-norm clipping, no
 *                 skip_nonfinite (no pre-pass: MPO_EINVAL); clip_value allowed
 * Stochastic-rounding draws: stream = rank, index inside the shard (as mpo_sharded_step).
 * The caller orders the call after every rank finished writing its gradients and before any
 * rank reads values or overwrites gradients again (cross-rank barriers); the kernel ends with
 * fence.acq_rel.sys. */
mpo_status mpo_p2p_sharded_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt,
                                void* const* value_peers, const void* const* grad_peers,
                                void* resid_shard, float* m_shard, float* v_shard,
                                int64_t n_total, const void* hp, mpo_stream stream);

/* A single-device multicast object bound to fresh device memory (cuMulticastCreate /
 * cuMulticastBindMem), for running the NVLS step at world 1 and in tests.  *uc_ptr / *mc_ptr
 * receive the unicast and multicast addresses of the same bytes; *mapped_bytes the size rounded
 * up to the multicast granularity.  Owned by the caller until mpo_nvls_free_local. */
mpo_status mpo_nvls_alloc_local(int64_t bytes, void** uc_ptr, void** mc_ptr, int64_t* mapped_bytes);
mpo_status mpo_nvls_free_local(void* uc_ptr, void* mc_ptr, int64_t mapped_bytes);

/* Diagnostic: checks the branch-free fast sqrt / division sequences of the step kernels against
 * the compiler's IEEE sqrtf() and `/`.  sqrt: ALL 2^32 binary32 patterns;
 * division: `pairs` operand pairs drawn from a counter-based generator keyed by `seed` (bit
 * patterns uniform over the accepted exponent window, plus fully random patterns).  Wherever an
 * input is accepted by the fast range check the two results must be bit-identical.
 *   counts: DEVICE array of 4 uint64, zeroed by the call, then accumulated in stream order:
 *           [0] sqrt mismatches, [1] division mismatches, [2] sqrt inputs on the fast path,
 *           [3] division pairs on the fast path. */
mpo_status mpo_selfcheck_fastmath(int64_t pairs, uint64_t seed, unsigned long long* counts,
                                  mpo_stream stream);

/* Thread-local description of the last non-OK status ("" if none). */
const char* mpo_last_error(void);

/* 1 if this build was compiled with -fmad=false (bit-exact mode), else 0. */
int32_t mpo_build_exact(void);

/* Number of kernels this library launched since load (for the bench's gpu_launches claim). */
int64_t mpo_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MPO_H */
