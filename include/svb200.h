/*
 * svb200.h -- C ABI of the B200-native gate-application hot path.
 *
 * The reference (qHiPSTER restated as the Python package `svsim`) has no FFI:
 * its hot path sits behind Python functions.  Each entry point below is the
 * drop-in for one of those functions; the host mirror in
 * paper_1601_07195_b200/ binds them with ctypes, validates arguments first
 * (raising the reference's exception types) and passes plain device pointers,
 * sizes and a cudaStream_t.  No torch types cross this boundary.
 *
 * Conventions (all entry points):
 *   - amplitudes are complex128 = interleaved (re, im) float64 = CUDA double2,
 *     16-byte aligned, 2^m contiguous elements (pkg/src/svsim/core.py:67-75);
 *   - updates are in place, stream-ordered and asynchronous; the caller owns
 *     every buffer (core.py LocalState; SURVEY.md 8b "conventions to keep");
 *   - a gate matrix is 8 doubles q11re q11im q12re q12im q21re q21im q22re q22im
 *     (row-major 2x2, pkg/src/svsim/kernels.py:36-68);
 *   - return 0 on success, SV_EINVAL for a rejected argument, SV_ECUDA for a
 *     CUDA launch/runtime error; sv_last_error() holds the message (per thread).
 *   - arithmetic reproduces the reference's rounding sequence exactly
 *     (kernels.py:120-131 mix()).
 */
#ifndef SVB200_H
#define SVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SV_OK 0
#define SV_EINVAL (-1)
#define SV_ECUDA (-2)

/* Largest fused tile exponent: one CTA keeps 2^SV_FUSED_MAX_TILE amplitudes
 * (128 KiB) resident in shared memory. */
#define SV_FUSED_MAX_TILE 13
/* Gates carried by one fused launch (kernel parameter space). */
#define SV_FUSED_MAX_GATES 256
/* Gates carried by one same-target stage (sv_exchange_stage). */
#define SV_STAGE_MAX_GATES 64
/* One local stage pass (SV_GROUP_STAGE): at most this many gates, whose targets
 * fall in at most SV_MSTAGE_MAX_TARGETS distinct qubits (controls anywhere). */
#define SV_MSTAGE_MAX_GATES 128
#define SV_MSTAGE_MAX_TARGETS 4
/* Scratch doubles sv_norm_sq needs (per-block partials + result). */
#define SV_NORM_SCRATCH 1025

/* One gate of a fused run: `control` = -1 for an uncontrolled gate.
 * Mirrors svsim GateOp (pkg/src/svsim/circuits.py:71-99). */
typedef struct {
  int32_t target;
  int32_t control;
  double q[8];
} sv_gate;

int sv_version(void);
const char *sv_last_error(void);
/* Number of CUDA kernels this library has launched (process lifetime). */
uint64_t sv_launch_count(void);

/* Replaces svsim.kernels.apply_single_raw (pkg/src/svsim/kernels.py:187-189):
 * pairs (i, i + 2^k) with bit k of i clear, 0 <= k < m. */
int sv_apply_single(void *amps, int m, int k, const double *q, void *stream);

/* Replaces svsim.kernels.apply_controlled_raw (kernels.py:192-196): pairs with
 * bit c set and bit t in {0,1}; c != t, both < m.  Touches only the bit-c = 1
 * half of the slice. */
int sv_apply_controlled(void *amps, int m, int c, int t, const double *q, void *stream);

/* Replaces the FusedBlockRun branch of svsim.fusion.execute_plan
 * (pkg/src/svsim/fusion.py:124-135), i.e. apply_block (kernels.py:225-240) on
 * every contiguous 2^l block: the gates are applied in order to each block
 * while it stays resident in shared memory, one HBM pass per launch.
 * Requires 1 <= l <= min(m, SV_FUSED_MAX_TILE), every gate qubit < l,
 * 1 <= ngates <= SV_FUSED_MAX_GATES. */
int sv_apply_fused(void *amps, int m, int l, const sv_gate *gates, int ngates, void *stream);

/* Native pass planner: applies an arbitrary local gate list (targets and
 * controls < m) in order, grouping it into as few HBM passes as the kernels
 * allow -- maximal runs of gates with target < tile (controls anywhere: above
 * the tile they are per-CTA predicates) go through the register-tiled kernel;
 * runs whose targets lie in at most SV_MSTAGE_MAX_TARGETS qubits go through one
 * multi-target stage pass (whichever covers a run more cheaply, by a B200 cost
 * model); anything else is a single-gate launch.  Bit-identical to applying the
 * gates one by one with sv_apply_single / sv_apply_controlled (the reference's
 * engine.py:88-95 loop).  tile = 0 picks min(m, SV_FUSED_MAX_TILE); otherwise
 * 9 <= tile <= min(m, SV_FUSED_MAX_TILE). */
int sv_apply_gates(void *amps, int m, const sv_gate *gates, int ngates, int tile, void *stream);

/* Launch-group kinds of the pass planner. */
#define SV_GROUP_GATES 0 /* one launch per gate (sv_apply_single / sv_apply_controlled) */
#define SV_GROUP_TILE 1  /* register-tiled run: targets < tile-SV_TILE_GATHER plus up to SV_TILE_GATHER higher bits */
/* Slice bits a register tile gathers (its top tile bits; the rest are runs of 2^(tile-8) amplitudes). */
#define SV_TILE_GATHER 8
#define SV_GROUP_STAGE 2 /* stage: targets in <= SV_MSTAGE_MAX_TARGETS qubits, 16 amplitudes per thread */
#define SV_GROUP_LOW 3   /* every target in qubits 0..5 (k_dlow: one warp per 256 amplitudes, two register
                          * layouts switched through a warp-private transpose).  Exact mode: speculative
                          * structure-specialised updates + one zero test + exact replay, bitwise equal to
                          * per-gate execution; tolerance mode: diagonal runs inside the block as product
                          * tables / per-stage factors, deferred butterfly factors */
#define SV_GROUP_STAGE2 4 /* tolerance mode only: <= 4 targets, then <= 4 others (a 4096-amplitude tile
                           * per CTA, two k_dstage programs around a shared-memory transpose) */

/* The planner of sv_apply_gates, exposed (pure host code, no GPU needed):
 * writes the end index and kind of each launch group, returns the number of
 * groups (or a negative error).  sv_apply_gates == sv_apply_group over these. */
int sv_plan_gates(int m, const sv_gate *gates, int ngates, int tile, int32_t *group_end, int32_t *group_kind,
                  int max_groups);

/* Execute one planned group (kind SV_GROUP_*), e.g. to time groups one by one. */
int sv_apply_group(void *amps, int m, int kind, const sv_gate *gates, int ngates, int tile, void *stream);

/* Flags of the *_ex planner entry points. */
#define SV_FLAG_TOLERANCE 1 /* FusionConfig(exact=False): stage groups run k_dstage, which collapses every
                             * diagonal gate whose control is outside the pass's four slot bits into one
                             * per-amplitude factor (values equal mix()'s within rounding, not bit for bit;
                             * north_star's 1e-12 sqrt(G) bound); the cost model plans for it.  0: exact. */
/* sv_apply_gates / sv_plan_gates / sv_apply_group with flags (SV_FLAG_*); flags = 0 is the exact
 * entry point.  No reference counterpart: the tolerance mode extends fusion.py:71-135's plans. */
int sv_apply_gates_ex(void *amps, int m, const sv_gate *gates, int ngates, int tile, int flags, void *stream);
int sv_plan_gates_ex(int m, const sv_gate *gates, int ngates, int tile, int flags, int32_t *group_end,
                     int32_t *group_kind, int max_groups);
int sv_apply_group_ex(void *amps, int m, int kind, const sv_gate *gates, int ngates, int tile, int flags,
                      void *stream);

/* How a two-phase tolerance group (SV_GROUP_STAGE2) will run -- pure host code, no GPU:
 * SV_SHAPE_INTERPRETED (the op interpreter of k_dstage2), SV_SHAPE_FORWARD / SV_SHAPE_INVERSE
 * (both phases have the shape of transform stages, the reference's build_qft stages
 * circuits.py:141-156 or their inverse: straight-line compiled phases, k_xstage2), or a
 * negative error when the gates are not a two-phase group.  No reference counterpart. */
#define SV_SHAPE_INTERPRETED 0
#define SV_SHAPE_FORWARD 1
#define SV_SHAPE_INVERSE 2
int sv_stage2_shape(int m, const sv_gate *gates, int ngates);
/* The same question for an exact stage group (SV_GROUP_STAGE): SV_SHAPE_FORWARD / SV_SHAPE_INVERSE when
 * the group is transform stages (or inverse stages) in circuit order (k_mstage with compiled control
 * flow; same arithmetic, same order, bit-identical), SV_SHAPE_INTERPRETED for the run-dispatched
 * kernel.  Pure host code. */
int sv_stage_shape(int m, const sv_gate *gates, int ngates);

/* Staged variant of sv_exchange for the NCCL data plane (NvlinkFabric(data_plane=
 * "nccl"), the reference's chunked pipeline distributed.py:205-290 over NCCL
 * send/recv): `buf` holds the partner's elements j0 .. j0+count_j-1 of this rank's
 * computing half (contiguous); the kernel updates mine[] in place and leaves the
 * partner's updated elements in buf for the return send.  c_local as sv_exchange
 * but < m-1 (the caller handles the half-selecting bit); j0 and count_j aligned
 * to 2^(c_local+1). */
int sv_exchange_chunk(void *mine, void *buf, int m, int own_is_zero, int c_local, const double *q, uint64_t j0,
                      uint64_t count_j, void *stream);

/* The reference's _pair_kernel on two contiguous chunk vectors (distributed.py:187-202): element i
 * of `mine` pairs with element i of `theirs`; own_is_zero decides the operand order (this rank
 * holds a0: keep mix(mine, theirs, q11, q12), return mix(mine, theirs, q21, q22); else the
 * roles swap).  Both are updated in place (theirs = the returned values).  The staged data
 * planes use it on packed chunks (case 5: the bit-c = 1 elements, distributed.py:341-422). */
int sv_pair_update(void *mine, void *theirs, uint64_t count, int own_is_zero, const double *q, void *stream);

/* A stage of gates that all target the same global qubit, applied in ONE
 * exchange (sv_exchange generalised to a gate list): each pair crosses NVLink
 * once each way.  Controls must be local (< m) or -1; the caller drops gates
 * whose control is a rank bit that is 0 on this rank (both partners agree).
 * 1 <= ngates <= 64; the targets are implied by the partner pairing. */
int sv_exchange_stage(void *mine, void *theirs, int m, int own_is_zero, const sv_gate *gates, int ngates,
                      void *stream);

/* Replaces one rank's side of the half exchange:
 * svsim.distributed._run_exchange + chunked_exchange_pipeline + _pair_kernel
 * (pkg/src/svsim/distributed.py:187-311) and the packed remote-target case
 * (:404-422).  `theirs` is the partner's slice mapped into this process
 * (sv_ipc_open), so transfer and update are one kernel: each element of the
 * computed half is read from both slices, the kept value is stored locally and
 * the returned value is stored straight into the partner's slice over NVLink.
 * own_is_zero selects the computed half (first half on the zero side);
 * c_local = -1 exchanges every element, c_local in [0, m) only those with
 * local bit c_local set (case 5 of perfmodel.py:30-38; c_local = m-1 leaves the
 * zero side idle, as distributed.py:348-349).  The caller orders the launch
 * between two partner barriers. */
int sv_exchange(void *mine, void *theirs, int m, int own_is_zero, int c_local, const double *q,
                void *stream);

/* Diagonal gate (q12 = q21 = 0 exactly) on a global qubit without an exchange
 * (replaces, behind NvlinkFabric(diagonal_local=True), the
 * exchange of distributed.py:314-422 for such gates).  Two launches per rank
 * with a partner fence between them:
 *   sv_diag_global -- own elements (those with local bit c_local set, or all
 *     for c_local = -1) *= q11 (zero side) or q22 (one side), in place; writes
 *     the sign map of the ORIGINAL elements into `signs` (2 bits per element:
 *     SV_DIAG_SIGN_BYTES(m) bytes) and sets *flag (device int) when a product
 *     has a zero component;
 *   sv_diag_fix -- if *flag: for those elements adds the signed-zero partner
 *     term q12 * partner (q21 on the one side) using the partner's sign map
 *     (`partner_signs`, its CUDA-IPC mapping), which makes the result equal the
 *     exchange's mix() bit for bit, sign of zero included. */
#define SV_DIAG_SIGN_BYTES(m) ((((uint64_t)1 << (m)) + 31) / 32 * 8)
int sv_diag_global(void *amps, int m, int own_is_zero, int c_local, const double *q, void *signs, int *flag,
                   void *stream);
int sv_diag_fix(void *amps, int m, int own_is_zero, int c_local, const double *q, const void *partner_signs,
                const int *flag, void *stream);

/* Swap global qubit G (the pairing bit of `theirs`) with local qubit l
 * (communication-avoiding remapping): afterwards this rank
 * holds the amplitudes whose bit G equals its bit l.  Elements with local bit
 * l = 1 - b (b = this rank's bit G; own_is_zero = !b) trade places with the
 * partner's elements with bit l = b: 2^(m+3) bytes per direction, half of an
 * in-place exchange.  Both partners call it between two barriers; each moves
 * half of the pairs.  2 <= m, 0 <= l < m. */
int sv_swap_global(void *mine, void *theirs, int m, int own_is_zero, int l, void *stream);

/* Sum of |a|^2 over the slice (qubit = -1) or over local bit `qubit` = 1
 * (core.py:147-167 partials).  Deterministic: fixed grid, fixed reduction
 * order.  `scratch` is a device buffer of SV_NORM_SCRATCH doubles; the result
 * lands in scratch[SV_NORM_SCRATCH - 1]. */
int sv_norm_sq(const void *amps, int m, int qubit, double *scratch, void *stream);

/* max_i |a_i - b_i| (complex modulus) over two slices of 2^m amplitudes (the bench's
 * full-size self-check: a circuit followed by its inverse restores the input).
 * Result in scratch[SV_NORM_SCRATCH - 1], as sv_norm_sq. */
int sv_max_abs_diff(const void *a, const void *b, int m, double *scratch, void *stream);

/* Seeded i.i.d. complex Gaussian amplitudes (Philox4x32-10 + Box-Muller),
 * element j of rank r drawn from counter (r << m) + j, so a sharded state
 * equals the unsharded one.  Not normalised: follow with sv_norm_sq/sv_scale. */
int sv_init_random(void *amps, int m, uint64_t seed, uint64_t rank, void *stream);

/* amps *= s (real scale). */
int sv_scale(void *amps, int m, double s, void *stream);

/* |basis> on this slice: zero everything, amps[local] = 1 if local >= 0. */
int sv_init_basis(void *amps, int m, int64_t local, void *stream);

/* Stream-ordered byte copy between any two UVA addresses (device, mapped
 * peer, pinned host): gather_full_state's NVLink read (distributed.py:462-482). */
int sv_copy(void *dst, const void *src, uint64_t nbytes, void *stream);

/* CUDA IPC for the exchange data plane (replaces the Transport ABC's byte
 * channel, distributed.py:60-92).  handle_out receives 64 bytes; offset_out the
 * byte offset of ptr inside its allocation. */
int sv_ipc_handle(const void *ptr, void *handle_out, uint64_t *offset_out);
int sv_ipc_open(const void *handle, uint64_t offset, void **ptr_out);
int sv_ipc_close(void *ptr, uint64_t offset);

#ifdef __cplusplus
}
#endif

#endif /* SVB200_H */
