// svb200.cu -- hand-written sm_100a kernels + C ABI for the gate-application hot path.
//
// See include/svb200.h for the ABI contract and DESIGN.md for the data layout,
// the roofline each kernel is held to and the parity argument.  Every kernel
// that touches amplitudes evaluates the reference's pair update
// (pkg/src/svsim/kernels.py:120-131) with the rounding sequence numpy uses:
//
//   cmul(r, a)  = ( fma(r.re, a.re, -(a.im*r.im)),  fma(r.re, a.im, a.re*r.im) )
//   mix(a0,a1,r0,r1) = cmul(r0,a0) + cmul(r1,a1)      (componentwise add)
//
// written with __fma_rn/__dmul_rn/__dadd_rn so nvcc cannot re-associate or
// contract differently; results are bit-identical to the reference and to
// the tests' CPU oracle, and independent of launch geometry, fusion and sharding.

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "svb200.h"

#define SV_ABI_VERSION 1

namespace {

thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int after_launch(const char *what, int nlaunch = 1) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add((uint64_t)nlaunch, std::memory_order_relaxed);
  return SV_OK;
}

struct GateQ {
  double v[8];  // q11re q11im q12re q12im q21re q21im q22re q22im
};

GateQ load_q(const double *q) {
  GateQ g;
  memcpy(g.v, q, sizeof(g.v));
  return g;
}

// ------------------------------------------------------------------ arithmetic

__device__ __forceinline__ double2 cmul(double rr, double ri, double2 a) {
  const double t_im = __dmul_rn(a.y, ri), t_re = __dmul_rn(a.x, ri);  // both products first
  return make_double2(__fma_rn(rr, a.x, -t_im), __fma_rn(rr, a.y, t_re));
}

__device__ __forceinline__ double2 mix(double2 a0, double2 a1, double r0r, double r0i, double r1r,
                                       double r1i) {
  const double2 x = cmul(r0r, r0i, a0);
  const double2 y = cmul(r1r, r1i, a1);
  return make_double2(__dadd_rn(x.x, y.x), __dadd_rn(x.y, y.y));
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int b) {
  const uint64_t lo = x & ((1ull << b) - 1ull);
  return ((x >> b) << (b + 1)) | lo;
}

__device__ __forceinline__ uint64_t insert_one(uint64_t x, int b) { return insert_zero(x, b) | (1ull << b); }

__device__ __forceinline__ double2 shfl_xor2(double2 v, int mask) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}

// ---------------------------------------------------------------- local kernels
//
// Index spaces.  MODE_SINGLE: the slice itself, pairs on bit tv.
// MODE_CTL: the 2^(m-1) "virtual" elements with bit c set (virtual index v maps
// to insert_one(v, c)); the gate is a single-qubit gate on virtual bit tv
// (tv = t if t < c else t-1), so the kernel reads and writes only the
// control-set half.  MODE_PRED (c = 0, where control-set elements interleave
// at 16 B inside every 32-B sector): the full slice is streamed, pairs whose
// bit c is clear are written back unchanged, so every sector is read and
// written whole instead of half-used.

constexpr int BLK = 256;
constexpr int UNROLL = 4;
constexpr int PUNROLL = 8;  // pair mode: 8 pairs (256 B of loads) in flight per thread
enum { MODE_SINGLE = 0, MODE_CTL = 1, MODE_PRED = 2 };

template <int MODE>
__device__ __forceinline__ uint64_t vmap(uint64_t v, int c) {
  return MODE == MODE_CTL ? insert_one(v, c) : v;
}

// Pair mode (tv >= 5): each thread owns PUNROLL pairs; a warp's 32 consecutive
// pairs give two fully coalesced 512-B streams (a[i0], a[i0 + 2^tv]).
template <int MODE>
__global__ void __launch_bounds__(BLK) k_pairs(double2 *__restrict__ a, uint64_t npairs, int tv, int c,
                                               GateQ q) {
  const uint64_t tb = 1ull << tv;
  const uint64_t p0 = (uint64_t)blockIdx.x * (BLK * PUNROLL) + threadIdx.x;
  double2 x0[PUNROLL], x1[PUNROLL];
  uint64_t i0[PUNROLL], i1[PUNROLL];
#pragma unroll
  for (int u = 0; u < PUNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    const uint64_t v0 = insert_zero(p, tv);
    i0[u] = vmap<MODE>(v0, c);
    i1[u] = vmap<MODE>(v0 | tb, c);
    if (p < npairs) {
      x0[u] = a[i0[u]];
      x1[u] = a[i1[u]];
    }
  }
#pragma unroll
  for (int u = 0; u < PUNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    if (p >= npairs) continue;
    double2 n0 = mix(x0[u], x1[u], q.v[0], q.v[1], q.v[2], q.v[3]);
    double2 n1 = mix(x0[u], x1[u], q.v[4], q.v[5], q.v[6], q.v[7]);
    if (MODE == MODE_PRED && !((i0[u] >> c) & 1ull)) {
      n0 = x0[u];
      n1 = x1[u];
    }
    a[i0[u]] = n0;
    a[i1[u]] = n1;
  }
}

// Shuffle mode (tv < 5): a warp streams 32 consecutive (virtual) elements per
// unroll step; the pair partner sits in lane ^ 2^tv.  Each lane produces one
// output with the operand order of the reference (a0 = bit-clear element).
template <int MODE>
__global__ void __launch_bounds__(BLK) k_shfl(double2 *__restrict__ a, uint64_t nvirt, int tv, int c,
                                              GateQ q) {
  const int lane = threadIdx.x & 31;
  const bool hi = (lane >> tv) & 1;
  const double r0r = hi ? q.v[4] : q.v[0], r0i = hi ? q.v[5] : q.v[1];
  const double r1r = hi ? q.v[6] : q.v[2], r1i = hi ? q.v[7] : q.v[3];
  const int mask = 1 << tv;
  const uint64_t v0 = (uint64_t)blockIdx.x * (BLK * UNROLL) + threadIdx.x;
  double2 x[UNROLL];
  uint64_t idx[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const uint64_t v = v0 + (uint64_t)u * BLK;
    idx[u] = vmap<MODE>(v, c);
    if (v < nvirt) x[u] = a[idx[u]];  // warp-uniform: nvirt is a multiple of 32
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const uint64_t v = v0 + (uint64_t)u * BLK;
    if (v >= nvirt) continue;
    const double2 o = shfl_xor2(x[u], mask);
    const double2 a0 = hi ? o : x[u];
    const double2 a1 = hi ? x[u] : o;
    double2 r = mix(a0, a1, r0r, r0i, r1r, r1i);
    if (MODE == MODE_PRED && !((idx[u] >> c) & 1ull)) r = x[u];
    a[idx[u]] = r;
  }
}

// ------------------------------------------------------------------ fused runs
//
// One CTA per 2^T tile: coalesced 16-B loads into shared memory, the run's
// gates applied in order on the resident tile (one __syncthreads per gate),
// one coalesced store.  One HBM read + write of the slice per launch no matter
// how many gates the run holds.

struct FusedParams {
  int ngates;
  int pad;
  sv_gate g[SV_FUSED_MAX_GATES];
};

template <int T>
struct FusedShape {
  static constexpr int NT = (T >= 10) ? 512 : ((1 << (T - 1)) < 32 ? 32 : (1 << (T - 1)));
  static constexpr int N = 1 << T;
};

template <int T>
__global__ void __launch_bounds__(FusedShape<T>::NT) k_fused(double2 *__restrict__ a, const FusedParams P) {
  constexpr int NT = FusedShape<T>::NT;
  constexpr int N = FusedShape<T>::N;
  extern __shared__ double2 s[];
  double2 *__restrict__ g = a + ((uint64_t)blockIdx.x << T);
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = tid; i < N; i += NT) s[i] = g[i];
  __syncthreads();
  for (int gi = 0; gi < P.ngates; ++gi) {
    const int t = P.g[gi].target, c = P.g[gi].control;
    const double q0 = P.g[gi].q[0], q1 = P.g[gi].q[1], q2 = P.g[gi].q[2], q3 = P.g[gi].q[3];
    const double q4 = P.g[gi].q[4], q5 = P.g[gi].q[5], q6 = P.g[gi].q[6], q7 = P.g[gi].q[7];
    const int tb = 1 << t;
    if (c < 0) {
      for (int p = tid; p < (N >> 1); p += NT) {
        const int i0 = (int)insert_zero((uint64_t)p, t);
        const double2 x0 = s[i0], x1 = s[i0 | tb];
        s[i0] = mix(x0, x1, q0, q1, q2, q3);
        s[i0 | tb] = mix(x0, x1, q4, q5, q6, q7);
      }
    } else {
      const int lo = c < t ? c : t, hi = c < t ? t : c;
      for (int p = tid; p < (N >> 2); p += NT) {
        const int i0 = (int)insert_zero(insert_zero((uint64_t)p, lo), hi) | (1 << c);
        const double2 x0 = s[i0], x1 = s[i0 | tb];
        s[i0] = mix(x0, x1, q0, q1, q2, q3);
        s[i0 | tb] = mix(x0, x1, q4, q5, q6, q7);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = tid; i < N; i += NT) g[i] = s[i];
}

// ------------------------------------------------- structure-specialised pair update
//
// The host classifies every gate once (classify_gate):
//   KIND_GENERAL  full mix() for both outputs (10 FP64 ops each);
//   KIND_DIAG     q12 == q21 == 0 exactly (any zero signs):  new0 = cmul(q11,a0) + cmul(q12,a1)
//                 where cmul(q12,a1) is a pair of signed zeros, so the add is the identity unless
//                 a component of cmul(q11,a0) is itself zero -- only then is the second product
//                 formed.  Bit-identical to mix(), ~40 % of its FP64 work;
//   KIND_PHASE    KIND_DIAG with q11 == 1 + (+-0)i exactly (R_k, S, T, Z-type phases):
//                 cmul(1,a0) == a0 whenever a0 has no zero component, so new0 is a0 untouched.
// Zero tests are integer tests on the bit patterns (ALU pipe, not FP64).

enum { KIND_GENERAL = 0, KIND_DIAG = 1, KIND_PHASE = 2, KIND_REAL = 3, KIND_HSHARE = 4, KIND_COUNT = 5 };
// Tolerance mode only (k_dstage): a Hadamard-like butterfly a0 + a1, a0 - a1 whose common real
// factor s is deferred into one per-thread scale applied after the pass.
constexpr int KIND_HBF = 5;

__device__ __forceinline__ bool nonzero2(double2 v) {
  const int mx = (__double2hiint(v.x) & 0x7fffffff) | __double2loint(v.x);
  const int my = (__double2hiint(v.y) & 0x7fffffff) | __double2loint(v.y);
  return (mx != 0) & (my != 0);
}

__device__ __forceinline__ double2 diag_out(double rr, double ri, double2 self, double zr, double zi,
                                            double2 other) {
  double2 r = cmul(rr, ri, self);
  if (!nonzero2(r)) {
    const double2 z = cmul(zr, zi, other);
    r = make_double2(__dadd_rn(r.x, z.x), __dadd_rn(r.y, z.y));
  }
  return r;
}

template <int KIND>
__device__ __forceinline__ void pair_update(double2 &a0, double2 &a1, const double *q) {
  double2 n0, n1;
  if (KIND == KIND_GENERAL) {
    // mix() for both outputs, every product formed first, then the fmas, then the adds (the
    // same rounding sequence; the order only helps ptxas keep a0/a1 in their registers)
    const double t0 = __dmul_rn(a0.y, q[1]), t1 = __dmul_rn(a0.x, q[1]);
    const double t2 = __dmul_rn(a1.y, q[3]), t3 = __dmul_rn(a1.x, q[3]);
    const double t4 = __dmul_rn(a0.y, q[5]), t5 = __dmul_rn(a0.x, q[5]);
    const double t6 = __dmul_rn(a1.y, q[7]), t7 = __dmul_rn(a1.x, q[7]);
    const double p0r = __fma_rn(q[0], a0.x, -t0), p0i = __fma_rn(q[0], a0.y, t1);
    const double p1r = __fma_rn(q[2], a1.x, -t2), p1i = __fma_rn(q[2], a1.y, t3);
    const double p2r = __fma_rn(q[4], a0.x, -t4), p2i = __fma_rn(q[4], a0.y, t5);
    const double p3r = __fma_rn(q[6], a1.x, -t6), p3i = __fma_rn(q[6], a1.y, t7);
    n0 = make_double2(__dadd_rn(p0r, p1r), __dadd_rn(p0i, p1i));
    n1 = make_double2(__dadd_rn(p2r, p3r), __dadd_rn(p2i, p3i));
  } else {
    if (KIND == KIND_PHASE && nonzero2(a0))
      n0 = a0;
    else
      n0 = diag_out(q[0], q[1], a0, q[2], q[3], a1);
    n1 = diag_out(q[6], q[7], a1, q[4], q[5], a0);
  }
  a0 = n0;
  a1 = n1;
}

// Speculative pair updates (the fused kernels test their final values for
// zeros and replay exactly if they see one -- see stage_gate_fast):
//   KIND_PHASE / KIND_DIAG  products only;
//   KIND_REAL    every imaginary part +-0: real products only, round(u.re * a) per component;
//   KIND_HSHARE  real with u00 = u01 = u10 = -u11 = s (Hadamard-like): the products s*a0, s*a1 are
//                shared by both outputs (round(-s*x) == -round(s*x)): 8 FP64 ops instead of 20.
// Each equals mix() up to the signs of zeros.
template <int KIND>
__device__ __forceinline__ void spec_pair(double2 &a0, double2 &a1, const double *q) {
  if (KIND == KIND_GENERAL) {
    pair_update<KIND_GENERAL>(a0, a1, q);
  } else if (KIND == KIND_PHASE) {
    a1 = cmul(q[6], q[7], a1);
  } else if (KIND == KIND_DIAG) {
    a0 = cmul(q[0], q[1], a0);
    a1 = cmul(q[6], q[7], a1);
  } else if (KIND == KIND_REAL) {
    const double2 n0 = make_double2(__dadd_rn(__dmul_rn(q[0], a0.x), __dmul_rn(q[2], a1.x)),
                                    __dadd_rn(__dmul_rn(q[0], a0.y), __dmul_rn(q[2], a1.y)));
    a1 = make_double2(__dadd_rn(__dmul_rn(q[4], a0.x), __dmul_rn(q[6], a1.x)),
                      __dadd_rn(__dmul_rn(q[4], a0.y), __dmul_rn(q[6], a1.y)));
    a0 = n0;
  } else if (KIND == KIND_HBF) {
    const double2 n0 = make_double2(__dadd_rn(a0.x, a1.x), __dadd_rn(a0.y, a1.y));
    a1 = make_double2(__dsub_rn(a0.x, a1.x), __dsub_rn(a0.y, a1.y));
    a0 = n0;
  } else {  // KIND_HSHARE
    const double s = q[0];
    const double2 p0 = make_double2(__dmul_rn(s, a0.x), __dmul_rn(s, a0.y));
    const double2 p1 = make_double2(__dmul_rn(s, a1.x), __dmul_rn(s, a1.y));
    a0 = make_double2(__dadd_rn(p0.x, p1.x), __dadd_rn(p0.y, p1.y));
    a1 = make_double2(__dsub_rn(p0.x, p1.x), __dsub_rn(p0.y, p1.y));
  }
}

// ------------------------------------------------------- register-tiled fused runs
//
// One CTA per 2^T tile (T = 9..13), TR = 4 "register qubits": each of the
// 2^(T-4) threads holds 16 amplitudes in registers, the amplitudes whose tile
// index has a fixed thread part and all 16 values of the 4 register bits S.
// A gate whose target is in S is applied entirely in registers; its control
// may be anywhere: a register bit (per-pair mask), a thread bit (per-thread
// predicate) or a bit above the tile (per-CTA predicate).  The host splits the
// gate list into segments with one register set each (greedy look-ahead over
// upcoming targets); between segments the tile is transposed through shared
// memory (XOR-swizzled so the 16-B accesses of each quarter warp hit distinct
// bank groups).  The first segment reuses the natural layout of the coalesced
// global load when its register set is the top four tile bits, and the last
// one stores straight to global when it ends in that layout.

#ifndef SV_TILE_TR
#define SV_TILE_TR 4  // register qubits per thread; TR = 3 measured slower (random 64-gate run 81 vs 66 ms)
#endif
constexpr int TR = SV_TILE_TR;
static_assert(TR == 3 || TR == 4, "tile register bits");
#ifndef SV_TILE_MINB
#define SV_TILE_MINB 2  // CTAs per SM for T <= 12 tiles (measured: 1 CTA with 255 registers is 1.6x slower)
#endif
constexpr int TRN = 1 << TR;
#ifndef SV_TILE_G
#define SV_TILE_G SV_TILE_GATHER  // gathered slice bits per tile (the top G tile bits; runs of 2^(T-G) amplitudes).
// Measured (random config-4-shape steps of 25 Haar gates, n = 30, T = 12): G = 4/5/6/7/8/9 ->
// 32.7/31.9/31.4/28.8/27.2/27.4 ms (fewer passes per circuit; same per-pass time).
#endif
constexpr int TG_BITS = SV_TILE_G;
static_assert(TG_BITS >= TR && TG_BITS <= 9, "gathered tile bits: TR..9 (T >= 9)");
constexpr uint32_t TFULL = (1u << TRN) - 1u;  // every register pair of a gate active

// registers j whose register bit b is set (a control on register bit b)
__host__ __device__ constexpr uint32_t reg_mask(int b) {
  return TFULL & (b == 0 ? 0xAAAAu : b == 1 ? 0xCCCCu : b == 2 ? 0xF0F0u : 0xFF00u);
}

struct TileHB {
  int v[TG_BITS];
};
constexpr int TILE_MAX_GATES = 256;
constexpr int TILE_MAX_SEGS = 64;

#ifndef SV_TILE_HDR64
#define SV_TILE_HDR64 1  // one 8-byte gate-header load (measured: 8 transform stages as one tile 46.7 -> 43.3 ms)
#endif

struct TileGate {
  int8_t tb;     // register bit of the target
  int8_t cmode;  // 0: none, 1: register bit cbit, 2: tile bit cbit (thread part), 3: above the tile
  int8_t cbit;
  int8_t kind;
  int32_t cabove;  // cmode 3: global index bit
  double q[8];
};
static_assert(offsetof(TileGate, cabove) == 4 && offsetof(TileGate, q) == 8, "8-byte gate header");

struct TileSeg {
  uint8_t S[4];       // tile bits held in register bits 0..TR-1 (ascending)
  uint8_t tbits[12];  // tile bit of thread-index bit b
  int16_t first, count;
  int8_t natural;
  int8_t plain;  // every gate of the segment is uncontrolled and general: the lean gate loop
  int8_t pad[2];
};

// A tile is 2^T amplitudes: tile bits 0..T-G-1 are slice bits 0..T-G-1
// (contiguous runs, coalesced), tile bits T-G..T-1 are the slice bits
// hb[0..G-1] (G = TG_BITS, ascending, any positions >= T-G).  hb = {T-G, ..,
// T-1} is the contiguous block of the reference's apply_block; other choices
// put high qubits into the tile so runs of gates on arbitrary targets fuse
// (the tile then is a strided gather).  The natural register layout: thread
// bits = tile bits 0..T-TR-1, register bits = tile bits T-TR..T-1.
struct TileParams {
  int nsegs;
  int last_natural;
  int hb[TG_BITS];
  TileSeg seg[TILE_MAX_SEGS];
  TileGate g[TILE_MAX_GATES];
};

template <int T>
__device__ __forceinline__ uint64_t tile_base(uint64_t b, const int (&hb)[TG_BITS]) {
  uint64_t x = b << (T - TG_BITS);
#pragma unroll
  for (int k = 0; k < TG_BITS; ++k) x = insert_zero(x, hb[k]);
  return x;
}

__device__ __forceinline__ int swz(int i) {
  int h = i >> 3;
  h ^= h >> 3;
  h ^= h >> 6;
  return i ^ (h & 7);
}

// swz is linear over GF(2) (shifts, XORs, a constant mask) and the thread part
// and the register masks occupy disjoint bits, so the slot of register j is
// swz(base) ^ XOR_{k in j} swz(m[k]).  Visiting the registers in Gray-code order
// turns the 16 addresses into one XOR each (instead of ~9 ALU ops per address).
// Global load / store of a thread's natural-layout registers: the offsets
// tid | XOR_{k in j} 2^hb[k] (disjoint bits), visited in Gray-code order.
template <int T, bool STORE>
__device__ __forceinline__ void tile_gxfer(double2 *__restrict__ a, double2 (&r)[TRN], uint64_t tile0, int tid,
                                           const int (&hb)[TG_BITS]) {
  constexpr int L = T - TG_BITS, RB = TG_BITS - TR;  // contiguous bits; gathered bits held by threads
  uint64_t off = tile0 | (uint64_t)(tid & ((1 << L) - 1));  // tile0 is zero on every tile bit
#pragma unroll
  for (int k = 0; k < RB; ++k) off |= (uint64_t)((tid >> (L + k)) & 1) << hb[k];
#pragma unroll
  for (int i = 0; i < TRN; ++i) {
    const int g = i ^ (i >> 1);
    if (i) off ^= 1ull << hb[RB + ((i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : 3)];
    if (STORE)
      a[off] = r[g];
    else
      r[g] = a[off];
  }
}

template <bool STORE>
__device__ __forceinline__ void tile_xfer(double2 *s, double2 (&r)[TRN], int base, const int (&m)[TR]) {
  int sm[TR];
#pragma unroll
  for (int k = 0; k < TR; ++k) sm[k] = swz(m[k]);
  int ad = swz(base);
#pragma unroll
  for (int i = 0; i < TRN; ++i) {
    const int g = i ^ (i >> 1);  // Gray code: g(i) and g(i-1) differ in bit ctz(i)
    if (i) ad ^= sm[(i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : 3];  // ctz(i), i < 16
    if (STORE)
      s[ad] = r[g];
    else
      r[g] = s[ad];
  }
}

// The TRN/2 register pairs of a gate on register bit TB, processed in groups
// of TG; for diagonal/phase gates the zero tests of a group are merged into
// one branch (see stage_gate).  FULL: every pair active (pm == TFULL).
constexpr int TG = 2;

#define PAIRS(k) ((((k) >> TB) << (TB + 1)) | ((k) & ((1 << TB) - 1)))  // k-th j with bit TB clear

// The exact update of one register bit's 8 pairs (mix() for general and real kinds; diagonal
// and phase kinds with per-group zero tests).
template <int TB, int KIND, bool FULL>
__device__ __forceinline__ void tile_gate_exact(double2 (&r)[TRN], uint32_t pm, const double *q) {
#pragma unroll
  for (int grp = 0; grp < TRN / 2 / TG; ++grp) {
    if (KIND == KIND_GENERAL || KIND >= KIND_REAL) {  // exact pass: real kinds run mix()
#pragma unroll
      for (int k = 0; k < TG; ++k) {
        const int j = PAIRS(grp * TG + k);
        if (FULL || ((pm >> j) & 1u)) pair_update<KIND_GENERAL>(r[j], r[j | (1 << TB)], q);
      }
    } else {
      double2 n0[TG], n1[TG];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < TG; ++k) {
        const int j = PAIRS(grp * TG + k);
        const bool act = FULL || ((pm >> j) & 1u);
        n0[k] = KIND == KIND_PHASE ? r[j] : cmul(q[0], q[1], r[j]);
        n1[k] = cmul(q[6], q[7], r[j | (1 << TB)]);
        bad |= act & !(nonzero2(n0[k]) & nonzero2(n1[k]));
      }
      if (bad) {
#pragma unroll
        for (int k = 0; k < TG; ++k) {
          const int j = PAIRS(grp * TG + k);
          if (FULL || ((pm >> j) & 1u)) pair_update<KIND_GENERAL>(r[j], r[j | (1 << TB)], q);
        }
      } else {
#pragma unroll
        for (int k = 0; k < TG; ++k) {
          const int j = PAIRS(grp * TG + k);
          if (FULL || ((pm >> j) & 1u)) {
            r[j] = n0[k];
            r[j | (1 << TB)] = n1[k];
          }
        }
      }
    }
  }
}

// spec (speculative pass, warp-uniform): diagonal/phase gates update in place
// with their products only; k_tile tests the final tile once and replays it
// from global memory with spec = false if any component is zero (see
// stage_gate_fast for why that one test is enough).
template <int TB, int KIND, bool FULL, bool SPEC>
__device__ __forceinline__ void tile_gate_k(double2 (&r)[TRN], uint32_t pm, const double *qp) {
  double q[8];  // once per gate in registers, not one constant-bank load per pair
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = qp[i];
  if (KIND != KIND_GENERAL && SPEC) {
#pragma unroll
    for (int k = 0; k < TRN / 2; ++k) {
      const int j = PAIRS(k);
      if (!(FULL || ((pm >> j) & 1u))) continue;
      spec_pair<KIND>(r[j], r[j | (1 << TB)], q);
    }
  } else {
    tile_gate_exact<TB, KIND, FULL>(r, pm, q);
  }
}

// One tile through the run: load (natural layout), segments with transposes,
// back to the natural layout in registers (the caller stores).
template <int T, bool SPEC>
__device__ __forceinline__ void tile_body(const double2 *__restrict__ a, uint64_t tile0, const int (&hb)[TG_BITS],
                                          int tid, const TileParams &P, double2 *s, double2 (&r)[TRN]) {
  constexpr int NT = 1 << (T - TR);
  tile_gxfer<T, false>(const_cast<double2 *>(a), r, tile0, tid, hb);
  // current layout: natural (register bits = top TR tile bits, thread bits ascending)
  int cbase = tid, c[TR];
#pragma unroll
  for (int k = 0; k < TR; ++k) c[k] = NT << k;
  bool touched = false;
  for (int sg = 0; sg < P.nsegs; ++sg) {
    const TileSeg &S = P.seg[sg];
    int mm[TR];
#pragma unroll
    for (int k = 0; k < TR; ++k) mm[k] = 1 << S.S[k];
    int base = 0;
#pragma unroll
    for (int b = 0; b < T - TR; ++b) base |= ((tid >> b) & 1) << S.tbits[b];
    if (!(sg == 0 && S.natural)) {
      if (touched) __syncthreads();
      tile_xfer<true>(s, r, cbase, c);
      __syncthreads();
      tile_xfer<false>(s, r, base, mm);
      touched = true;
    }
    cbase = base;
#pragma unroll
    for (int k = 0; k < TR; ++k) c[k] = mm[k];
#ifndef SV_TILE_NO_PLAIN
    if (S.plain) {  // one dispatch level (register bit) instead of three: fewer register shuffles
      for (int gi = S.first; gi < S.first + S.count; ++gi) {
        const TileGate &G = P.g[gi];
        switch (G.tb) {
          case 0: tile_gate_k<0, KIND_GENERAL, true, SPEC>(r, TFULL, G.q); break;
          case 1: tile_gate_k<1, KIND_GENERAL, true, SPEC>(r, TFULL, G.q); break;
          case 2: tile_gate_k<2, KIND_GENERAL, true, SPEC>(r, TFULL, G.q); break;
          default: tile_gate_k<TR - 1, KIND_GENERAL, true, SPEC>(r, TFULL, G.q); break;
        }
      }
      continue;
    }
#endif
    for (int gi = S.first; gi < S.first + S.count; ++gi) {
      const TileGate &G = P.g[gi];
#if SV_TILE_HDR64
      // tb, cmode, cbit, kind, cabove: one uniform 8-byte load instead of four byte loads
      const uint64_t hd = *reinterpret_cast<const uint64_t *>(&G);
      const int g_tb = (int)(hd & 0xff), g_cmode = (int)((hd >> 8) & 0xff), g_cbit = (int)((hd >> 16) & 0xff);
      const int g_kind = (int)((hd >> 24) & 0xff), g_cabove = (int)(hd >> 32);
#else
      const int g_tb = G.tb, g_cmode = G.cmode, g_cbit = G.cbit, g_kind = G.kind, g_cabove = G.cabove;
#endif
      uint32_t pm = TFULL;
      if (g_cmode == 1)
        pm = g_cbit == 0 ? reg_mask(0) : g_cbit == 1 ? reg_mask(1) : g_cbit == 2 ? reg_mask(2) : reg_mask(3);
      else if (g_cmode == 2)
        pm = ((base >> g_cbit) & 1) ? TFULL : 0u;
      else if (g_cmode == 3)
        pm = ((tile0 >> g_cabove) & 1ull) ? TFULL : 0u;
      if (pm == 0u) continue;  // control decided per thread / CTA: clear
      // one flat dispatch on (register bit, kind, all pairs or a register-bit control); a
      // compile-time mask per control slot (100 cases) measured slower: 64 gates 49.5 -> 54.8 ms
      const int kind = (!SPEC && g_kind >= KIND_REAL) ? KIND_GENERAL : g_kind;
      switch ((g_tb * KIND_COUNT + kind) * 2 + (pm != TFULL)) {
#define TF_CASE(TB_, K_, P_)                                                                       \
  case ((TB_)*KIND_COUNT + (K_)) * 2 + (P_):                                                      \
    tile_gate_k<((TB_) < TR ? (TB_) : TR - 1), K_, (P_) == 0, SPEC>(r, pm, G.q);                 \
    break;
#define TF_K(TB_, K_) TF_CASE(TB_, K_, 0) TF_CASE(TB_, K_, 1)
#define TF_TB(TB_) TF_K(TB_, KIND_GENERAL) TF_K(TB_, KIND_DIAG) TF_K(TB_, KIND_PHASE) TF_K(TB_, KIND_REAL) TF_K(TB_, KIND_HSHARE)
        TF_TB(0) TF_TB(1) TF_TB(2) TF_TB(3)
#undef TF_TB
#undef TF_K
#undef TF_CASE
        default: break;
      }
    }
  }
  if (!P.last_natural) {
    if (touched) __syncthreads();
    tile_xfer<true>(s, r, cbase, c);
    __syncthreads();
    int nat[TR];
#pragma unroll
    for (int k = 0; k < TR; ++k) nat[k] = NT << k;
    tile_xfer<false>(s, r, tid, nat);
  }
}

// The exact replay of one tile (rare: a zero component in the speculative
// result).  Out of line, so the hot kernel does not carry a second copy of
// the body in its register allocation (inlined, the pair spilled ~3 KB per
// thread at the 128-register cap); the call site keeps only a few scalars live.
template <int T>
__device__ __noinline__ void tile_replay(double2 *__restrict__ a, uint64_t tile0, TileHB h, const TileParams *P,
                                         double2 *s) {
  int hb[TG_BITS];
#pragma unroll
  for (int k = 0; k < TG_BITS; ++k) hb[k] = h.v[k];
  const int tid = threadIdx.x;
  double2 r[TRN];
  tile_body<T, false>(a, tile0, hb, tid, *P, s, r);
  tile_gxfer<T, true>(a, r, tile0, tid, hb);
}

// SPEC = true when the run is mostly diagonal/phase gates (host-chosen):
// speculative in-place updates, one zero test of the final tile, and on any
// zero component the whole tile is replayed exactly from global memory
// (nothing has been stored yet).  SPEC = false: the exact path.
template <int T, bool SPEC>
#ifndef SV_TILE_THREADS_SM
#define SV_TILE_THREADS_SM 512  // resident threads per SM the register budget must allow (0: SV_TILE_MINB CTAs); T = 11 at
// 512 (4 CTAs) instead of 256 (2): random 25-gate steps 32.1 -> 26.7 ms; 768 (80 registers) spills and is slower
#endif
__global__ void __launch_bounds__(1 << (T - TR), (T <= 12) ? (SV_TILE_THREADS_SM ? SV_TILE_THREADS_SM / (1 << (T - TR)) : SV_TILE_MINB) : 1)
    k_tile(double2 *__restrict__ a, const __grid_constant__ TileParams P) {
  extern __shared__ double2 s[];
  int hb[TG_BITS];
#pragma unroll
  for (int k = 0; k < TG_BITS; ++k) hb[k] = P.hb[k];
  const uint64_t tile0 = tile_base<T>(blockIdx.x, hb);  // every non-tile slice bit of this CTA
  const int tid = threadIdx.x;
  double2 r[TRN];
  tile_body<T, SPEC>(a, tile0, hb, tid, P, s, r);
  if (SPEC) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < TRN; ++j) ok &= nonzero2(r[j]);
    if (__syncthreads_or(!ok)) {
      TileHB h;
#pragma unroll
      for (int k = 0; k < TG_BITS; ++k) h.v[k] = hb[k];
      tile_replay<T>(a, tile0, h, &P, s);
      return;
    }
  }
  tile_gxfer<T, true>(a, r, tile0, tid, hb);
}

// ------------------------------------------------- same-target stages (exchange)
//
// A run of gates sharing one target (any controls, any structure) applied to
// pairs held in registers, in order -- e.g. a transform stage H(k), R(k, c) for
// every c < k.  Used by k_exchange_stage, where the target is a global qubit
// and the pair is (own element, partner element over NVLink); local stages go
// through k_mstage.  SUNROLL pairs per thread.

constexpr int STAGE_MAX_GATES = 64;

struct StageGate {
  uint64_t cmask;  // 1 << control; 0: uncontrolled
  int32_t kind;
  int32_t pad;
  double q[8];
};

struct StageParams {
  int ngates;
  int pad;
  StageGate g[STAGE_MAX_GATES];
};

#ifndef SV_SUNROLL
#define SV_SUNROLL 2  // measured best of 1/2/4/8 for the former local stage kernel (resident warps hide the per-gate chains)
#endif
constexpr int SUNROLL = SV_SUNROLL;

// One gate of a stage on U register pairs.  ok0[u] caches nonzero2(x0[u]):
// a phase gate leaves x0 untouched on its fast path, so a stage of phases
// tests each x0 once instead of once per gate.  Inactive pairs (control bit
// clear) cost one test and a branch (warp-uniform unless the control is one
// of the five lowest pair-index bits).
template <int KIND, int U>
__device__ __forceinline__ void stage_gate(double2 (&x0)[U], double2 (&x1)[U], bool (&ok0)[U],
                                           const uint64_t (&idx)[U], uint64_t cm, const double *qp) {
  double q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = qp[i];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (cm && !(idx[u] & cm)) continue;
    if (KIND == KIND_GENERAL) {
      pair_update<KIND_GENERAL>(x0[u], x1[u], q);
      ok0[u] = nonzero2(x0[u]);
      continue;
    }
    const double2 n1 = cmul(q[6], q[7], x1[u]);
    if (KIND == KIND_PHASE) {
      if (__builtin_expect(ok0[u] & nonzero2(n1), 1)) {
        x1[u] = n1;
        continue;
      }
    } else {
      const double2 n0 = cmul(q[0], q[1], x0[u]);
      if (__builtin_expect(nonzero2(n0) & nonzero2(n1), 1)) {
        x0[u] = n0;
        x1[u] = n1;
        ok0[u] = true;
        continue;
      }
    }
    pair_update<KIND_GENERAL>(x0[u], x1[u], q);  // exact: the definition itself
    ok0[u] = nonzero2(x0[u]);
  }
}

__device__ __forceinline__ void stage_gate_any(int kind, double2 (&x0)[SUNROLL], double2 (&x1)[SUNROLL],
                                               bool (&ok0)[SUNROLL], const uint64_t (&idx)[SUNROLL], uint64_t cm,
                                               const double *q) {
  if (kind == KIND_PHASE)
    stage_gate<KIND_PHASE, SUNROLL>(x0, x1, ok0, idx, cm, q);
  else if (kind == KIND_DIAG)
    stage_gate<KIND_DIAG, SUNROLL>(x0, x1, ok0, idx, cm, q);
  else
    stage_gate<KIND_GENERAL, SUNROLL>(x0, x1, ok0, idx, cm, q);
}

// Speculative fast path: general gates run the full mix(); diagonal and phase
// gates update in place with their products only.  The result is tested ONCE,
// after the whole stage:
//   Dropping the zero-matrix terms of mix() only ever changes the sign of a
//   zero: cmul(0, a) is a signed zero and x + (+-0) == x for x != 0.  And
//   values that agree up to the signs of their zeros stay that way through
//   any later mul/fma/add (a +-0 operand gives a +-0 product, which again only
//   matters when the other addend is zero).  So the fast path's final pairs
//   equal the exact ones except possibly where a final component is +-0.
// A thread with any zero component in its final pairs reloads them (nothing is
// stored before the stage is done) and replays the stage through
// stage_apply_exact; everyone else stores the fast result.  No per-gate tests.
template <int KIND>
__device__ __forceinline__ void stage_gate_fast(double2 (&x0)[SUNROLL], double2 (&x1)[SUNROLL],
                                                const uint64_t (&idx)[SUNROLL], uint64_t cm, const double *qp) {
  double q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = qp[i];
#pragma unroll
  for (int u = 0; u < SUNROLL; ++u) {
    if (cm && !(idx[u] & cm)) continue;
    if (KIND == KIND_GENERAL) {
      pair_update<KIND_GENERAL>(x0[u], x1[u], q);
    } else if (KIND == KIND_PHASE) {
      x1[u] = cmul(q[6], q[7], x1[u]);
    } else {
      x0[u] = cmul(q[0], q[1], x0[u]);
      x1[u] = cmul(q[6], q[7], x1[u]);
    }
  }
}

template <int SIG>
__device__ __forceinline__ bool stage_apply_fast(double2 (&x0)[SUNROLL], double2 (&x1)[SUNROLL],
                                                 const uint64_t (&idx)[SUNROLL], const StageParams &P) {
  int gi = 0;
  if (SIG == 1) {
    const StageGate &G = P.g[0];
    const uint64_t cm = G.cmask;
    if (G.kind == KIND_GENERAL)
      stage_gate_fast<KIND_GENERAL>(x0, x1, idx, cm, G.q);
    else if (G.kind == KIND_DIAG)
      stage_gate_fast<KIND_DIAG>(x0, x1, idx, cm, G.q);
    else
      stage_gate_fast<KIND_PHASE>(x0, x1, idx, cm, G.q);
    // The pairs of a thread differ only in the index bits that separate the unrolled
    // rows; any other control bit has the same value for all of them, so one test
    // (on a 32-bit word when it can) decides the whole row set.
    uint64_t rows = 0;
#pragma unroll
    for (int u = 1; u < SUNROLL; ++u) rows |= idx[u] ^ idx[0];
#pragma unroll 2
    for (gi = 1; gi < P.ngates; ++gi) {
      const StageGate &H = P.g[gi];
      const uint64_t cm = H.cmask;
      const double qr = H.q[6], qi = H.q[7];
      if (cm && !(cm & rows)) {
        if (!(idx[0] & cm)) continue;
#pragma unroll
        for (int u = 0; u < SUNROLL; ++u) x1[u] = cmul(qr, qi, x1[u]);
        continue;
      }
#pragma unroll
      for (int u = 0; u < SUNROLL; ++u) {
        if (cm && !(idx[u] & cm)) continue;
        x1[u] = cmul(qr, qi, x1[u]);
      }
    }
  } else {
    for (; gi < P.ngates; ++gi) {
      const StageGate &G = P.g[gi];
      const uint64_t cm = G.cmask;
      if (G.kind == KIND_PHASE)
        stage_gate_fast<KIND_PHASE>(x0, x1, idx, cm, G.q);
      else if (G.kind == KIND_DIAG)
        stage_gate_fast<KIND_DIAG>(x0, x1, idx, cm, G.q);
      else
        stage_gate_fast<KIND_GENERAL>(x0, x1, idx, cm, G.q);
    }
  }
  bool ok = true;
#pragma unroll
  for (int u = 0; u < SUNROLL; ++u) ok &= nonzero2(x0[u]) & nonzero2(x1[u]);
  return !ok;
}

// The exact path (replay): per-gate zero tests, falls back to mix() per pair.
// SIG 0: any mix of kinds.  SIG 1: gate 0 of any kind, every later gate a phase.
template <int SIG>
__device__ __forceinline__ void stage_apply_exact(double2 (&x0)[SUNROLL], double2 (&x1)[SUNROLL],
                                               const uint64_t (&idx)[SUNROLL], const StageParams &P) {
  bool ok0[SUNROLL];
#pragma unroll
  for (int u = 0; u < SUNROLL; ++u) ok0[u] = nonzero2(x0[u]);
  if (SIG == 1) {
    const StageGate &G = P.g[0];
    stage_gate_any(G.kind, x0, x1, ok0, idx, G.cmask, G.q);
    for (int gi = 1; gi < P.ngates; ++gi) {
      const StageGate &H = P.g[gi];
      stage_gate<KIND_PHASE, SUNROLL>(x0, x1, ok0, idx, H.cmask, H.q);
    }
  } else {
    for (int gi = 0; gi < P.ngates; ++gi) {
      const StageGate &G = P.g[gi];
      stage_gate_any(G.kind, x0, x1, ok0, idx, G.cmask, G.q);
    }
  }
}

// ------------------------------------------------------------ multi-target stages
//
// A run of gates whose targets lie in at most MS_K = 4 slice bits ("slots"),
// controls anywhere, in ONE HBM pass: each thread holds the 16 amplitudes that
// span the four slot bits and applies the whole run in registers -- e.g. four
// consecutive transform stages H(k), R(k, c) for all c < k.  A run with fewer
// targets is padded with the most used control bits, which turns those
// controls into compile-time pair patterns.
//
// A control on any other bit is decided per thread.  Above the bits that vary
// across a warp it is warp-uniform, so the warp classifies 32 gates at a time
// (one per lane) and ballots them into a mask of the gates that act anywhere in
// the warp, then visits only those, in order: a gate whose control is clear
// for the whole warp costs nothing.  Controls on lane bits stay per-lane (a
// divergent skip).
//
// Updates: general complex gates run mix() (exact); "real" gates (every
// imaginary part +-0) keep only the real products, Hadamard-like ones
// (u00 = u01 = u10 = -u11, real) also share them between the two outputs
// (8 FP64 ops per pair instead of 20); diagonal and phase gates only multiply.
// Each differs from mix() at most in the sign of a zero, so one zero test of
// the final eight amplitudes decides (see stage_gate_fast); a thread that sees
// a zero replays its group exactly, out of line (ms_replay).

#ifndef SV_MS_MINB
// Threads per SM the register budget must allow, in units of 256.  Measured, QFT(30):
// 8 amplitudes per thread (MS_K = 3): 2, 3, 4 -> 149, 120, 85 ms; 16 amplitudes (MS_K = 4):
// 512 / 640 / 768 / 896 threads -> 95 / 80 / 76.6 / 82 ms.  At 768 (80 registers) ptxas keeps
// ~1 KB per thread in local memory and the kernel is still fastest: it is bound by FP64
// latency with too few warps, not by the L1 traffic of the spills.
#define SV_MS_MINB 3
#endif
#ifndef SV_MS_K
#define SV_MS_K SV_MSTAGE_MAX_TARGETS  // slot bits per thread (2^MS_K amplitudes in registers)
#endif
constexpr int MS_K = SV_MS_K;
static_assert(MS_K == 3 || MS_K == 4, "stage slot bits");
constexpr int MS_N = 1 << MS_K;
#ifndef SV_MS_BLK
#define SV_MS_BLK 256  // K = 4, 3 CTAs/SM: 64/256 threads per CTA -> QFT(30) 80.3/76.6 ms (128: 79.1)
#endif
constexpr int MS_BLK = SV_MS_BLK;
constexpr int MS_MAX = SV_MSTAGE_MAX_GATES;
#ifndef SV_MS_HILANE
#define SV_MS_HILANE 1  // measured: QFT(30) 72.2 -> 69.5 ms
#endif

struct MsGate {
  int32_t code;  // (kind * MS_K + slot) * (MS_K + 1) + control slot (MS_K: none / not a slot)
  int32_t pad;
  double q[8];
};

// A run: consecutive gates with one code, inside one 32-gate ballot chunk h,
// at chunk bits lo..hi.  The kernel dispatches once per run and loops over the
// run's gates that act in the warp with the update compiled for that code.
struct MsRun {
  uint32_t range;  // chunk bits lo..hi of the run, precomputed on the host
  uint8_t code, h, lo, hi;
};

struct MsParams {
  int32_t ngates;
  int32_t nruns;
  int32_t bits[MS_K];     // slice bit of each slot, ascending
  alignas(8) uint8_t cbit[MS_MAX];  // control of gate g when it is not a slot bit, else 0xFF
                                    // (read 8 at a time: the alignment is required)
  MsRun run[MS_MAX + MS_MAX / 32];
  MsGate g[MS_MAX];
  int32_t hl[2];   // SV_MS_HILANE: slice bits of lane bits 3, 4 (-1: lanes on the low non-slot bits)
  int32_t ins[MS_K + 2];  // zero-insert positions of a group's base, ascending (slots, hl)
  int32_t nins;
};

// k-th amplitude index j of a thread with bit S set (and bit C set when C is a slot)
template <int S, int C>
__host__ __device__ constexpr int ms_hit(int k) {
  int seen = 0;
  for (int j = 0; j < MS_N; ++j) {
    if (!((j >> S) & 1) || (C < MS_K && !((j >> C) & 1))) continue;
    if (seen++ == k) return j;
  }
  return -1;
}

#ifndef SV_MS_ILP
// Amplitudes of a phase update whose products are formed before any of their fmas (1: one at a
// time, the compiler's order).  Measured, QFT(30): at the 80-register cap (768 threads per SM)
// ptxas keeps ONE pair of temporaries whatever the source order, and the grouping only adds
// moves (68.7 -> 69.9 ms); with 96 / 128 registers it interleaves 4+ products per warp but the
// lost warps cost more (640 threads 73.7 ms, 512 threads 92.7 ms).  tools/micro/fp64_ilp_probe.cu:
// two warps per scheduler with one amplitude in flight each already reach 75 % of the FP64 pipe.
#define SV_MS_ILP 1
#endif

// r[j] = cmul(qr + i qi, r[j]) for the amplitudes ms_hit<S, C>(0..N-1), SV_MS_ILP at a time
template <int S, int C>
__device__ __forceinline__ void ms_scale_hits(double2 (&r)[MS_N], double qr, double qi) {
  constexpr int N = (C < MS_K) ? MS_N / 4 : MS_N / 2;
  constexpr int G = SV_MS_ILP < N ? SV_MS_ILP : N;
#pragma unroll
  for (int k0 = 0; k0 < N; k0 += G) {
    double tr[G], ti[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = ms_hit<S, C>(k0 + u);
      tr[u] = __dmul_rn(r[j].y, qi);
      ti[u] = __dmul_rn(r[j].x, qi);
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = ms_hit<S, C>(k0 + u);
      r[j] = make_double2(__fma_rn(qr, r[j].x, -tr[u]), __fma_rn(qr, r[j].y, ti[u]));
    }
  }
}

// gate on slot S, control slot C (MS_K: none), all pairs of the thread
template <int S, int C, int KIND>
__device__ __forceinline__ void ms_apply(double2 (&r)[MS_N], const double *qp) {
  if constexpr (SV_MS_ILP > 1 && KIND == KIND_PHASE) {
    // a1 = cmul(q[6] + i q[7], a1): the same rounding sequence as spec_pair
    ms_scale_hits<S, C>(r, qp[6], qp[7]);
  } else {
    double q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = qp[i];
#pragma unroll
    for (int j = 0; j < MS_N; ++j) {
      if ((j >> S) & 1) continue;
      if (C < MS_K && !((j >> C) & 1)) continue;
      spec_pair<KIND>(r[j], r[j | (1 << S)], q);
    }
  }
}

// The gates of one run that act in this warp (act: chunk bits), in order; a
// gate in lane_dep has its control on a lane bit and is skipped per lane.
template <int S, int C, int KIND>
__device__ __forceinline__ void ms_loop(double2 (&r)[MS_N], uint32_t act, uint32_t lane_dep, int g0, uint64_t base,
                                        const MsParams &P) {
  if (!lane_dep) {  // the common case: one path through the loop, no per-gate test
    while (act) {
      const int b = __ffs(act) - 1;
      act &= act - 1;
      ms_apply<S, C, KIND>(r, P.g[g0 + b].q);
    }
    return;
  }
  while (act) {
    const int b = __ffs(act) - 1;
    act &= act - 1;
    const int gi = g0 + b;
    if (((lane_dep >> b) & 1u) && !((base >> P.cbit[gi]) & 1ull)) continue;
    ms_apply<S, C, KIND>(r, P.g[gi].q);
  }
}

__device__ __forceinline__ void ms_dispatch(int code, double2 (&r)[MS_N], uint32_t act, uint32_t lane_dep, int g0,
                                            uint64_t base, const MsParams &P) {
  switch (code) {
#define MS_CASE(K_, S_, C_)                            \
  case ((K_) * MS_K + (S_)) * (MS_K + 1) + (C_):      \
    ms_loop<S_, C_, K_>(r, act, lane_dep, g0, base, P); \
    break;
#if SV_MS_K == 3
#define MS_CASES_S(K_, S_) MS_CASE(K_, S_, 0) MS_CASE(K_, S_, 1) MS_CASE(K_, S_, 2) MS_CASE(K_, S_, 3)
#define MS_CASES(K_) MS_CASES_S(K_, 0) MS_CASES_S(K_, 1) MS_CASES_S(K_, 2)
#else
#define MS_CASES_S(K_, S_) \
  MS_CASE(K_, S_, 0) MS_CASE(K_, S_, 1) MS_CASE(K_, S_, 2) MS_CASE(K_, S_, 3) MS_CASE(K_, S_, 4)
#define MS_CASES(K_) MS_CASES_S(K_, 0) MS_CASES_S(K_, 1) MS_CASES_S(K_, 2) MS_CASES_S(K_, 3)
#endif
    MS_CASES(KIND_GENERAL) MS_CASES(KIND_DIAG) MS_CASES(KIND_PHASE) MS_CASES(KIND_REAL) MS_CASES(KIND_HSHARE)
#undef MS_CASES
#undef MS_CASES_S
#undef MS_CASE
    default: break;
  }
}

__device__ __forceinline__ uint64_t ms_off(int j, const uint64_t (&b)[MS_K]) {
  uint64_t o = 0;
#pragma unroll
  for (int s = 0; s < MS_K; ++s) o |= ((j >> s) & 1) ? b[s] : 0ull;
  return o;
}

// A stage group shaped like transform stages (the reference's build_qft, circuits.py:141-156),
// compiled: for slots s descending -- the slot's uncontrolled Hadamard-like gate, its phase gates
// controlled by the lower slots (descending), then its phase gates controlled from outside the
// slots (runs rlo..rhi-1 of MsParams.run) -- in exactly the circuit's order, so every amplitude
// sees mix()'s rounding sequence as in the dispatched path; only the control flow differs
// (no per-run switch over 100 specialised loops: 14 code blocks instead).  -1: absent.
struct XmParams {
  int32_t h[MS_K];
  int32_t ins[MS_K][MS_K];
  int32_t rlo[MS_K], rhi[MS_K];
  int32_t inverse, pad;  // inverse transform stages: slots ascending, each [outside phases, in-slot phases
                         // (control slots ascending), butterfly]
};

template <int S>
__device__ __forceinline__ void xm_slot(double2 (&r)[MS_N], uint64_t base, const MsParams &P, const XmParams &X,
                                        const uint32_t (&M)[4], const uint32_t (&L)[4]) {
  if (X.h[S] >= 0) ms_apply<S, MS_K, KIND_HSHARE>(r, P.g[X.h[S]].q);
  if (S > 2 && X.ins[S][2] >= 0) ms_apply<S, (S > 2 ? 2 : 0), KIND_PHASE>(r, P.g[X.ins[S][2]].q);
  if (S > 1 && X.ins[S][1] >= 0) ms_apply<S, (S > 1 ? 1 : 0), KIND_PHASE>(r, P.g[X.ins[S][1]].q);
  if (S > 0 && X.ins[S][0] >= 0) ms_apply<S, (S > 0 ? 0 : 1), KIND_PHASE>(r, P.g[X.ins[S][0]].q);
  for (int ri = X.rlo[S]; ri < X.rhi[S]; ++ri) {
    const MsRun R = P.run[ri];
    const uint32_t mh = R.h == 0 ? M[0] : R.h == 1 ? M[1] : R.h == 2 ? M[2] : M[3];
    const uint32_t lh = R.h == 0 ? L[0] : R.h == 1 ? L[1] : R.h == 2 ? L[2] : L[3];
    const uint32_t act = mh & R.range;
    if (act) ms_loop<S, MS_K, KIND_PHASE>(r, act, lh & R.range, 32 * R.h, base, P);
  }
}

template <int S>
__device__ __forceinline__ void xm_slot_inv(double2 (&r)[MS_N], uint64_t base, const MsParams &P, const XmParams &X,
                                            const uint32_t (&M)[4], const uint32_t (&L)[4]) {
  for (int ri = X.rlo[S]; ri < X.rhi[S]; ++ri) {
    const MsRun R = P.run[ri];
    const uint32_t mh = R.h == 0 ? M[0] : R.h == 1 ? M[1] : R.h == 2 ? M[2] : M[3];
    const uint32_t lh = R.h == 0 ? L[0] : R.h == 1 ? L[1] : R.h == 2 ? L[2] : L[3];
    const uint32_t act = mh & R.range;
    if (act) ms_loop<S, MS_K, KIND_PHASE>(r, act, lh & R.range, 32 * R.h, base, P);
  }
  if (S > 0 && X.ins[S][0] >= 0) ms_apply<S, (S > 0 ? 0 : 1), KIND_PHASE>(r, P.g[X.ins[S][0]].q);
  if (S > 1 && X.ins[S][1] >= 0) ms_apply<S, (S > 1 ? 1 : 0), KIND_PHASE>(r, P.g[X.ins[S][1]].q);
  if (S > 2 && X.ins[S][2] >= 0) ms_apply<S, (S > 2 ? 2 : 0), KIND_PHASE>(r, P.g[X.ins[S][2]].q);
  if (X.h[S] >= 0) ms_apply<S, MS_K, KIND_HSHARE>(r, P.g[X.h[S]].q);
}

// The speculative run (all 32 lanes of the warp take part).  XF: the compiled transform shape.
template <bool XF>
__device__ __forceinline__ void ms_run(double2 (&r)[MS_N], uint64_t base, const MsParams &P, const XmParams &X) {
  const int lane = threadIdx.x & 31;
  uint64_t vary = base ^ __shfl_sync(0xffffffffu, base, 0);  // index bits that differ between lanes
  vary = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(vary >> 32)) << 32) |
         __reduce_or_sync(0xffffffffu, (unsigned)vary);
  const uint64_t *cw = reinterpret_cast<const uint64_t *>(P.cbit);  // 8 control bytes per word
  static_assert(offsetof(MsParams, cbit) % 8 == 0, "cbit words must be 8-byte aligned");
  static_assert(MS_MAX == 128, "four ballot chunks");
  uint32_t M0 = 0, M1 = 0, M2 = 0, M3 = 0, L0 = 0, L1 = 0, L2 = 0, L3 = 0;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    if (32 * h >= P.ngates) break;
    const bool valid = 32 * h + lane < P.ngates;
    // four uniform word loads and a select instead of 32 divergent constant loads
    const uint64_t w0 = cw[4 * h], w1 = cw[4 * h + 1], w2 = cw[4 * h + 2], w3 = cw[4 * h + 3];
    const int sel = lane >> 3;
    const uint64_t w = sel == 0 ? w0 : sel == 1 ? w1 : sel == 2 ? w2 : w3;
    const unsigned c = (unsigned)(w >> ((lane & 7) * 8)) & 0xFFu;
    const bool mem = valid && c != 0xFFu;
    const bool dep = mem && ((vary >> c) & 1ull);
    const uint32_t mb = __ballot_sync(0xffffffffu, valid && (!mem || dep || ((base >> c) & 1ull)));
    const uint32_t lb = __ballot_sync(0xffffffffu, dep);
    if (h == 0) M0 = mb, L0 = lb;
    if (h == 1) M1 = mb, L1 = lb;
    if (h == 2) M2 = mb, L2 = lb;
    if (h == 3) M3 = mb, L3 = lb;
  }
  if (XF) {
    static_assert(MS_K == 4, "compiled stage groups assume four slots");
    const uint32_t M[4] = {M0, M1, M2, M3}, L[4] = {L0, L1, L2, L3};
    if (X.inverse) {
      xm_slot_inv<0>(r, base, P, X, M, L);
      xm_slot_inv<1>(r, base, P, X, M, L);
      xm_slot_inv<2>(r, base, P, X, M, L);
      xm_slot_inv<3>(r, base, P, X, M, L);
      return;
    }
    xm_slot<3>(r, base, P, X, M, L);
    xm_slot<2>(r, base, P, X, M, L);
    xm_slot<1>(r, base, P, X, M, L);
    xm_slot<0>(r, base, P, X, M, L);
    return;
  }
  for (int ri = 0; ri < P.nruns; ++ri) {
    const MsRun R = P.run[ri];
    const uint32_t range = R.range;
    const uint32_t mh = R.h == 0 ? M0 : R.h == 1 ? M1 : R.h == 2 ? M2 : M3;
    const uint32_t lh = R.h == 0 ? L0 : R.h == 1 ? L1 : R.h == 2 ? L2 : L3;
    const uint32_t act = mh & range;
    if (act) ms_dispatch(R.code, r, act, lh & range, 32 * R.h, base, P);
  }
}

template <int S>
__device__ __forceinline__ void ms_exact(double2 (&r)[MS_N], int cs, const double *q) {
#pragma unroll
  for (int j = 0; j < MS_N; ++j) {
    if ((j >> S) & 1) continue;
    if (cs < MS_K && !((j >> cs) & 1)) continue;
    pair_update<KIND_GENERAL>(r[j], r[j | (1 << S)], q);  // the definition itself
  }
}

// All-zero groups (basis states and the sparse early stages of their transforms) through a
// whole pass on SIGN BITS: zeros stay zeros under mix(), and the IEEE sign of each result
// is a boolean function of the operands' signs -- a product of zeros has the XOR of the
// signs, a round-to-nearest sum (or fma addend) of two zeros is -0 only if both are.  With
// the 16 real and 16 imaginary signs of the group packed in two words, cmul(r, x) of every
// pair at once is re = (r.re ^ x.re) & ~(x.im ^ r.im), im = (r.re ^ x.im) & (x.re ^ r.im)
// (cmul's fma(rr, x.re, -(x.im * ri)) and fma(rr, x.im, x.re * ri)), and mix() ANDs two of
// them: ~25 integer ops per gate instead of 160 FP64 ops, bit-identical to mix().
__device__ __forceinline__ uint32_t sgn_mask(double v) { return signbit(v) ? 0xFFFFu : 0u; }

__device__ __noinline__ void ms_replay_zero(double2 *__restrict__ a, uint64_t base, const MsParams *P,
                                            const uint64_t (&b)[MS_K], uint32_t sre, uint32_t sim) {
  for (int gi = 0; gi < P->ngates; ++gi) {
    const int c = P->cbit[gi];
    if (c != 0xFF && !((base >> c) & 1ull)) continue;
    const int code = P->g[gi].code;
    const int cs = code % (MS_K + 1), s = (code / (MS_K + 1)) % MS_K;
    const double *q = P->g[gi].q;
    // pairs (j, j | 1<<s) with bit s of j clear (and bit cs set for a slot control)
    uint32_t m0 = 0;
#pragma unroll
    for (int j = 0; j < MS_N; ++j)
      if (!((j >> s) & 1) && (cs >= MS_K || ((j >> cs) & 1))) m0 |= 1u << j;
    const int sh = 1 << s;
    const uint32_t a0r = sre & m0, a0i = sim & m0, a1r = (sre >> sh) & m0, a1i = (sim >> sh) & m0;
    auto cm_re = [&](int k, uint32_t xr, uint32_t xi) {
      return (sgn_mask(q[2 * k]) ^ xr) & ~(xi ^ sgn_mask(q[2 * k + 1])) & m0;
    };
    auto cm_im = [&](int k, uint32_t xr, uint32_t xi) {
      return (sgn_mask(q[2 * k]) ^ xi) & (xr ^ sgn_mask(q[2 * k + 1])) & m0;
    };
    const uint32_t n0r = cm_re(0, a0r, a0i) & cm_re(1, a1r, a1i), n0i = cm_im(0, a0r, a0i) & cm_im(1, a1r, a1i);
    const uint32_t n1r = cm_re(2, a0r, a0i) & cm_re(3, a1r, a1i), n1i = cm_im(2, a0r, a0i) & cm_im(3, a1r, a1i);
    const uint32_t keep = ~(m0 | (m0 << sh));
    sre = (sre & keep) | n0r | (n1r << sh);
    sim = (sim & keep) | n0i | (n1i << sh);
  }
#pragma unroll
  for (int j = 0; j < MS_N; ++j)
    a[base | ms_off(j, b)] = make_double2((sre >> j) & 1u ? -0.0 : 0.0, (sim >> j) & 1u ? -0.0 : 0.0);
}

// Exact replay of one thread's group from global memory (nothing stored yet).
__device__ __noinline__ void ms_replay(double2 *__restrict__ a, uint64_t base, const MsParams *P) {
  uint64_t b[MS_K];
#pragma unroll
  for (int s = 0; s < MS_K; ++s) b[s] = 1ull << P->bits[s];
  double2 r[MS_N];
#pragma unroll
  for (int j = 0; j < MS_N; ++j) r[j] = a[base | ms_off(j, b)];
  bool allzero = true;
  uint32_t sre = 0, sim = 0;
#pragma unroll
  for (int j = 0; j < MS_N; ++j) {
    allzero &= ((__double2hiint(r[j].x) & 0x7fffffff) | __double2loint(r[j].x) |
                (__double2hiint(r[j].y) & 0x7fffffff) | __double2loint(r[j].y)) == 0;
    sre |= (signbit(r[j].x) ? 1u : 0u) << j;
    sim |= (signbit(r[j].y) ? 1u : 0u) << j;
  }
  if (allzero) {
    ms_replay_zero(a, base, P, b, sre, sim);
    return;
  }
  for (int gi = 0; gi < P->ngates; ++gi) {
    const int c = P->cbit[gi];
    if (c != 0xFF && !((base >> c) & 1ull)) continue;
    const int code = P->g[gi].code;
    const int cs = code % (MS_K + 1), s = (code / (MS_K + 1)) % MS_K;
    if (s == 0)
      ms_exact<0>(r, cs, P->g[gi].q);
    else if (s == 1)
      ms_exact<1>(r, cs, P->g[gi].q);
    else if (MS_K == 3 || s == 2)
      ms_exact<2>(r, cs, P->g[gi].q);
    else
      ms_exact<MS_K - 1>(r, cs, P->g[gi].q);
  }
#pragma unroll
  for (int j = 0; j < MS_N; ++j) a[base | ms_off(j, b)] = r[j];
}


// Async 16-B global -> shared copies (L2 only): the next group streams in while this one computes.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

#ifndef SV_MS_THREADS
#define SV_MS_THREADS (SV_MS_MINB * 256)  // resident threads per SM the register budget must allow
#endif
#ifndef SV_MS_BLK_XF
#define SV_MS_BLK_XF 128  // CTA size of the compiled variant: 128 / 256 -> QFT(30) 55.0 / 56.2 ms (same box)
#endif
template <bool XF>
constexpr int ms_blk() { return XF ? SV_MS_BLK_XF : MS_BLK; }
template <bool XF>
__global__ void __launch_bounds__(ms_blk<XF>(), SV_MS_THREADS / ms_blk<XF>()) k_mstage(
    double2 *__restrict__ a, uint64_t ngroups, const __grid_constant__ MsParams P,
    const __grid_constant__ XmParams X) {
  const uint64_t p = (uint64_t)blockIdx.x * ms_blk<XF>() + threadIdx.x;
  uint64_t b[MS_K], base = p;
#pragma unroll
  for (int s = 0; s < MS_K; ++s) b[s] = 1ull << P.bits[s];
#if SV_MS_HILANE
  if (P.hl[0] >= 0) {
    // lanes 0..2 on slice bits 0..2 (128-B runs), lanes 3, 4 on two high bits that no gate of the
    // group is controlled by: fewer lane-dependent controls (a lane-dependent gate costs double)
    base = (p & 7ull) | ((p >> 5) << 3);
    for (int i = 0; i < P.nins; ++i) base = insert_zero(base, P.ins[i]);
    base |= (((p >> 3) & 1ull) << P.hl[0]) | (((p >> 4) & 1ull) << P.hl[1]);
  } else
#endif
  {
#pragma unroll
    for (int s = 0; s < MS_K; ++s) base = insert_zero(base, P.bits[s]);
  }
  const bool live = p < ngroups;
  double2 r[MS_N];
#pragma unroll
  for (int j = 0; j < MS_N; ++j) r[j] = live ? a[base | ms_off(j, b)] : make_double2(1.0, 1.0);
  ms_run<XF>(r, base, P, X);
  bool ok = true;
#pragma unroll
  for (int j = 0; j < MS_N; ++j) ok &= nonzero2(r[j]);
  if (!live) return;
  if (__builtin_expect(!ok, 0)) {
    ms_replay(a, base, &P);
    return;
  }
#pragma unroll
  for (int j = 0; j < MS_N; ++j) a[base | ms_off(j, b)] = r[j];
}

// ------------------------------------- tolerance-mode stage passes (FusionConfig exact=False)
//
// The same thread layout as k_mstage (16 amplitudes spanning four slot bits,
// every other index bit fixed per thread), but the gate list is compiled on the
// host into a program that no longer reproduces mix()'s rounding sequence,
// only its value (north_star: fused gates checked under max-abs <= 1e-12 sqrt(G)):
//   fold   a diagonal gate on slot s whose control is not a slot (or absent):
//          for a thread it means "multiply every amplitude with slot bit s = 1
//          by d1 (= 0: by d0)" when the thread's own control bit is set.  The
//          consecutive folds of one slot (a transform stage's R(k, c) for every
//          c outside the pass) form a fold group whose product is a function of
//          the thread's index bits only; k_dtable tabulates it per index byte
//          (256 products per byte, built once per launch), so the group costs a
//          thread one table load and one complex multiply per index byte.
//   GATE   any other gate (general / real / Hadamard-like updates, diagonal
//          gates controlled by another slot): in registers, as in k_mstage.
//   FLUSH  multiply slot s's amplitudes by their fold group's product; emitted
//          before the next non-diagonal gate whose target is s (a factor that
//          depends only on bit s and the fixed bits commutes with every gate
//          that does not target s) and at the end of the pass.
// No zero tests, no replay.

constexpr int DS_MAX = 256, DS_QMAX = 1280, DS_MAXG = 32;
enum { DS_GATE = 0, DS_FLUSH = 2 };

struct DsParams {
  int32_t nops, nbytes;   // nbytes: index bytes a fold table covers (ceil(m / 8))
  int32_t nfg;            // fold groups
  uint32_t has0;          // bit g: group g has a d0 != 1 factor (first 32 groups)
  double scale;           // product of the deferred butterfly factors (KIND_HBF)
  int32_t bits[MS_K];
  const double2 *tab;     // k_dtable output: per group [T1: nbytes x 256][T0: nbytes x 256]
  uint64_t hdr[DS_MAX];   // type 0-1 | slot 2-3 | cmode 4-5 (2: control on a non-slot bit) |
                          // flags 6 (FLUSH: apply T0 too) | cbit 8-13 | code / group 16-23 | q offset 32-63
  double q[DS_QMAX];
};

struct DtFold {
  int8_t group, c;  // c: control slice bit, -1 uncontrolled
  int16_t pad;
  int32_t pad2;
  double d[4];      // d0 re, im, d1 re, im
};

constexpr int DT_MAXF = 2 * MS_MAX;  // folded gates per launch (two phases of k_dstage2)

struct DtParams {
  int32_t nfold, nbytes;
  double2 *tab;
  DtFold f[DT_MAXF];
};

// One block per (group, index byte, table kind); thread v = the byte's value.
__global__ void __launch_bounds__(256) k_dtable(const __grid_constant__ DtParams P) {
  const int g = blockIdx.x / (2 * P.nbytes), k = (blockIdx.x / 2) % P.nbytes, one = (blockIdx.x & 1) == 0;
  const int v = threadIdx.x;
  double2 prod = make_double2(1.0, 0.0);
  for (int i = 0; i < P.nfold; ++i) {
    const DtFold &f = P.f[i];
    if (f.group != g) continue;
    const bool act = f.c < 0 ? k == 0 : ((f.c >> 3) == k && ((v >> (f.c & 7)) & 1));
    if (act) prod = cmul(one ? f.d[2] : f.d[0], one ? f.d[3] : f.d[1], prod);
  }
  P.tab[((size_t)(g * 2 + (one ? 0 : 1)) * P.nbytes + k) * 256 + v] = prod;
}

__device__ __forceinline__ double2 cmul2(double2 f, double2 a) { return cmul(f.x, f.y, a); }

template <int NB>
__device__ __forceinline__ double2 ds_factor(const double2 *__restrict__ t, uint64_t base) {
  double2 e[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) e[k] = t[k * 256 + ((base >> (8 * k)) & 255u)];  // all loads first
  double2 f = e[0];
#pragma unroll
  for (int k = 1; k < NB; ++k) f = cmul2(e[k], f);
  return f;
}

template <int S>
__device__ __forceinline__ void ds_flush(double2 (&r)[MS_N], double2 f1, double2 f0, bool do0) {
#pragma unroll
  for (int j = 0; j < MS_N; ++j) {
    if ((j >> S) & 1)
      r[j] = cmul2(f1, r[j]);
    else if (do0)
      r[j] = cmul2(f0, r[j]);
  }
}

__device__ __forceinline__ void ds_gate(int code, double2 (&r)[MS_N], const double *q) {
  switch (code) {
#define DS_CASE(K_, S_, C_)                       \
  case ((K_) * MS_K + (S_)) * (MS_K + 1) + (C_): \
    ms_apply<S_, C_, K_>(r, q);                   \
    break;
#if SV_MS_K == 3
#define DS_CASES_S(K_, S_) DS_CASE(K_, S_, 0) DS_CASE(K_, S_, 1) DS_CASE(K_, S_, 2) DS_CASE(K_, S_, 3)
#define DS_CASES(K_) DS_CASES_S(K_, 0) DS_CASES_S(K_, 1) DS_CASES_S(K_, 2)
#else
#define DS_CASES_S(K_, S_) \
  DS_CASE(K_, S_, 0) DS_CASE(K_, S_, 1) DS_CASE(K_, S_, 2) DS_CASE(K_, S_, 3) DS_CASE(K_, S_, 4)
#define DS_CASES(K_) DS_CASES_S(K_, 0) DS_CASES_S(K_, 1) DS_CASES_S(K_, 2) DS_CASES_S(K_, 3)
#endif
    DS_CASES(KIND_GENERAL) DS_CASES(KIND_DIAG) DS_CASES(KIND_PHASE) DS_CASES(KIND_REAL) DS_CASES(KIND_HSHARE)
    DS_CASES(KIND_HBF)
#undef DS_CASES
#undef DS_CASES_S
#undef DS_CASE
    default: break;
  }
}

#ifndef SV_DS_MINB
#define SV_DS_MINB 2  // 256-thread CTAs per SM
#endif
#ifndef SV_DS_GRAY
#define SV_DS_GRAY 1  // element addresses in Gray-code order (one XOR each)
#endif
#ifndef SV_DS_HBF
#define SV_DS_HBF 1  // uncontrolled Hadamard-like gates as unscaled butterflies, factor applied once
#endif

__device__ __forceinline__ uint64_t ds_base(uint64_t p, const int32_t (&bits)[MS_K]) {
  uint64_t base = p;
#pragma unroll
  for (int s = 0; s < MS_K; ++s) base = insert_zero(base, bits[s]);
  return base;
}

// Persistent: each thread walks groups p, p + stride, ...; group i+1's 16 amplitudes are copied
// into this thread's shared-memory slots (cp.async) while group i is updated in registers, so
// HBM reads stay in flight through the compute.  NB = index bytes of the fold tables.
template <int NB>
__global__ void __launch_bounds__(256, SV_DS_MINB) k_dstage(double2 *__restrict__ a, uint64_t ngroups,
                                                           const __grid_constant__ DsParams P) {
  extern __shared__ double2 stage_smem[];  // [MS_N][256]: this thread's slots are a column
  double2(*stage)[256] = reinterpret_cast<double2(*)[256]>(stage_smem);
  const int tid = threadIdx.x;
  uint64_t b[MS_K];
#pragma unroll
  for (int s = 0; s < MS_K; ++s) b[s] = 1ull << P.bits[s];
  const uint64_t stride = (uint64_t)gridDim.x * 256;
  uint64_t p = (uint64_t)blockIdx.x * 256 + tid;
  // the 16 elements of a group in Gray-code order: one XOR per address (base has zeros at the slots)
#define DS_GRAY(BASE, BODY)                                                                   \
  {                                                                                           \
    uint64_t ix = (BASE);                                                                     \
    _Pragma("unroll") for (int i = 0; i < MS_N; ++i) {                                        \
      const int j = i ^ (i >> 1);                                                             \
      if (SV_DS_GRAY) {                                                                       \
        if (i) ix ^= b[(i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : MS_K - 1];                    \
      } else {                                                                                \
        ix = (BASE) | ms_off(j, b);                                                           \
      }                                                                                       \
      BODY;                                                                                   \
    }                                                                                         \
  }
  if (p < ngroups) DS_GRAY(ds_base(p, P.bits), cp_async16(&stage[j][tid], a + ix));
  cp_async_commit();
  const int nb = NB;
  for (; p < ngroups; p += stride) {
    const uint64_t base = ds_base(p, P.bits);
    double2 r[MS_N];
    cp_async_wait_all();
#pragma unroll
    for (int j = 0; j < MS_N; ++j) r[j] = stage[j][tid];
    const uint64_t pn = p + stride;
    if (pn < ngroups) DS_GRAY(ds_base(pn, P.bits), cp_async16(&stage[j][tid], a + ix));
    cp_async_commit();
    for (int i = 0; i < P.nops; ++i) {
      const uint64_t h = P.hdr[i];
      const int s = (int)((h >> 2) & 3u);
      if ((h & 3u) == DS_FLUSH) {
        const double2 *t = P.tab + (size_t)((h >> 16) & 0xffu) * 2 * nb * 256;
        const bool do0 = (h >> 6) & 1u;
        const double2 f1 = ds_factor<NB>(t, base);
        const double2 f0 = do0 ? ds_factor<NB>(t + nb * 256, base) : make_double2(1.0, 0.0);
        switch (s) {
          case 0: ds_flush<0>(r, f1, f0, do0); break;
          case 1: ds_flush<1>(r, f1, f0, do0); break;
          case 2: ds_flush<2>(r, f1, f0, do0); break;
          default: ds_flush<MS_K - 1>(r, f1, f0, do0); break;
        }
        continue;
      }
      if (((h >> 4) & 3u) == 2u && !((base >> ((h >> 8) & 63u)) & 1ull)) continue;  // control clear here
      ds_gate((int)((h >> 16) & 0xffu), r, P.q + (h >> 32));
    }
    if (P.scale != 1.0) {  // the deferred Hadamard factors
      const double sc = P.scale;
#pragma unroll
      for (int j = 0; j < MS_N; ++j) r[j] = make_double2(r[j].x * sc, r[j].y * sc);
    }
    DS_GRAY(base, a[ix] = r[j]);
  }
#undef DS_GRAY
  cp_async_wait_all();
}

// ----------------------- two-phase tolerance stage passes: eight stage targets per HBM pass
//
// k_dstage2: one CTA per 4096-amplitude tile spanning four coalescing low bits L, four
// targets S1 and four targets S2.  Phase 1 holds, per thread, the 16 elements over S1
// (thread bits = L and S2) and runs the S1 program; a shared-memory transpose gives each
// thread the 16 elements over S2 (thread bits = L and S1) for the S2 program; the tile is
// stored.  Each phase is a k_dstage program (folds, GATE, FLUSH ops) -- a fold group of
// phase 1 may depend on S2 bits because every phase-1 group is flushed before the
// transpose.  Eight transform stages per pass instead of four.

constexpr int DS2_MAX = 3 * MS_MAX / 2 + MS_K, DS2_QMAX = 8 * MS_MAX;  // every gate of a phase fits

struct Ds2Params {
  int32_t nops[2], nbytes, pad;
  int32_t s1[MS_K], s2[MS_K], lb[MS_K];  // phase-1 slots, phase-2 slots, coalescing low bits
  int32_t tb[3 * MS_K];                   // all twelve tile bits, ascending
  double scale;
  const double2 *tab;
  uint64_t hdr[2][DS2_MAX];
  double q[2][DS2_QMAX];
};

template <int NB>
__device__ __forceinline__ void ds_exec(double2 (&r)[MS_N], uint64_t base, const uint64_t *hdr, int nops,
                                        const double *qv, const double2 *tab) {
  for (int i = 0; i < nops; ++i) {
    const uint64_t h = hdr[i];
    const int s = (int)((h >> 2) & 3u);
    if ((h & 3u) == DS_FLUSH) {
      const double2 *t = tab + (size_t)((h >> 16) & 0xffu) * 2 * NB * 256;
      const bool do0 = (h >> 6) & 1u;
      const double2 f1 = ds_factor<NB>(t, base);
      const double2 f0 = do0 ? ds_factor<NB>(t + NB * 256, base) : make_double2(1.0, 0.0);
      switch (s) {
        case 0: ds_flush<0>(r, f1, f0, do0); break;
        case 1: ds_flush<1>(r, f1, f0, do0); break;
        case 2: ds_flush<2>(r, f1, f0, do0); break;
        default: ds_flush<MS_K - 1>(r, f1, f0, do0); break;
      }
      continue;
    }
    if (((h >> 4) & 3u) == 2u && !((base >> ((h >> 8) & 63u)) & 1ull)) continue;  // control clear here
    ds_gate((int)((h >> 16) & 0xffu), r, qv + (h >> 32));
  }
}

__device__ __forceinline__ uint64_t spread4(int v, const int32_t (&bits)[MS_K]) {
  uint64_t x = 0;
#pragma unroll
  for (int k = 0; k < MS_K; ++k) x |= (uint64_t)((v >> k) & 1) << bits[k];
  return x;
}

#ifndef SV_DS2_MINB
#define SV_DS2_MINB 2
#endif

// Persistent; the tile buffer doubles as the prefetch buffer: once phase 2 has its registers,
// the next tile's phase-1 elements stream into it (cp.async, each thread its own column)
// while phase 2 computes and stores.  PT carries the tile geometry (s1, s2, lb, tb, scale);
// F1 / F2 run the two phases on a thread's 16 registers.
// (A variant with a separate 64 KiB prefetch buffer and a half-tile transpose buffer shared by the
// CTA's even and odd warps through named barriers -- the next tile in flight during the whole of
// this one -- measured slower: QFT(30) compiled passes 9.1-9.4 ms vs 6.7-7.2 ms; removed.)
constexpr int DS2_SMEM = 4096 * (int)sizeof(double2);

template <class PT, class F1, class F2>
__device__ __forceinline__ void ds2_tiles(double2 *__restrict__ a, uint64_t ntiles, const PT &P, double2 *tile,
                                          F1 phase1, F2 phase2) {
  const int t = threadIdx.x, lo = t & 15, hi = t >> 4;
  uint64_t b1[MS_K], b2[MS_K];
#pragma unroll
  for (int k = 0; k < MS_K; ++k) b1[k] = 1ull << P.s1[k], b2[k] = 1ull << P.s2[k];
  const uint64_t lpart = spread4(lo, P.lb);
  const uint64_t part1 = lpart | spread4(hi, P.s2), part2 = lpart | spread4(hi, P.s1);
  auto cta_base = [&](uint64_t id) {
    uint64_t cta = id;
#pragma unroll
    for (int k = 0; k < 3 * MS_K; ++k) cta = insert_zero(cta, P.tb[k]);
    return cta;
  };
  uint64_t id = blockIdx.x;
  if (id < ntiles) {
    const uint64_t cta0 = cta_base(id);
#pragma unroll
    for (int j = 0; j < MS_N; ++j) cp_async16(&tile[j * 256 + t], a + (cta0 | part1 | ms_off(j, b1)));
  }
  cp_async_commit();
  for (; id < ntiles; id += gridDim.x) {
    // the tile base is recomputed here and for the prefetch below rather than carried: carried,
    // ptxas spills it and every warp waits ~12 % of its time on the reload before the stores
    const uint64_t cta = cta_base(id);
    const uint64_t base1 = cta | part1, base2 = cta | part2;
    // a phase's per-thread factors are fetched while its registers are not live yet (the
    // prefetched column still in flight; the tile in shared memory between the transposes)
    typename F1::Prep f1;
    phase1.prep(base1, f1);
    double2 r[MS_N];
    cp_async_wait_all();
#pragma unroll
    for (int j = 0; j < MS_N; ++j) r[j] = tile[j * 256 + t];
    phase1.run(r, base1, f1);
    __syncthreads();  // every thread has its prefetched column
#pragma unroll
    for (int j = 0; j < MS_N; ++j) tile[lo | (j << 4) | (hi << 8)] = r[j];
    typename F2::Prep f2;
    phase2.prep(base2, f2);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < MS_N; ++j) r[j] = tile[lo | (hi << 4) | (j << 8)];
    __syncthreads();  // the transpose is read: the buffer takes the next tile
    const uint64_t nid = id + gridDim.x;
    if (nid < ntiles) {
      const uint64_t ncta = cta_base(nid);
#pragma unroll
      for (int j = 0; j < MS_N; ++j) cp_async16(&tile[j * 256 + t], a + (ncta | part1 | ms_off(j, b1)));
    }
    cp_async_commit();
    phase2.run(r, base2, f2);
    if (P.scale != 1.0) {
      const double sc = P.scale;
#pragma unroll
      for (int j = 0; j < MS_N; ++j) r[j] = make_double2(r[j].x * sc, r[j].y * sc);
    }
#pragma unroll
    for (int j = 0; j < MS_N; ++j) a[base2 | ms_off(j, b2)] = r[j];
  }
  cp_async_wait_all();
}


// the interpreter as a ds2_tiles phase: nothing to prepare
template <int NB>
struct DsInterp {
  struct Prep {};
  const uint64_t *hdr;
  int nops;
  const double *qv;
  const double2 *tab;
  __device__ __forceinline__ void prep(uint64_t, Prep &) const {}
  __device__ __forceinline__ void run(double2 (&r)[MS_N], uint64_t base, const Prep &) const {
    ds_exec<NB>(r, base, hdr, nops, qv, tab);
  }
};

template <int NB>
__global__ void __launch_bounds__(256, SV_DS2_MINB) k_dstage2(double2 *__restrict__ a, uint64_t ntiles,
                                                             const __grid_constant__ Ds2Params P) {
  extern __shared__ double2 tile[];  // transpose: lo | s1 << 4 | s2 << 8; prefetch: j * 256 + thread
  ds2_tiles(a, ntiles, P, tile, DsInterp<NB>{P.hdr[0], P.nops[0], P.q[0], P.tab},
            DsInterp<NB>{P.hdr[1], P.nops[1], P.q[1], P.tab});
}

// ---------------------------------------------- compiled transform phases (tolerance mode)
//
// The op interpreter above pays a header load, a decode and a branch tree per op -- about as
// many issue slots as the FP64 work of a transform pass, and long dependent latencies with 16
// warps per SM.  A phase whose gate list has the shape of transform stages,
//   forward:  for slots s descending   [butterfly on s]  then  phases on s (controls: lower slots or non-slots)
//   inverse:  for slots s ascending    phases on s (same controls)  then  [butterfly on s]
// (the stages of the reference's build_qft / its inverse, circuits.py:141-156) runs as straight-line
// code instead: per slot one butterfly over the 8 pairs and ONE complex factor per amplitude with
// the slot bit set -- fold-table product (controls outside the slots) times the host-multiplied
// product of the in-slot phases, indexed by the amplitude's lower slot bits.
struct XfPhase {
  int32_t hmask;  // bit s: slot s has its Hadamard-like butterfly
  int32_t fmask;  // bit s: slot s has a fold group, group[s]
  int32_t pmask;  // bit s: slot s has in-slot controlled phases, phw[s][1 .. 2^s - 1]
  int32_t pad;
  int32_t group[MS_K];
  double2 phw[MS_K][MS_N / 2];  // phw[s][k]: product of slot s's phases whose control slots are the set bits of k
};

struct Xf2Params {
  int32_t nbytes, pad;
  int32_t s1[MS_K], s2[MS_K], lb[MS_K];
  int32_t tb[3 * MS_K];
  double scale;
  const double2 *tab;
  XfPhase ph[2];
};

template <int S>
__device__ __forceinline__ void xf_bfly(double2 (&r)[MS_N]) {
#pragma unroll
  for (int j = 0; j < MS_N; ++j) {
    if ((j >> S) & 1) continue;
    spec_pair<KIND_HBF>(r[j], r[j | (1 << S)], nullptr);
  }
}

// r[j] *= f * phw[S][j's lower slot bits] for every j with bit S set.  FULL: the slot has a fold
// factor and (S > 0) in-slot phases -- no tests, no selects.
template <int S, bool FULL>
__device__ __forceinline__ void xf_diag(double2 (&r)[MS_N], const XfPhase &X, double2 f) {
  constexpr int NK = 1 << S;
  const bool hasf = FULL || ((X.fmask >> S) & 1), hasp = FULL ? S > 0 : ((X.pmask >> S) & 1);
  if (!hasp) {
    if (!hasf) return;
#pragma unroll
    for (int j = 0; j < MS_N; ++j)
      if ((j >> S) & 1) r[j] = cmul2(f, r[j]);
    return;
  }
  double2 w[NK];
  w[0] = f;
#pragma unroll
  for (int k = 1; k < NK; ++k) w[k] = hasf ? cmul2(f, X.phw[S][k]) : X.phw[S][k];
#pragma unroll
  for (int j = 0; j < MS_N; ++j) {
    if (!((j >> S) & 1)) continue;
    const int k = j & (NK - 1);
    if (k == 0) {
      if (hasf) r[j] = cmul2(w[0], r[j]);
    } else {
      r[j] = cmul2(w[k], r[j]);
    }
  }
}

template <int S, bool INV, bool FULL>
__device__ __forceinline__ void xf_slot(double2 (&r)[MS_N], const XfPhase &X, double2 f) {
  if (INV) xf_diag<S, FULL>(r, X, f);
  if (FULL || ((X.hmask >> S) & 1)) xf_bfly<S>(r);
  if (!INV) xf_diag<S, FULL>(r, X, f);
}

// A compiled transform phase as a ds2_tiles phase.  prep: the four slots' fold factors (table
// loads, then their products); run: the straight-line slot updates.
template <int NB, bool INV, bool FULL>
struct XfRun {
  struct Prep {
    double2 f[MS_K];
  };
  const XfPhase &X;
  const double2 *__restrict__ tab;
  __device__ __forceinline__ void prep(uint64_t base, Prep &p) const {
    static_assert(MS_K == 4, "compiled transform phases assume four slots");
    double2 e[MS_K][NB];
#pragma unroll
    for (int s = 0; s < MS_K; ++s) {
      const bool hasf = FULL || ((X.fmask >> s) & 1);
      const double2 *t = tab + (size_t)(hasf ? X.group[s] : 0) * 2 * NB * 256;
#pragma unroll
      for (int k = 0; k < NB; ++k) e[s][k] = hasf ? t[k * 256 + ((base >> (8 * k)) & 255u)] : make_double2(1.0, 0.0);
    }
#pragma unroll
    for (int s = 0; s < MS_K; ++s) {
      p.f[s] = e[s][0];
      if (FULL || ((X.fmask >> s) & 1)) {
#pragma unroll
        for (int k = 1; k < NB; ++k) p.f[s] = cmul2(e[s][k], p.f[s]);
      }
    }
  }
  __device__ __forceinline__ void run(double2 (&r)[MS_N], uint64_t, const Prep &p) const {
    if (!INV) {
      xf_slot<3, false, FULL>(r, X, p.f[3]);
      xf_slot<2, false, FULL>(r, X, p.f[2]);
      xf_slot<1, false, FULL>(r, X, p.f[1]);
      xf_slot<0, false, FULL>(r, X, p.f[0]);
    } else {
      xf_slot<0, true, FULL>(r, X, p.f[0]);
      xf_slot<1, true, FULL>(r, X, p.f[1]);
      xf_slot<2, true, FULL>(r, X, p.f[2]);
      xf_slot<3, true, FULL>(r, X, p.f[3]);
    }
  }
};

// FULL: both phases have every butterfly, every fold group and every in-slot phase set (the
// bulk passes of a transform); otherwise the masks are tested.
template <int NB, bool INV, bool FULL>
__global__ void __launch_bounds__(256, SV_DS2_MINB) k_xstage2(double2 *__restrict__ a, uint64_t ntiles,
                                                             const __grid_constant__ Xf2Params P) {
  extern __shared__ double2 tile[];
  ds2_tiles(a, ntiles, P, tile, XfRun<NB, INV, FULL>{P.ph[0], P.tab}, XfRun<NB, INV, FULL>{P.ph[1], P.tab});
}

// The single-phase form (a tolerance stage group of at most four targets shaped like transform
// stages): k_dstage's persistent, column-prefetching skeleton around one compiled phase.
struct Xf1Params {
  int32_t nbytes, pad;
  int32_t bits[MS_K];
  double scale;
  const double2 *tab;
  XfPhase ph;
};

template <int NB, bool INV>
__global__ void __launch_bounds__(256, SV_DS_MINB) k_xstage(double2 *__restrict__ a, uint64_t ngroups,
                                                           const __grid_constant__ Xf1Params P) {
  extern __shared__ double2 stage_smem[];  // [MS_N][256]: this thread's slots are a column
  double2(*stage)[256] = reinterpret_cast<double2(*)[256]>(stage_smem);
  const int tid = threadIdx.x;
  uint64_t b[MS_K];
#pragma unroll
  for (int s = 0; s < MS_K; ++s) b[s] = 1ull << P.bits[s];
  const uint64_t stride = (uint64_t)gridDim.x * 256;
  uint64_t p = (uint64_t)blockIdx.x * 256 + tid;
  const XfRun<NB, INV, false> phase{P.ph, P.tab};
  if (p < ngroups) {
    const uint64_t base = ds_base(p, P.bits);
#pragma unroll
    for (int j = 0; j < MS_N; ++j) cp_async16(&stage[j][tid], a + (base | ms_off(j, b)));
  }
  cp_async_commit();
  for (; p < ngroups; p += stride) {
    const uint64_t base = ds_base(p, P.bits);
    typename XfRun<NB, INV, false>::Prep f;
    phase.prep(base, f);
    double2 r[MS_N];
    cp_async_wait_all();
#pragma unroll
    for (int j = 0; j < MS_N; ++j) r[j] = stage[j][tid];
    const uint64_t pn = p + stride;
    if (pn < ngroups) {
      const uint64_t nbase = ds_base(pn, P.bits);
#pragma unroll
      for (int j = 0; j < MS_N; ++j) cp_async16(&stage[j][tid], a + (nbase | ms_off(j, b)));
    }
    cp_async_commit();
    phase.run(r, base, f);
    if (P.scale != 1.0) {
      const double sc = P.scale;
#pragma unroll
      for (int j = 0; j < MS_N; ++j) r[j] = make_double2(r[j].x * sc, r[j].y * sc);
    }
#pragma unroll
    for (int j = 0; j < MS_N; ++j) a[base | ms_off(j, b)] = r[j];
  }
  cp_async_wait_all();
}

// ------------------------------ tolerance-mode low-bit passes (targets in slice bits 0..5)
//
// One warp per 256-amplitude block (slice bits 0..7); each lane holds 8 elements in one of
// two layouts: H -- registers on bits 3, 4, 5, lanes on bits 0, 1, 2, 6, 7; L -- registers
// on bits 0, 1, 2, lanes on bits 3..7.  Every gate's target is a register bit of the
// current layout (the host inserts a layout switch -- a transpose through the warp's
// XOR-swizzled shared memory -- when needed), so updates never shuffle.  A run of diagonal
// gates whose target and control lie in bits 0..5 (a transform stage's R(k, c) for all
// c < k <= 5) is ONE 64-entry product table (built on the host): one complex multiply per
// element.  Uncontrolled Hadamard-like gates run as unscaled butterflies with their factor
// applied once at the end.  Controls: register bits -> pair predicates, lane bits (incl.
// 6, 7) -> lane predicates, bits >= 8 -> warp-uniform.  Values equal the reference's within
// rounding (FusionConfig exact=False).

constexpr int DL_BITS = 6, DL_MAX = 96, DL_TABMAX = 12;
enum { DL_GATE = 0, DL_TABLE = 1, DL_LAYOUT = 2, DL_STAGE = 3 };

struct DlParams {
  int32_t nops, ntab;
  double scale;  // deferred butterfly factors
  uint64_t hdr[2 * DL_MAX + DL_TABMAX];  // type 0-1 | register bit 2-3 | kind 4-7 | cmode 8-9 (0 none,
                                         // 1 register bit, 2 lane-or-above bit) | cbit 10-15 (register
                                         // bit or slice bit) | index 16-31 (gate, table; layout: 0 H, 1 L)
  double q[DL_MAX][8];
  double2 tab[DL_TABMAX][64];
  // DL_STAGE (a diagonal run of phase gates on ONE target that is a register bit): the factor of
  // an amplitude with the target bit set = stl[lane & 7] (controls on the layout's three lane
  // bits below bit 6, and the uncontrolled phases) * str[its other two register bits]
  int32_t nst, pad;
  double2 stl[DL_TABMAX][8];
  double2 str[DL_TABMAX][4];
  // exact mode, the tail of a transform (stages t = t0..0 of build_qft, circuits.py:141-156: H(t),
  // then R(t, c) for c = t-1..0): xq[t] = index in q[] of H(t) (-1: stage absent); the program
  // then runs as straight-line code (dl_xtail) and hdr[] only serves the exact replay
  int32_t compiled, pad2;
  int32_t xq[DL_BITS];
};

__device__ __forceinline__ int dl_x(int layout, int lane, int j) {  // slice bits 0..7 of (lane, reg j)
  return layout ? (j | (lane << 3)) : ((lane & 7) | (j << 3) | ((lane >> 3) << 6));
}
__device__ __forceinline__ int dl_swz(int x) { return x ^ ((x >> 3) & 7); }

template <int RB, int KIND>
__device__ __forceinline__ void dl_gate(double2 (&r)[8], uint32_t pm, const double *q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = ((k >> RB) << (RB + 1)) | (k & ((1 << RB) - 1));
    if ((pm >> j) & 1u) spec_pair<KIND>(r[j], r[j | (1 << RB)], q);
  }
}

template <int RB>
__device__ __forceinline__ void dl_gate_exact(double2 (&r)[8], uint32_t pm, const double *q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = ((k >> RB) << (RB + 1)) | (k & ((1 << RB) - 1));
    if ((pm >> j) & 1u) pair_update<KIND_GENERAL>(r[j], r[j | (1 << RB)], q);
  }
}

#ifndef SV_DL_PREFETCH
#define SV_DL_PREFETCH 0  // 1: the next block loads before this block's gates (the 32 extra registers spill at
// three CTAs per SM and cost a CTA at two: QFT(30) tail 7.17 ms; 0 with four CTAs per SM: 5.96 ms)
#endif

template <int LAYOUT>
__device__ __forceinline__ void dl_table(double2 (&r)[8], const double2 *__restrict__ t, int lane) {
  // tables are stored XOR-swizzled (entry x at dl_swz(x)): layout H reads x = (lane & 7) | (j << 3),
  // layout L x = ((lane & 7) << 3) | j; either way a quarter warp hits 8 distinct 16-B columns
  const int l7 = lane & 7;
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = cmul2(t[LAYOUT ? ((l7 << 3) | (j ^ l7)) : ((j << 3) | (l7 ^ j))], r[j]);
}

template <int FROM>
__device__ __forceinline__ void dl_transpose(double2 (&r)[8], double2 *buf, int lane) {
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) buf[dl_swz(dl_x(FROM, lane, j))] = r[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = buf[dl_swz(dl_x(1 - FROM, lane, j))];
}

// One stage's phases on register bit RB: eight table loads per lane (dl_table) become one.
template <int RB>
__device__ __forceinline__ void dl_stage(double2 (&r)[8], double2 lf, const double2 *__restrict__ rf) {
  double2 w[4];
  w[0] = lf;
#pragma unroll
  for (int k = 1; k < 4; ++k) w[k] = cmul2(lf, rf[k]);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (!((j >> RB) & 1)) continue;
    const int k = ((j >> (RB + 1)) << RB) | (j & ((1 << RB) - 1));  // j without bit RB
    r[j] = cmul2(w[k], r[j]);
  }
}

// ---- the compiled exact transform tail (same updates as the interpreted exact program, in order)
template <int RB>
__device__ __forceinline__ void xl_h(double2 (&r)[8], const double *q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = ((k >> RB) << (RB + 1)) | (k & ((1 << RB) - 1));
    spec_pair<KIND_HSHARE>(r[j], r[j | (1 << RB)], q);
  }
}
// phase on register bit RB controlled by register bit CB / by a lane predicate
template <int RB, int CB>
__device__ __forceinline__ void xl_ph_reg(double2 (&r)[8], const double *q) {
  const double qr = q[6], qi = q[7];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (((j >> RB) & 1) && ((j >> CB) & 1)) r[j] = cmul(qr, qi, r[j]);
}
template <int RB>
__device__ __forceinline__ void xl_ph_lane(double2 (&r)[8], const double *q, bool on) {
  if (!on) return;
  const double qr = q[6], qi = q[7];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if ((j >> RB) & 1) r[j] = cmul(qr, qi, r[j]);
}

__device__ __forceinline__ int dl_xtail(double2 (&r)[8], const DlParams &P, double2 *buf, int lane) {
  const bool l2 = lane & 4, l1 = lane & 2, l0 = lane & 1;  // slice bits 2, 1, 0 in layout H
  if (P.xq[5] >= 0) {
    const int g = P.xq[5];
    xl_h<2>(r, P.q[g]);
    xl_ph_reg<2, 1>(r, P.q[g + 1]);
    xl_ph_reg<2, 0>(r, P.q[g + 2]);
    xl_ph_lane<2>(r, P.q[g + 3], l2);
    xl_ph_lane<2>(r, P.q[g + 4], l1);
    xl_ph_lane<2>(r, P.q[g + 5], l0);
  }
  if (P.xq[4] >= 0) {
    const int g = P.xq[4];
    xl_h<1>(r, P.q[g]);
    xl_ph_reg<1, 0>(r, P.q[g + 1]);
    xl_ph_lane<1>(r, P.q[g + 2], l2);
    xl_ph_lane<1>(r, P.q[g + 3], l1);
    xl_ph_lane<1>(r, P.q[g + 4], l0);
  }
  if (P.xq[3] >= 0) {
    const int g = P.xq[3];
    xl_h<0>(r, P.q[g]);
    xl_ph_lane<0>(r, P.q[g + 1], l2);
    xl_ph_lane<0>(r, P.q[g + 2], l1);
    xl_ph_lane<0>(r, P.q[g + 3], l0);
  }
  if (P.xq[2] < 0 && P.xq[1] < 0 && P.xq[0] < 0) return 0;
  dl_transpose<0>(r, buf, lane);  // registers on slice bits 0, 1, 2
  if (P.xq[2] >= 0) {
    const int g = P.xq[2];
    xl_h<2>(r, P.q[g]);
    xl_ph_reg<2, 1>(r, P.q[g + 1]);
    xl_ph_reg<2, 0>(r, P.q[g + 2]);
  }
  if (P.xq[1] >= 0) {
    const int g = P.xq[1];
    xl_h<1>(r, P.q[g]);
    xl_ph_reg<1, 0>(r, P.q[g + 1]);
  }
  if (P.xq[0] >= 0) xl_h<0>(r, P.q[P.xq[0]]);
  return 1;
}

// The inverse tail: stages t = 0..t0, each [R(t, c) for c = 0..t-1, then the butterfly]; xq[t] = index of
// the stage's first gate.  Registers on bits 0, 1, 2 first, then on bits 3, 4, 5 (the store layout).
__device__ __forceinline__ int dl_xtail_inv(double2 (&r)[8], const DlParams &P, double2 *buf, int lane) {
  dl_transpose<0>(r, buf, lane);  // registers on slice bits 0, 1, 2
  if (P.xq[0] >= 0) xl_h<0>(r, P.q[P.xq[0]]);
  if (P.xq[1] >= 0) {
    const int g = P.xq[1];
    xl_ph_reg<1, 0>(r, P.q[g]);
    xl_h<1>(r, P.q[g + 1]);
  }
  if (P.xq[2] >= 0) {
    const int g = P.xq[2];
    xl_ph_reg<2, 0>(r, P.q[g]);
    xl_ph_reg<2, 1>(r, P.q[g + 1]);
    xl_h<2>(r, P.q[g + 2]);
  }
  if (P.xq[3] < 0 && P.xq[4] < 0 && P.xq[5] < 0) return 1;
  dl_transpose<1>(r, buf, lane);  // registers on slice bits 3, 4, 5
  const bool l2 = lane & 4, l1 = lane & 2, l0 = lane & 1;
  if (P.xq[3] >= 0) {
    const int g = P.xq[3];
    xl_ph_lane<0>(r, P.q[g], l0);
    xl_ph_lane<0>(r, P.q[g + 1], l1);
    xl_ph_lane<0>(r, P.q[g + 2], l2);
    xl_h<0>(r, P.q[g + 3]);
  }
  if (P.xq[4] >= 0) {
    const int g = P.xq[4];
    xl_ph_lane<1>(r, P.q[g], l0);
    xl_ph_lane<1>(r, P.q[g + 1], l1);
    xl_ph_lane<1>(r, P.q[g + 2], l2);
    xl_ph_reg<1, 0>(r, P.q[g + 3]);
    xl_h<1>(r, P.q[g + 4]);
  }
  if (P.xq[5] >= 0) {
    const int g = P.xq[5];
    xl_ph_lane<2>(r, P.q[g], l0);
    xl_ph_lane<2>(r, P.q[g + 1], l1);
    xl_ph_lane<2>(r, P.q[g + 2], l2);
    xl_ph_reg<2, 0>(r, P.q[g + 3]);
    xl_ph_reg<2, 1>(r, P.q[g + 4]);
    xl_h<2>(r, P.q[g + 5]);
  }
  return 0;
}

// The op program of one warp's block.  REPLAY: every gate through mix() itself (pair_update
// <KIND_GENERAL>), the exact pass of the bitwise mode; returns the final layout.
template <bool REPLAY>
__device__ __forceinline__ int dl_run(double2 (&r)[8], const DlParams &P, const double2 *tab, const double2 *stl,
                                      double2 *buf, int lane, uint64_t base) {
  int layout = 0;
  for (int i = 0; i < P.nops; ++i) {
    const uint64_t h = P.hdr[i];
    const int type = (int)(h & 3u), idx = (int)((h >> 16) & 0xffffu);
    if (type == DL_LAYOUT) {
      if (layout)
        dl_transpose<1>(r, buf, lane);
      else
        dl_transpose<0>(r, buf, lane);
      layout = idx;
      continue;
    }
    if (type == DL_TABLE) {
      if (REPLAY) continue;  // exact programs have no tables
      if (layout)
        dl_table<1>(r, tab + idx * 64, lane);
      else
        dl_table<0>(r, tab + idx * 64, lane);
      continue;
    }
    if (type == DL_STAGE) {
      if (REPLAY) continue;
      const double2 lf = stl[idx * 8 + (lane & 7)];
      const int rbt = (int)((h >> 2) & 3u);
      if (rbt == 0)
        dl_stage<0>(r, lf, P.str[idx]);
      else if (rbt == 1)
        dl_stage<1>(r, lf, P.str[idx]);
      else
        dl_stage<2>(r, lf, P.str[idx]);
      continue;
    }
    const int cmode = (int)((h >> 8) & 3u), cbit = (int)((h >> 10) & 63u);
    uint32_t pm = 0xffu;
    if (cmode == 1) {
      pm = cbit == 0 ? 0xAAu : cbit == 1 ? 0xCCu : 0xF0u;  // registers whose bit cbit is set
    } else if (cmode == 2) {
      const int x0 = dl_x(layout, lane, 0);  // this lane's bits; cbit is not a register bit here
      const bool on = cbit < 8 ? ((x0 >> cbit) & 1) : ((base >> cbit) & 1ull);
      if (!on) continue;
    }
    const double *q = P.q[idx];
    const int rb = (int)((h >> 2) & 3u), kind = (int)((h >> 4) & 15u);
    if (REPLAY) {
      if (rb == 0)
        dl_gate_exact<0>(r, pm, q);
      else if (rb == 1)
        dl_gate_exact<1>(r, pm, q);
      else
        dl_gate_exact<2>(r, pm, q);
      continue;
    }
    switch (rb * 8 + kind) {
#define DL_CASE(RB_, K_) \
  case (RB_)*8 + (K_): dl_gate<RB_, K_>(r, pm, q); break;
#define DL_KINDS(RB_) DL_CASE(RB_, KIND_GENERAL) DL_CASE(RB_, KIND_DIAG) DL_CASE(RB_, KIND_PHASE) \
  DL_CASE(RB_, KIND_REAL) DL_CASE(RB_, KIND_HSHARE) DL_CASE(RB_, KIND_HBF)
      DL_KINDS(0) DL_KINDS(1) DL_KINDS(2)
#undef DL_KINDS
#undef DL_CASE
      default: break;
    }
  }
  return layout;
}

#ifndef SV_DL_MINB
#define SV_DL_MINB 4
#endif
// EXACT (the bitwise mode: a program of GATE / LAYOUT ops only, no tables, no deferred factors):
// the structure-specialised updates differ from mix() only in the sign of a zero, so the warp tests
// its final block once and, on any zero component, reloads the block (nothing is stored yet) and
// replays the program through mix() -- the scheme of k_tile / k_mstage (see "speculative pair updates").
#ifndef SV_DL_MINB_EXACT
// CTAs per SM of the exact variant (it carries the replay): 4 / 3 / 2 -> 64 / 80 / 125 registers,
// 128 / 64 / 0 B of spills, QFT(30) tail 8.46 / 8.45 / 5.95 ms
#define SV_DL_MINB_EXACT 2
#endif
template <bool EXACT>
__global__ void __launch_bounds__(256, EXACT ? SV_DL_MINB_EXACT : SV_DL_MINB) k_dlow(double2 *__restrict__ a, uint64_t nblocks,
                                                         const __grid_constant__ DlParams P) {
  __shared__ double2 tab[DL_TABMAX * 64];
  __shared__ double2 xp[8][256];  // one 4 KiB transpose buffer per warp
  __shared__ double2 stl[DL_TABMAX * 8];
  for (int i = threadIdx.x; i < P.ntab * 64; i += 256) tab[(i & ~63) | dl_swz(i & 63)] = P.tab[i >> 6][i & 63];
  for (int i = threadIdx.x; i < P.nst * 8; i += 256) stl[i] = P.stl[i >> 3][i & 7];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 *buf = xp[w];
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  uint64_t blk = (uint64_t)blockIdx.x * 8 + w;
  if (blk >= nblocks) return;
#if SV_DL_PREFETCH
  double2 nx[8];  // the next block's elements, loaded before this block's gates
#pragma unroll
  for (int j = 0; j < 8; ++j) nx[j] = a[(blk << 8) + dl_x(0, lane, j)];
#endif
  for (; blk < nblocks; blk += nw) {
    const uint64_t base = blk << 8;
    double2 r[8];
#if SV_DL_PREFETCH
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = nx[j];
    if (blk + nw < nblocks) {
#pragma unroll
      for (int j = 0; j < 8; ++j) nx[j] = a[((blk + nw) << 8) + dl_x(0, lane, j)];
    }
#else
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[base + dl_x(0, lane, j)];
#endif
    int layout = !(EXACT && P.compiled) ? dl_run<false>(r, P, tab, stl, buf, lane, base)
                 : P.compiled == 2   ? dl_xtail_inv(r, P, buf, lane)
                                     : dl_xtail(r, P, buf, lane);
    if (EXACT) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 8; ++j) ok &= nonzero2(r[j]);
      if (__any_sync(0xffffffffu, !ok)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[base + dl_x(0, lane, j)];
        layout = dl_run<true>(r, P, tab, stl, buf, lane, base);
      }
    } else if (P.scale != 1.0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = make_double2(r[j].x * P.scale, r[j].y * P.scale);
    }
    if (layout) dl_transpose<1>(r, buf, lane);  // back to layout H for the store
#pragma unroll
    for (int j = 0; j < 8; ++j) a[base + dl_x(0, lane, j)] = r[j];
  }
}

// ------------------------------------------------ diagonal gates on a global qubit
//
// a diagonal gate (q12 = q21 = 0 exactly) on a global target
// needs no exchange -- the reference's pair update new0 = q11*a0 + q12*a1
// (distributed.py:187-202, mix() of kernels.py:120-124) is P = cmul(d, own)
// plus S = cmul(z, partner) with z a signed-zero matrix entry, and S is a
// signed zero: x + S == x for x != 0.  So each rank multiplies its own
// elements in place (P), and only where P has a zero component does the exact
// result depend on the partner -- through the SIGN BITS of the partner's
// original element alone.  k_diag_global therefore also writes a 2-bit-per-
// element sign map of its original elements (1/64 of the slice) and raises a
// flag when any P has a zero component; after a fence, k_diag_fix (a no-op
// unless the flag is up) re-forms P + S for exactly those elements from the
// partner's sign map, read through its CUDA-IPC mapping.  Bit-identical to
// the exchange, zero signs included; non-finite partner amplitudes (outside
// the normalised-state contract) are not propagated.
// Sign map layout: two 32-bit words per 32 consecutive elements, bit l of word
// 2w (2w+1) = sign of element 32w+l's real (imaginary) part.

__global__ void __launch_bounds__(BLK) k_diag_global(double2 *__restrict__ a, uint64_t n, int c, double dr,
                                                     double di, uint32_t *__restrict__ signs, int *flag) {
  // each warp takes DG consecutive 32-element groups per iteration, loads first (ILP)
  constexpr int DG = 4;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * BLK + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * BLK) >> 5;
  const uint64_t ngroups = (n + 31) >> 5;
  bool zero = false;
  for (uint64_t g0 = warp * DG; g0 < ngroups; g0 += nwarps * DG) {
    double2 x[DG];
    bool act[DG];
#pragma unroll
    for (int u = 0; u < DG; ++u) {
      const uint64_t i = ((g0 + u) << 5) + lane;
      act[u] = g0 + u < ngroups && i < n && (c < 0 || ((i >> c) & 1ull));
      x[u] = act[u] ? a[i] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < DG; ++u) {
      const uint64_t g = g0 + u;
      const uint32_t sre = __ballot_sync(0xffffffffu, act[u] && signbit(x[u].x));
      const uint32_t sim = __ballot_sync(0xffffffffu, act[u] && signbit(x[u].y));
      if (lane == 0 && g < ngroups && (c < 5 || (((g << 5) >> c) & 1ull))) {
        signs[2 * g] = sre;
        signs[2 * g + 1] = sim;
      }
      if (act[u]) {
        const double2 pv = cmul(dr, di, x[u]);
        zero |= !nonzero2(pv);
        a[(g << 5) + lane] = pv;
      }
    }
  }
  if (__syncthreads_or(zero) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void __launch_bounds__(BLK) k_diag_fix(double2 *__restrict__ a, uint64_t n, int c, double zr, double zi,
                                                  const uint32_t *__restrict__ psigns, const int *flag) {
  if (*(volatile const int *)flag == 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * BLK;
  for (uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x; i < n; i += stride) {
    if (c >= 0 && !((i >> c) & 1ull)) continue;
    const double2 pv = a[i];
    if (nonzero2(pv)) continue;  // P + (+-0) == P: already exact
    const uint32_t l = (uint32_t)(i & 31);
    const uint32_t wre = psigns[2 * (i >> 5)], wim = psigns[2 * (i >> 5) + 1];
    // cmul(z, w) with z a signed zero depends on w only through its sign bits: +-1 stands in for w
    const double2 w = make_double2(((wre >> l) & 1u) ? -1.0 : 1.0, ((wim >> l) & 1u) ? -1.0 : 1.0);
    const double2 sv = cmul(zr, zi, w);
    a[i] = make_double2(__dadd_rn(pv.x, sv.x), __dadd_rn(pv.y, sv.y));
  }
}


// ---------------------------------------------------------------- half exchange
//
// One rank's side of the pairwise exchange, transfer fused with the update:
// `theirs` is the partner slice mapped through CUDA IPC, so a[j] of the
// partner is a 16-B NVLink load and the returned element a 16-B NVLink store.
// Every CTA streams its own chunk; thousands of CTAs in flight overlap the
// remote traffic with the local read/update/write (the paper's T = max(Tcomp,
// Tcomm) pipeline, distributed.py:205-290, without staging buffers).

// Make this CTA's remote stores performed at system scope before it retires,
// so the stream-ordered fence that follows the grid publishes them to the
// partner: the barrier orders every thread's stores before thread 0's
// cumulative fence.sc.sys (one fence per CTA instead of one per thread).
__device__ __forceinline__ void cta_release_system() {
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

__global__ void __launch_bounds__(BLK) k_exchange(double2 *__restrict__ mine, double2 *__restrict__ theirs,
                                                  uint64_t count, uint64_t base, int c_local, int own_is_zero,
                                                  GateQ q) {
  const uint64_t p0 = (uint64_t)blockIdx.x * (BLK * UNROLL) + threadIdx.x;
  double2 am[UNROLL], at[UNROLL];
  uint64_t jj[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    jj[u] = base + (c_local >= 0 ? insert_one(p, c_local) : p);
    if (p < count) {
      am[u] = mine[jj[u]];
      at[u] = theirs[jj[u]];
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    if (p >= count) continue;
    double2 keep, ret;
    if (own_is_zero) {  // a0 = mine, a1 = theirs
      keep = mix(am[u], at[u], q.v[0], q.v[1], q.v[2], q.v[3]);
      ret = mix(am[u], at[u], q.v[4], q.v[5], q.v[6], q.v[7]);
    } else {  // a0 = theirs, a1 = mine
      keep = mix(at[u], am[u], q.v[4], q.v[5], q.v[6], q.v[7]);
      ret = mix(at[u], am[u], q.v[0], q.v[1], q.v[2], q.v[3]);
    }
    mine[jj[u]] = keep;
    theirs[jj[u]] = ret;
  }
  cta_release_system();
}

// ------------------------------------------------ global <-> local qubit swap
//
// SURVEY.md 8(f)4 (PAPER.md:478 future work): instead of exchanging for every
// gate on a global qubit G, swap G with a local qubit l once -- afterwards the
// logical qubit is local and its gates run in HBM.  With b the rank's bit G,
// the swap moves (rank b, bit l = 1-b) <-> (rank 1-b, bit l = b): half of each
// slice, 2^(m+3) B per direction (the in-place exchange moves 2^(m+4)).  One
// thread owns each element pair (reads both, writes both), the zero side the
// first half of the pair space, so the partners never race.  Pure data
// movement: results stay bit-identical.
__global__ void __launch_bounds__(BLK) k_swap_global(double2 *__restrict__ mine, double2 *__restrict__ theirs,
                                                     uint64_t count, uint64_t j0, int l, int b) {
  const uint64_t p0 = (uint64_t)blockIdx.x * (BLK * UNROLL) + threadIdx.x;
  double2 x[UNROLL], y[UNROLL];
  uint64_t im[UNROLL], it[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    const uint64_t j = j0 + p, z = insert_zero(j, l);
    im[u] = b ? z : (z | (1ull << l));  // own half with bit l = 1 - b
    it[u] = b ? (z | (1ull << l)) : z;  // partner half with bit l = b
    if (p < count) {
      x[u] = mine[im[u]];
      y[u] = theirs[it[u]];
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    if (p0 + (uint64_t)u * BLK >= count) continue;
    mine[im[u]] = y[u];
    theirs[it[u]] = x[u];
  }
  cta_release_system();
}

// A whole stage of gates sharing one global target in ONE exchange: every
// pair crosses NVLink once each way however many gates the stage holds
// (controls: local bits -> per-element predicate; rank bits were resolved on
// the host, both partners see the same list).
template <int SIG>
__global__ void __launch_bounds__(BLK) k_exchange_stage(double2 *__restrict__ mine, double2 *__restrict__ theirs,
                                                        uint64_t count, uint64_t base, int own_is_zero,
                                                        const StageParams P) {
  const uint64_t p0 = (uint64_t)blockIdx.x * (BLK * SUNROLL) + threadIdx.x;
  double2 x0[SUNROLL], x1[SUNROLL];
  uint64_t jj[SUNROLL];
#pragma unroll
  for (int u = 0; u < SUNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    jj[u] = base + p;
    if (p < count) {
      const double2 am = mine[jj[u]], at = theirs[jj[u]];
      x0[u] = own_is_zero ? am : at;
      x1[u] = own_is_zero ? at : am;
    } else {
      x0[u] = x1[u] = make_double2(1.0, 1.0);
    }
  }
  if (__builtin_expect(stage_apply_fast<SIG>(x0, x1, jj, P), 0)) {
#pragma unroll
    for (int u = 0; u < SUNROLL; ++u) {
      if (p0 + (uint64_t)u * BLK < count) {
        const double2 am = mine[jj[u]], at = theirs[jj[u]];
        x0[u] = own_is_zero ? am : at;
        x1[u] = own_is_zero ? at : am;
      }
    }
    stage_apply_exact<SIG>(x0, x1, jj, P);
  }
#pragma unroll
  for (int u = 0; u < SUNROLL; ++u) {
    const uint64_t p = p0 + (uint64_t)u * BLK;
    if (p >= count) continue;
    mine[jj[u]] = own_is_zero ? x0[u] : x1[u];
    theirs[jj[u]] = own_is_zero ? x1[u] : x0[u];
  }
  cta_release_system();
}

// ------------------------------------------------------------ register helpers

constexpr int NORM_BLOCKS = SV_NORM_SCRATCH - 1;  // 1024

__global__ void __launch_bounds__(BLK) k_norm_partial(const double2 *__restrict__ a, uint64_t n, int qubit,
                                                      double *__restrict__ partial) {
  __shared__ double red[BLK];
  double acc = 0.0;
  const uint64_t stride = (uint64_t)NORM_BLOCKS * BLK;
  for (uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x; i < n; i += stride) {
    if (qubit >= 0 && !((i >> qubit) & 1ull)) continue;
    const double2 v = a[i];
    acc = __fma_rn(v.x, v.x, acc);
    acc = __fma_rn(v.y, v.y, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = BLK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(BLK) k_norm_final(double *__restrict__ partial) {
  __shared__ double red[BLK];
  double acc = 0.0;
  for (int i = threadIdx.x; i < NORM_BLOCKS; i += BLK) acc += partial[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = BLK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[NORM_BLOCKS] = red[0];
}

// max |a_i - b_i| (complex modulus) over two slices: the full-size self-checks (a circuit
// then its inverse restores the input).  Fixed grid; max is order-independent.
__global__ void __launch_bounds__(BLK) k_maxdiff_partial(const double2 *__restrict__ a,
                                                         const double2 *__restrict__ b, uint64_t n,
                                                         double *__restrict__ partial) {
  __shared__ double red[BLK];
  double acc = 0.0;
  const uint64_t stride = (uint64_t)NORM_BLOCKS * BLK;
  for (uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x; i < n; i += stride) {
    const double2 x = a[i], y = b[i];
    acc = fmax(acc, hypot(x.x - y.x, x.y - y.y));  // NaN-free inputs: fmax keeps the max
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = BLK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(BLK) k_max_final(double *__restrict__ partial) {
  __shared__ double red[BLK];
  double acc = 0.0;
  for (int i = threadIdx.x; i < NORM_BLOCKS; i += BLK) acc = fmax(acc, partial[i]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = BLK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[NORM_BLOCKS] = red[0];
}

// Philox4x32-10 (Salmon et al., SC'11), counter = global amplitude index.
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}

__global__ void __launch_bounds__(BLK) k_init_random(double2 *__restrict__ a, uint64_t n, uint64_t gbase,
                                                     uint64_t seed) {
  const uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x;
  if (i >= n) return;
  const uint64_t g = gbase + i;
  const uint4 r = philox(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0x51u, 0x7u),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t b1 = ((uint64_t)r.x << 32) | r.y, b2 = ((uint64_t)r.z << 32) | r.w;
  const double u1 = ((double)(b1 >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
  const double u2 = (double)(b2 >> 11) * 0x1.0p-53;          // [0, 1)
  const double rad = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  a[i] = make_double2(rad * cs, rad * sn);
}

__global__ void __launch_bounds__(BLK) k_scale(double2 *__restrict__ a, uint64_t n, double s) {
  for (uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLK) {
    const double2 v = a[i];
    a[i] = make_double2(v.x * s, v.y * s);
  }
}

__global__ void __launch_bounds__(BLK) k_basis(double2 *__restrict__ a, uint64_t n, int64_t local) {
  for (uint64_t i = (uint64_t)blockIdx.x * BLK + threadIdx.x; i < n; i += (uint64_t)gridDim.x * BLK)
    a[i] = make_double2((int64_t)i == local ? 1.0 : 0.0, 0.0);
}

// ------------------------------------------------------------------ host side

bool bad_ptr(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

unsigned grid_for(uint64_t items, uint64_t per_block) {
  return (unsigned)((items + per_block - 1) / per_block);
}

unsigned fill_grid(uint64_t n) {
  uint64_t g = (n + BLK - 1) / BLK;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(g < cap ? (g ? g : 1) : cap);
}

// Launch a single-qubit update on (virtual) target tv of an index space of
// 2^vbits elements; the mode decides the address map.
template <int MODE>
int launch_local(double2 *a, int vbits, int tv, int c, const GateQ &q, cudaStream_t st, const char *what) {
  const uint64_t nvirt = 1ull << vbits;
  if (vbits >= 5 && tv < 5) {
    k_shfl<MODE><<<grid_for(nvirt, BLK * UNROLL), BLK, 0, st>>>(a, nvirt, tv, c, q);
  } else {
    const uint64_t np = nvirt >> 1;
    k_pairs<MODE><<<grid_for(np, BLK * PUNROLL), BLK, 0, st>>>(a, np, tv, c, q);
  }
  return after_launch(what);
}

template <int T>
int launch_fused_t(double2 *a, int m, const FusedParams &P, cudaStream_t st) {
  const size_t smem = sizeof(double2) << T;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_fused<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(SV_ECUDA, "sv_apply_fused: smem attribute: %s", cudaGetErrorString(e));
  }
  const uint64_t nblocks = 1ull << (m - T);
  k_fused<T><<<(unsigned)nblocks, FusedShape<T>::NT, smem, st>>>(a, P);
  return after_launch("sv_apply_fused");
}

int launch_fused(double2 *a, int m, int T, const FusedParams &P, cudaStream_t st) {
  switch (T) {
    case 1: return launch_fused_t<1>(a, m, P, st);
    case 2: return launch_fused_t<2>(a, m, P, st);
    case 3: return launch_fused_t<3>(a, m, P, st);
    case 4: return launch_fused_t<4>(a, m, P, st);
    case 5: return launch_fused_t<5>(a, m, P, st);
    case 6: return launch_fused_t<6>(a, m, P, st);
    case 7: return launch_fused_t<7>(a, m, P, st);
    case 8: return launch_fused_t<8>(a, m, P, st);
    case 9: return launch_fused_t<9>(a, m, P, st);
    case 10: return launch_fused_t<10>(a, m, P, st);
    case 11: return launch_fused_t<11>(a, m, P, st);
    case 12: return launch_fused_t<12>(a, m, P, st);
    case 13: return launch_fused_t<13>(a, m, P, st);
    default: return fail(SV_EINVAL, "sv_apply_fused: tile exponent %d unsupported", T);
  }
}

// Kind for the speculative fused kernels (tile, stage): KIND_* above.
int gate_kind(const double *q) {
  const bool z12 = q[2] == 0.0 && q[3] == 0.0, z21 = q[4] == 0.0 && q[5] == 0.0;
  if (z12 && z21) return (q[0] == 1.0 && q[1] == 0.0) ? KIND_PHASE : KIND_DIAG;
  if (!(q[1] == 0.0 && q[3] == 0.0 && q[5] == 0.0 && q[7] == 0.0)) return KIND_GENERAL;
  return (q[0] == q[2] && q[0] == q[4] && q[0] == -q[6]) ? KIND_HSHARE : KIND_REAL;
}

int classify_kind(const double *q) {
  const bool z12 = q[2] == 0.0 && q[3] == 0.0, z21 = q[4] == 0.0 && q[5] == 0.0;
  if (!(z12 && z21)) return KIND_GENERAL;
  return (q[0] == 1.0 && q[1] == 0.0) ? KIND_PHASE : KIND_DIAG;
}

// Segment a run of gates (all targets < T, controls anywhere) for k_tile.
// Greedy: the register set is the next four distinct targets (padded with the
// natural bits T-1, T-2, ...); a segment extends while targets stay in it.
// Returns the number of gates planned (limited by the parameter arrays).
#ifndef SV_TILE_WARPCTL
#define SV_TILE_WARPCTL 1  // measured: 64 half-controlled gates 50.9 -> 49.5 ms, controlled steps -1 %
#endif

int plan_tile(const sv_gate *gates, int n, int T, const int (&hb)[TG_BITS], TileParams &P) {
  P.nsegs = 0;
  for (int k = 0; k < TG_BITS; ++k) P.hb[k] = hb[k];
  auto tbit = [&](int g) {  // slice bit -> tile bit, -1 outside the tile
    if (g < T - TG_BITS) return g;
    for (int k = 0; k < TG_BITS; ++k)
      if (hb[k] == g) return T - TG_BITS + k;
    return -1;
  };
  int gi = 0;
  while (gi < n && gi < TILE_MAX_GATES && P.nsegs < TILE_MAX_SEGS) {
    int S[TR], ns = 0;
    auto in_s = [&](int b) {
      for (int i = 0; i < ns; ++i)
        if (S[i] == b) return true;
      return false;
    };
    for (int j = gi; j < n && ns < TR; ++j)
      if (!in_s(tbit(gates[j].target))) S[ns++] = tbit(gates[j].target);
    for (int b = T - 1; b >= 0 && ns < TR; --b)
      if (!in_s(b)) S[ns++] = b;
    std::sort(S, S + TR);
    TileSeg &seg = P.seg[P.nsegs];
    memset(&seg, 0, sizeof(seg));
    int L[16], nl = 0;
    for (int b = 0; b < T; ++b)
      if (!in_s(b)) L[nl++] = b;
    // thread bits 0..2 (one quarter warp) on tile bits of distinct residue mod 3:
    // with the swizzle, the quarter warp's 16-B accesses then hit 8 bank groups.
    bool used[16] = {};
#if SV_TILE_WARPCTL
    // Controls of this segment on non-register tile bits go to warp bits (thread
    // bits 5..): a warp-uniform skip instead of half the lanes idling.
    int wsel[16], nw = 0;
    {
      int cnt[16] = {};
      for (int j = gi; j < n && j < TILE_MAX_GATES && in_s(tbit(gates[j].target)); ++j) {
        const int c = gates[j].control, tc = c < 0 ? -1 : tbit(c);
        if (tc >= 0 && !in_s(tc))
          for (int i = 0; i < nl; ++i)
            if (L[i] == tc) ++cnt[i];
      }
      const int nwb = nl - 5 > 0 ? nl - 5 : 0;  // warp bits of a 2^(T-TR)-thread CTA
      for (int w = 0; w < nwb; ++w) {
        int best = -1;
        for (int i = 0; i < nl; ++i)
          if (!used[i] && cnt[i] > 0 && (best < 0 || cnt[i] > cnt[best])) best = i;
        if (best < 0) break;
        used[best] = true;
        wsel[nw++] = best;
      }
    }
#endif
    int nt = 0;
    for (int res = 0; res < 3; ++res)
      for (int i = 0; i < nl; ++i)
        if (!used[i] && L[i] % 3 == res) {
          used[i] = true;
          seg.tbits[nt++] = (uint8_t)L[i];
          break;
        }
    for (int i = 0; i < nl; ++i)
      if (!used[i]) seg.tbits[nt++] = (uint8_t)L[i];
#if SV_TILE_WARPCTL
    for (int w = nw - 1; w >= 0; --w) seg.tbits[nt++] = (uint8_t)L[wsel[w]];
#endif
    bool natural = true;
    for (int b = 0; b < TR; ++b) natural &= S[b] == T - TR + b;
    for (int b = 0; b < T - TR; ++b) natural &= seg.tbits[b] == b;
    for (int b = 0; b < TR; ++b) seg.S[b] = (uint8_t)S[b];
    seg.natural = natural ? 1 : 0;
    seg.first = (int16_t)gi;
    while (gi < n && gi < TILE_MAX_GATES && in_s(tbit(gates[gi].target))) {
      const sv_gate &src = gates[gi];
      TileGate &G = P.g[gi];
      memset(&G, 0, sizeof(G));
      for (int b = 0; b < TR; ++b)
        if (S[b] == tbit(src.target)) G.tb = (int8_t)b;
      const int c = src.control, tc = c < 0 ? -1 : tbit(c);
      if (c < 0) {
        G.cmode = 0;
      } else if (tc >= 0 && in_s(tc)) {
        G.cmode = 1;
        for (int b = 0; b < TR; ++b)
          if (S[b] == tc) G.cbit = (int8_t)b;
      } else if (tc >= 0) {
        G.cmode = 2;
        G.cbit = (int8_t)tc;
      } else {
        G.cmode = 3;
        G.cabove = c;
      }
      G.kind = (int8_t)gate_kind(src.q);
      memcpy(G.q, src.q, sizeof(G.q));
      ++gi;
    }
    seg.count = (int16_t)(gi - seg.first);
    bool plain = true;
    for (int k = seg.first; k < gi; ++k) plain &= P.g[k].cmode == 0 && P.g[k].kind == KIND_GENERAL;
    seg.plain = plain ? 1 : 0;
    ++P.nsegs;
  }
  P.last_natural = P.seg[P.nsegs - 1].natural;
  return gi;
}

template <int T, bool SPEC>
int launch_tile_ts(double2 *a, int m, const TileParams &P, cudaStream_t st) {
  const size_t smem = sizeof(double2) << T;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_tile<T, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(SV_ECUDA, "tile: smem attribute: %s", cudaGetErrorString(e));
  }
  k_tile<T, SPEC><<<(unsigned)(1ull << (m - T)), 1 << (T - TR), smem, st>>>(a, P);
  return after_launch("k_tile");
}

template <int T>
int launch_tile_t(double2 *a, int m, const TileParams &P, cudaStream_t st) {
  int ndiag = 0, ngates = 0;
  for (int s = 0; s < P.nsegs; ++s) ngates = P.seg[s].first + P.seg[s].count;
  for (int i = 0; i < ngates; ++i) ndiag += P.g[i].kind != KIND_GENERAL;
  // speculation pays when diagonal/phase updates dominate the run (transform tails)
  return 2 * ndiag >= ngates ? launch_tile_ts<T, true>(a, m, P, st) : launch_tile_ts<T, false>(a, m, P, st);
}


int launch_tile(double2 *a, int m, int T, const TileParams &P, cudaStream_t st) {
  switch (T) {
    case 9: return launch_tile_t<9>(a, m, P, st);
    case 10: return launch_tile_t<10>(a, m, P, st);
    case 11: return launch_tile_t<11>(a, m, P, st);
    case 12: return launch_tile_t<12>(a, m, P, st);
    case 13: return launch_tile_t<13>(a, m, P, st);
    default: return fail(SV_EINVAL, "tile exponent %d unsupported", T);
  }
}

// Run gates (targets in the tile: < T-4 or in hb; controls anywhere) through
// k_tile, as many launches as the parameter arrays need.
int run_tile(double2 *a, int m, int T, const int (&hb)[TG_BITS], const sv_gate *gates, int n, cudaStream_t st) {
  static thread_local TileParams P;  // ~20 KB: keep it off the stack
  int off = 0;
  while (off < n) {
    const int used = plan_tile(gates + off, n - off, T, hb, P);
    const int rc = launch_tile(a, m, T, P, st);
    if (rc != SV_OK) return rc;
    off += used;
  }
  return SV_OK;
}

int launch_gate(double2 *a, int m, const sv_gate &g, cudaStream_t st) {
  const GateQ q = load_q(g.q);
  if (g.control < 0) return launch_local<MODE_SINGLE>(a, m, g.target, 0, q, st, "single");
  if (g.control == 0) return launch_local<MODE_PRED>(a, m, g.target, 0, q, st, "controlled");
  const int tv = g.target < g.control ? g.target : g.target - 1;
  return launch_local<MODE_CTL>(a, m - 1, tv, g.control, q, st, "controlled");
}

int stage_sig(const StageParams &P) {
  for (int i = 1; i < P.ngates; ++i)
    if (P.g[i].kind != KIND_PHASE) return 0;
  return 1;
}

#ifndef SV_XM
#define SV_XM 1  // compiled exact stage groups (k_mstage<true>) for transform-shaped gate lists
#endif

// Is the stage group (P already built from gates[0..n)) shaped like transform stages in exactly
// the order the compiled path executes (see XmParams)?  Fills X.
// forward: slots descending, a block = [butterfly][in-slot phases, control slots descending][outside
// phases]; inverse: slots ascending, a block = [outside phases][in-slot phases, ascending][butterfly].
bool match_xm_dir(const sv_gate *gates, int n, const MsParams &P, XmParams &X, bool inverse) {
  memset(&X, 0xFF, sizeof(X));  // every index -1
  for (int s = 0; s < MS_K; ++s) X.rlo[s] = X.rhi[s] = 0;
  X.inverse = inverse ? 1 : 0;
  X.pad = 0;
  auto slot = [&](int b) {
    for (int s = 0; s < MS_K; ++s)
      if (P.bits[s] == b) return s;
    return MS_K;
  };
  // phase of a block -- forward: 0 butterfly / nothing yet, 1 in-slot, 2 outside;
  //                     inverse: 0 outside / nothing yet, 1 in-slot, 2 butterfly seen (closed)
  int cur = -1, stage = 0, last_in = 0;
  int glo[MS_K], ghi[MS_K];
  for (int s = 0; s < MS_K; ++s) glo[s] = ghi[s] = -1;
  for (int k = 0; k < n; ++k) {
    const sv_gate &g = gates[k];
    const int s = slot(g.target), kind = gate_kind(g.q), c = g.control, cs = c >= 0 ? slot(c) : MS_K;
    if (s == MS_K) return false;
    const bool bfly = kind == KIND_HSHARE && c < 0;
    if (s != cur) {  // a new block: slots strictly descending (forward) / ascending (inverse)
      if (cur >= 0 && (inverse ? s < cur : s > cur)) return false;
      cur = s;
      stage = 0;
      last_in = inverse ? -1 : s;
      if (!inverse && bfly) {
        X.h[s] = k;
        continue;
      }
    }
    if (inverse && bfly) {
      if (stage == 2) return false;
      X.h[s] = k;
      stage = 2;
      continue;
    }
    if (kind != KIND_PHASE || c < 0) return false;
    if (inverse && stage == 2) return false;  // nothing of this slot after its butterfly
    if (cs < MS_K) {  // in-slot: lower slots only, in the order the compiled path applies them
      if (cs >= s) return false;
      if (inverse ? cs <= last_in : (stage > 1 || cs >= last_in)) return false;
      stage = 1;
      last_in = cs;
      X.ins[s][cs] = k;
    } else {
      if (inverse ? stage != 0 : false) return false;  // inverse: outside phases come first
      if (glo[s] < 0) glo[s] = k;
      if (!inverse) stage = 2;
      ghi[s] = k + 1;
    }
  }
  // the outside gates of a slot share one code: they are covered by consecutive runs
  for (int s = 0; s < MS_K; ++s) {
    if (glo[s] < 0) continue;
    int lo = -1, hi = -1;
    for (int ri = 0; ri < P.nruns; ++ri) {
      const int first = 32 * P.run[ri].h + P.run[ri].lo, last = 32 * P.run[ri].h + P.run[ri].hi;
      if (first >= glo[s] && last < ghi[s]) {
        if (lo < 0) lo = ri;
        hi = ri + 1;
      } else if (!(last < glo[s] || first >= ghi[s])) {
        return false;  // a run straddles the range (cannot happen: runs never mix codes)
      }
    }
    if (lo < 0) return false;
    X.rlo[s] = lo;
    X.rhi[s] = hi;
  }
  return true;
}

bool match_xm(const sv_gate *gates, int n, const MsParams &P, XmParams &X) {
#if SV_XM
  if (match_xm_dir(gates, n, P, X, false) || match_xm_dir(gates, n, P, X, true)) return true;
#endif
  memset(&X, 0xFF, sizeof(X));
  for (int s = 0; s < MS_K; ++s) X.rlo[s] = X.rhi[s] = 0;
  X.inverse = 0;
  return false;
}

// One multi-target stage launch: gates[0..n) with targets in <= MS_K bits.
// Host part of a stage launch: MsParams (slots, runs, lane layout) and, for a transform-shaped
// group, the compiled plan X (*compiled = 1).
int build_mstage(int m, const sv_gate *gates, int n, MsParams &P, XmParams &X, int *compiled) {
  if (n < 1 || n > MS_MAX) return fail(SV_EINVAL, "stage group: %d gates not in [1, %d]", n, MS_MAX);
  if (m < MS_K) return fail(SV_EINVAL, "stage group: m=%d below %d", m, MS_K);
  int bits[MS_K], nb = 0;
  for (int k = 0; k < n; ++k) {
    const int t = gates[k].target;
    bool in = false;
    for (int s = 0; s < nb; ++s) in |= bits[s] == t;
    if (in) continue;
    if (nb == MS_K) return fail(SV_EINVAL, "stage group: more than %d distinct targets", MS_K);
    bits[nb++] = t;
  }
  // pad with the most used other controls (their gates become pair patterns), then high bits
  int uses[64] = {0};
  for (int k = 0; k < n; ++k)
    if (gates[k].control >= 0) ++uses[gates[k].control];
  while (nb < MS_K) {
    int best = -1;
    for (int b = m - 1; b >= 0; --b) {
      bool in = false;
      for (int s = 0; s < nb; ++s) in |= bits[s] == b;
      if (!in && (best < 0 || uses[b] > uses[best])) best = b;
    }
    bits[nb++] = best;
  }
  std::sort(bits, bits + MS_K);
  P.ngates = n;
  for (int s = 0; s < MS_K; ++s) P.bits[s] = bits[s];
  memset(P.cbit, 0xFF, sizeof(P.cbit));
  auto slot = [&](int b) {
    for (int s = 0; s < MS_K; ++s)
      if (bits[s] == b) return s;
    return MS_K;
  };
  for (int k = 0; k < n; ++k) {
    const int c = gates[k].control, cs = c >= 0 ? slot(c) : MS_K;
    if (c >= 0 && cs == MS_K) P.cbit[k] = (uint8_t)c;
    P.g[k].code = (gate_kind(gates[k].q) * MS_K + slot(gates[k].target)) * (MS_K + 1) + cs;
    P.g[k].pad = 0;
    memcpy(P.g[k].q, gates[k].q, sizeof(P.g[k].q));
  }
  // Runs split where the control moves between lane bits (per-lane test) and the rest, so the
  // kernel runs the test-free loop for every run without lane-bit controls.
  uint64_t lanes = 0x1F;  // slice bits that differ across the 32 lanes of a warp
  for (int s = 0; s < MS_K; ++s) lanes = ((lanes >> bits[s]) << (bits[s] + 1)) | (lanes & ((1ull << bits[s]) - 1));
  P.hl[0] = P.hl[1] = -1;
  P.nins = 0;
#if SV_MS_HILANE
  {
    // two highest bits that are neither slots nor controls of the group, above the lane bits
    // they would replace; only when slice bits 0..2 are not slots
    bool low_free = true;
    for (int s = 0; s < MS_K; ++s) low_free &= bits[s] > 2;
    int h[2], nh = 0;
    for (int bt = m - 1; bt >= 5 && nh < 2 && low_free; --bt) {
      bool used = uses[bt] > 0;
      for (int s = 0; s < MS_K; ++s) used |= bits[s] == bt;
      if (!used) h[nh++] = bt;
    }
    const uint64_t ldefault = lanes;
    if (nh == 2 && (ldefault & ((1ull << h[0]) | (1ull << h[1]))) == 0) {
      bool lane_ctl = false;  // only worth it when the default lanes carry controls of the group
      for (int b = 3; b < 64; ++b)
        if (((ldefault >> b) & 1ull) && uses[b] > 0) lane_ctl = true;
      if (lane_ctl && m - MS_K >= 5) {
        P.hl[0] = h[1];
        P.hl[1] = h[0];
        int ins[MS_K + 2], ni = 0;
        for (int s = 0; s < MS_K; ++s) ins[ni++] = bits[s];
        ins[ni++] = h[0];
        ins[ni++] = h[1];
        std::sort(ins, ins + ni);
        for (int i = 0; i < ni; ++i) P.ins[i] = ins[i];
        P.nins = ni;
        lanes = 0x7ull | (1ull << h[0]) | (1ull << h[1]);
      }
    }
  }
#endif
  auto lane_dep = [&](int k) { return P.cbit[k] != 0xFF && ((lanes >> P.cbit[k]) & 1ull); };
  P.nruns = 0;
  for (int k = 0; k < n; ++k) {
    MsRun &R = P.run[P.nruns];
    const bool extend = k > 0 && R.code == P.g[k].code && R.h == k / 32 && lane_dep(k) == lane_dep(k - 1);
    if (!extend) {
      MsRun &N = P.run[k > 0 ? ++P.nruns : P.nruns];
      N.code = (uint8_t)P.g[k].code;
      N.h = (uint8_t)(k / 32);
      N.lo = (uint8_t)(k % 32);
    }
    P.run[P.nruns].hi = (uint8_t)(k % 32);
  }
  ++P.nruns;
  for (int ri = 0; ri < P.nruns; ++ri) {
    MsRun &R = P.run[ri];
    R.range = (R.hi == 31 ? 0xffffffffu : ((2u << R.hi) - 1u)) & ~((1u << R.lo) - 1u);
  }
  *compiled = match_xm(gates, n, P, X) ? 1 : 0;
  return SV_OK;
}

int run_mstage(double2 *a, int m, const sv_gate *gates, int n, cudaStream_t st) {
  static thread_local MsParams P;
  XmParams X;
  int compiled = 0;
  const int rc = build_mstage(m, gates, n, P, X, &compiled);
  if (rc != SV_OK) return rc;
  const uint64_t ng = 1ull << (m - MS_K);
  if (compiled)
    k_mstage<true><<<grid_for(ng, ms_blk<true>()), ms_blk<true>(), 0, st>>>(a, ng, P, X);
  else
    k_mstage<false><<<grid_for(ng, ms_blk<false>()), ms_blk<false>(), 0, st>>>(a, ng, P, X);
  return after_launch("k_mstage");
}

// Per-device ring of fold-table buffers for k_dstage (the library's only cached device state,
// besides nothing else: allocated once per device, never freed).  A launch takes the next
// slot, so up to DT_SLOTS launches may be in flight on concurrent streams.
constexpr int DT_SLOTS = 64;
constexpr size_t DT_SLOT_BYTES = (size_t)DS_MAXG * 2 * 8 * 256 * sizeof(double2);  // 32 groups, 8 bytes of index

double2 *dtable_slot() {
  static std::mutex mu;
  static double2 *ring[64] = {};
  static std::atomic<unsigned> next[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!ring[dev]) {
      void *p = nullptr;
      if (cudaMalloc(&p, DT_SLOTS * DT_SLOT_BYTES) != cudaSuccess) return nullptr;
      ring[dev] = (double2 *)p;
    }
  }
  const unsigned k = next[dev].fetch_add(1u) % DT_SLOTS;
  return ring[dev] + k * (DT_SLOT_BYTES / sizeof(double2));
}

// Compile one k_dstage program: gates with targets in the four slot bits `bits` (ascending)
// into GATE / FLUSH ops; fold gates go to T (group ids continue from *ngroups).  Returns
// SV_OK or an error; capacities are checked.
struct DsCompiled {
  int nops = 0, nq = 0;
  double scale = 1.0;
};

int compile_ds(const sv_gate *gates, int n, const int (&bits)[MS_K], uint64_t *hdr, int hcap, double *qv,
               int qcap, DtParams &T, int *ngroups, bool *has0, DsCompiled &out) {
  auto slot = [&](int b) {
    for (int s = 0; s < MS_K; ++s)
      if (bits[s] == b) return s;
    return MS_K;
  };
  int open_group[MS_K];
  for (int s = 0; s < MS_K; ++s) open_group[s] = -1;
  bool overflow = false;
  auto emit = [&](uint64_t lo, const double *q, int nd) {
    if (out.nops >= hcap || out.nq + nd > qcap) {
      overflow = true;
      return;
    }
    hdr[out.nops++] = lo | ((uint64_t)out.nq << 32);
    if (nd) memcpy(qv + out.nq, q, sizeof(double) * nd);
    out.nq += nd;
  };
  auto flush = [&](int s) {
    const int g = open_group[s];
    emit((uint64_t)DS_FLUSH | ((uint64_t)s << 2) | ((uint64_t)(has0[g] ? 1 : 0) << 6) | ((uint64_t)g << 16),
         nullptr, 0);
    open_group[s] = -1;
  };
  for (int k = 0; k < n; ++k) {
    const sv_gate &g = gates[k];
    const int s = slot(g.target), c = g.control, cs = c >= 0 ? slot(c) : MS_K;
    if (s == MS_K) return fail(SV_EINVAL, "tolerance stage: target %d is not a slot", g.target);
    const int kind = gate_kind(g.q);
    const bool diag = kind == KIND_DIAG || kind == KIND_PHASE;
    if (diag && cs == MS_K) {
      if (open_group[s] < 0) {
        if (*ngroups == DS_MAXG) return fail(SV_EINVAL, "tolerance stage: more than %d fold groups", DS_MAXG);
        if (T.nfold >= DT_MAXF) return fail(SV_EINVAL, "tolerance stage: more than %d folded gates", DT_MAXF);
        open_group[s] = (*ngroups)++;
      }
      if (T.nfold >= DT_MAXF) return fail(SV_EINVAL, "tolerance stage: more than %d folded gates", DT_MAXF);
      DtFold &f = T.f[T.nfold++];
      f.group = (int8_t)open_group[s];
      f.c = (int8_t)c;
      f.pad = 0;
      f.pad2 = 0;
      f.d[0] = g.q[0];
      f.d[1] = g.q[1];
      f.d[2] = g.q[6];
      f.d[3] = g.q[7];
      has0[open_group[s]] |= !(g.q[0] == 1.0 && g.q[1] == 0.0);
      continue;
    }
    if (!diag && open_group[s] >= 0) flush(s);
    // an uncontrolled Hadamard-like gate: unscaled butterfly, its real factor deferred to one
    // multiply of every amplitude after the pass (it applies to all of them)
    const bool hbf = SV_DS_HBF && kind == KIND_HSHARE && c < 0;
    if (hbf) out.scale *= g.q[0];
    const int code = ((hbf ? KIND_HBF : kind) * MS_K + s) * (MS_K + 1) + cs;
    const uint64_t cm = (c >= 0 && cs == MS_K) ? (2ull << 4) | ((uint64_t)(c & 63) << 8) : 0ull;
    emit((uint64_t)DS_GATE | ((uint64_t)s << 2) | cm | ((uint64_t)code << 16), g.q, 8);
  }
  for (int s = 0; s < MS_K; ++s)
    if (open_group[s] >= 0) flush(s);
  if (overflow) return fail(SV_EINVAL, "tolerance stage: program exceeds %d ops / %d gate words", hcap, qcap);
  return SV_OK;
}

// Slot bits of a gate run: its distinct targets (at most MS_K), padded with high bits that are
// neither in `avoid` nor any gate's control, then any free bit; ascending.
int ds_slots(const sv_gate *gates, int n, int m, uint64_t avoid, int (&bits)[MS_K]) {
  int nb = 0;
  for (int k = 0; k < n; ++k) {
    const int t = gates[k].target;
    bool in = false;
    for (int s = 0; s < nb; ++s) in |= bits[s] == t;
    if (in) continue;
    if (nb == MS_K) return fail(SV_EINVAL, "tolerance stage: more than %d distinct targets", MS_K);
    bits[nb++] = t;
  }
  uint64_t ctl = 0;
  for (int k = 0; k < n; ++k)
    if (gates[k].control >= 0) ctl |= 1ull << gates[k].control;
  for (int pass = 0; pass < 2; ++pass)
    for (int b = m - 1; b >= 0 && nb < MS_K; --b) {
      bool in = (avoid >> b) & 1ull;
      for (int s = 0; s < nb; ++s) in |= bits[s] == b;
      if (!in && (pass == 1 || !((ctl >> b) & 1ull))) bits[nb++] = b;
    }
  if (nb < MS_K) return fail(SV_EINVAL, "tolerance stage: m=%d too small for the slots", m);
  std::sort(bits, bits + MS_K);
  return SV_OK;
}

int launch_dtable(DtParams &T, int ngroups, int nbytes, cudaStream_t st, const double2 **tab_out) {
  *tab_out = nullptr;
  if (!ngroups) return SV_OK;
  double2 *tab = dtable_slot();
  if (!tab) return fail(SV_ECUDA, "tolerance stage: fold-table buffer allocation failed");
  T.nbytes = nbytes;
  T.tab = tab;
  *tab_out = tab;
  k_dtable<<<ngroups * nbytes * 2, 256, 0, st>>>(T);
  return after_launch("k_dtable");
}

// Does the gate run have the shape of transform stages over the slots `bits` (see XfPhase)?
// Blocks in strictly descending (forward) or ascending (inverse) slot order; a block is the
// slot's uncontrolled Hadamard-like gate (at most one; first in a forward block, last in an
// inverse one) and phase gates diag(1, e) on the slot controlled by a lower slot, a non-slot
// bit or nothing.  On a match fills X, appends the fold gates to T (groups continue from
// *ngroups) and multiplies *scale by the butterflies' factors.
bool match_xform(const sv_gate *gates, int n, const int (&bits)[MS_K], bool inverse, XfPhase &X, DtParams &T,
                 int *ngroups, double *scale) {
  auto slot = [&](int b) {
    for (int s = 0; s < MS_K; ++s)
      if (bits[s] == b) return s;
    return MS_K;
  };
  // pass 1: validate, count what would be appended
  int cur = -1, nfold = 0, ngrp = 0;
  bool closed = false, seen[MS_K] = {}, hasfold[MS_K] = {};
  for (int k = 0; k < n; ++k) {
    const sv_gate &g = gates[k];
    const int s = slot(g.target), kind = gate_kind(g.q);
    if (s == MS_K) return false;
    if (s != cur) {  // a new block
      if (seen[s]) return false;
      if (cur >= 0 && (inverse ? s < cur : s > cur)) return false;
      seen[s] = true;
      cur = s;
      closed = false;
    }
    if (kind == KIND_HSHARE && g.control < 0) {
      if (closed) return false;
      if (!inverse) {
        // forward: the butterfly opens its block
        if (k > 0 && slot(gates[k - 1].target) == s) return false;
      } else {
        closed = true;  // inverse: nothing of this slot may follow
      }
      continue;
    }
    if (kind != KIND_PHASE || closed) return false;
    const int cs = g.control >= 0 ? slot(g.control) : MS_K;
    if (cs < MS_K) {
      if (cs >= s) return false;
    } else {
      if (!hasfold[s]) ++ngrp;
      hasfold[s] = true;
      ++nfold;
    }
  }
  if (*ngroups + ngrp > DS_MAXG || T.nfold + nfold > DT_MAXF) return false;
  // pass 2: fill
  memset(&X, 0, sizeof(X));
  for (int s = 0; s < MS_K; ++s)
    for (int k = 0; k < MS_N / 2; ++k) X.phw[s][k] = make_double2(1.0, 0.0);
  for (int k = 0; k < n; ++k) {
    const sv_gate &g = gates[k];
    const int s = slot(g.target), kind = gate_kind(g.q);
    if (kind == KIND_HSHARE && g.control < 0) {
      X.hmask |= 1 << s;
      *scale *= g.q[0];
      continue;
    }
    const int cs = g.control >= 0 ? slot(g.control) : MS_K;
    if (cs < MS_K) {
      X.pmask |= 1 << s;
      for (int j = 0; j < (1 << s); ++j) {
        if (!((j >> cs) & 1)) continue;
        const double2 w = X.phw[s][j];
        X.phw[s][j] = make_double2(w.x * g.q[6] - w.y * g.q[7], w.x * g.q[7] + w.y * g.q[6]);
      }
    } else {
      if (!((X.fmask >> s) & 1)) {
        X.fmask |= 1 << s;
        X.group[s] = (*ngroups)++;
      }
      DtFold &f = T.f[T.nfold++];
      f.group = (int8_t)X.group[s];
      f.c = (int8_t)g.control;
      f.pad = 0;
      f.pad2 = 0;
      f.d[0] = 1.0;
      f.d[1] = 0.0;
      f.d[2] = g.q[6];
      f.d[3] = g.q[7];
    }
  }
  return true;
}

#ifndef SV_XFORM
#define SV_XFORM 1  // compiled transform phases (k_xstage2) when both phases of a two-phase pass match
#endif

template <int NB, bool INV, bool FULL>
void launch_xstage2_t(double2 *a, uint64_t ntiles, const Xf2Params &X, cudaStream_t st) {
  constexpr int SMEM = DS2_SMEM;
  static int per = 0, nsm = 0;
  if (!per) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_xstage2<NB, INV, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_xstage2<NB, INV, FULL>, 256, SMEM) != cudaSuccess ||
        per < 1)
      per = 1;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)nsm * per);
  k_xstage2<NB, INV, FULL><<<grid, 256, SMEM, st>>>(a, ntiles, X);
}

template <bool INV>
bool launch_xstage2(double2 *a, uint64_t ntiles, const Xf2Params &X, cudaStream_t st) {
  bool full = true;
  for (int p = 0; p < 2; ++p) full &= X.ph[p].hmask == 0xF && X.ph[p].fmask == 0xF && X.ph[p].pmask == 0xE;
#define XS2_CASE(NB_)                                                \
  case NB_:                                                          \
    if (full)                                                        \
      launch_xstage2_t<NB_, INV, true>(a, ntiles, X, st);            \
    else                                                             \
      launch_xstage2_t<NB_, INV, false>(a, ntiles, X, st);           \
    return true;
  switch (X.nbytes) {
    XS2_CASE(2) XS2_CASE(3) XS2_CASE(4) XS2_CASE(5)
    default: return false;
  }
#undef XS2_CASE
}

// The slot sets of a two-phase group (gates[0..split) on S1, the rest on S2) and its coalescing bits.
int stage2_slots(int m, const sv_gate *gates, int n, int split, int (&s1)[MS_K], int (&s2)[MS_K], int (&lb)[MS_K]) {
  if (m < 3 * MS_K + 1) return fail(SV_EINVAL, "two-phase stage: m=%d below %d", m, 3 * MS_K + 1);
  if (split < 1 || split >= n) return fail(SV_EINVAL, "two-phase stage: split %d outside (0, %d)", split, n);
  int rc = ds_slots(gates, split, m, 0, s1);
  if (rc) return rc;
  uint64_t used = 0;
  for (int k = 0; k < MS_K; ++k) used |= 1ull << s1[k];
  rc = ds_slots(gates + split, n - split, m, used, s2);
  if (rc) return rc;
  for (int k = 0; k < MS_K; ++k) used |= 1ull << s2[k];
  for (int k = 0; k < n; ++k) {  // phase 1 must not touch S2 targets, nor phase 2 S1 targets
    const bool in1 = (used >> gates[k].target) & 1ull;
    bool is1 = false;
    for (int q = 0; q < MS_K; ++q) is1 |= s1[q] == gates[k].target;
    if (!in1 || (k < split) != is1) return fail(SV_EINVAL, "two-phase stage: gate %d targets the wrong phase", k);
  }
  int nl = 0;
  for (int b = 0; b < m && nl < MS_K; ++b)
    if (!((used >> b) & 1ull)) lb[nl++] = b;
  if (nl < MS_K) return fail(SV_EINVAL, "two-phase stage: no room for the coalescing bits");
  return SV_OK;
}

// 0: the interpreter; 1 / 2: both phases compile as forward / inverse transform stages (fills X, T).
int stage2_shape(int m, const sv_gate *gates, int n, int split, const int (&s1)[MS_K], const int (&s2)[MS_K],
                 Xf2Params &X, DtParams &T, int *ngroups, double *scale) {
#if SV_XFORM
  const int nbytes = (m + 7) / 8;
  if (nbytes < 2 || nbytes > 5) return 0;
  for (int inverse = 0; inverse < 2; ++inverse) {
    T.nfold = 0;
    *ngroups = 0;
    *scale = 1.0;
    if (match_xform(gates, split, s1, inverse != 0, X.ph[0], T, ngroups, scale) &&
        match_xform(gates + split, n - split, s2, inverse != 0, X.ph[1], T, ngroups, scale))
      return 1 + inverse;
  }
#endif
  return 0;
}

// Index bytes the fold tables of a compiled launch really need: up to the highest fold control
// (the product over higher bytes is 1), at least 2 (the smallest instantiation).
int fold_bytes(const DtParams &T, int nbytes) {
  int top = 0;
  for (int i = 0; i < T.nfold; ++i) top = T.f[i].c > top ? T.f[i].c : top;
  const int need = top / 8 + 1;
  return need < 2 ? 2 : need < nbytes ? need : nbytes;
}

// Two-phase tolerance stage launch (k_dstage2): gates[0..split) target S1, gates[split..n) S2.
int run_dstage2(double2 *a, int m, const sv_gate *gates, int n, int split, cudaStream_t st) {
  static thread_local Ds2Params P;
  static thread_local DtParams T;
  int s1[MS_K], s2[MS_K], lb[MS_K];
  int rc = stage2_slots(m, gates, n, split, s1, s2, lb);
  if (rc) return rc;
  const int nbytes = (m + 7) / 8;
  const uint64_t ntiles = 1ull << (m - 3 * MS_K);
  {  // both phases shaped like transform stages: the compiled kernel
    static thread_local Xf2Params X;
    int ng = 0;
    double scale = 1.0;
    const int shape = stage2_shape(m, gates, n, split, s1, s2, X, T, &ng, &scale);
    if (shape) {
      const int nb = fold_bytes(T, nbytes);  // QFT(30): 4 / 3 / 2 bytes for the three passes
      rc = launch_dtable(T, ng, nb, st, &X.tab);
      if (rc) return rc;
      X.nbytes = nb;
      X.scale = scale;
      int xt[3 * MS_K], nx = 0;
      for (int k = 0; k < MS_K; ++k) {
        X.s1[k] = s1[k], X.s2[k] = s2[k], X.lb[k] = lb[k];
        xt[nx++] = s1[k], xt[nx++] = s2[k], xt[nx++] = lb[k];
      }
      std::sort(xt, xt + nx);
      for (int k = 0; k < nx; ++k) X.tb[k] = xt[k];
      if (shape == 2 ? launch_xstage2<true>(a, ntiles, X, st) : launch_xstage2<false>(a, ntiles, X, st))
        return after_launch("k_xstage2");
    }
  }
  T.nfold = 0;
  int ngroups = 0;
  bool has0[DS_MAXG] = {};
  DsCompiled c1, c2;
  rc = compile_ds(gates, split, s1, P.hdr[0], DS2_MAX, P.q[0], DS2_QMAX, T, &ngroups, has0, c1);
  if (rc) return rc;
  rc = compile_ds(gates + split, n - split, s2, P.hdr[1], DS2_MAX, P.q[1], DS2_QMAX, T, &ngroups, has0, c2);
  if (rc) return rc;
  rc = launch_dtable(T, ngroups, nbytes, st, &P.tab);
  if (rc) return rc;
  P.nops[0] = c1.nops;
  P.nops[1] = c2.nops;
  P.nbytes = nbytes;
  P.scale = c1.scale * c2.scale;
  int tb[3 * MS_K], nt = 0;
  for (int k = 0; k < MS_K; ++k) {
    P.s1[k] = s1[k], P.s2[k] = s2[k], P.lb[k] = lb[k];
    tb[nt++] = s1[k], tb[nt++] = s2[k], tb[nt++] = lb[k];
  }
  std::sort(tb, tb + nt);
  for (int k = 0; k < nt; ++k) P.tb[k] = tb[k];
  constexpr int SMEM = DS2_SMEM;
  static int per = 0, nsm = 0;
  if (!per) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_dstage2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_dstage2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dstage2<4>, 256, SMEM) != cudaSuccess || per < 1)
      per = 1;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)nsm * per);
  switch (nbytes) {
    case 1: k_dstage2<1><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 2: k_dstage2<2><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 3: k_dstage2<3><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 4: k_dstage2<4><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 5: k_dstage2<5><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 6: k_dstage2<6><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    case 7: k_dstage2<7><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
    default: k_dstage2<8><<<grid, 256, SMEM, st>>>(a, ntiles, P); break;
  }
  return after_launch("k_dstage2");
}

template <int NB, bool INV>
int launch_xstage_t(double2 *a, int m, const Xf1Params &X, cudaStream_t st) {
  constexpr int SMEM = MS_N * 256 * (int)sizeof(double2);
  static int per = 0, nsm = 0;
  if (!per) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_xstage<NB, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_xstage<NB, INV>, 256, SMEM) != cudaSuccess || per < 1)
      per = 1;
  }
  const uint64_t ng = 1ull << (m - MS_K);
  const unsigned grid = (unsigned)std::min<uint64_t>(grid_for(ng, 256), (uint64_t)nsm * per);
  k_xstage<NB, INV><<<grid, 256, SMEM, st>>>(a, ng, X);
  return after_launch("k_xstage");
}

template <bool INV>
int launch_xstage(double2 *a, int m, const Xf1Params &X, cudaStream_t st) {
  switch (X.nbytes) {
    case 2: return launch_xstage_t<2, INV>(a, m, X, st);
    case 3: return launch_xstage_t<3, INV>(a, m, X, st);
    case 4: return launch_xstage_t<4, INV>(a, m, X, st);
    default: return launch_xstage_t<5, INV>(a, m, X, st);
  }
}

// Tolerance-mode stage launch (k_dtable + k_dstage): compile gates[0..n) (targets in <= MS_K
// bits) into GATE / FLUSH ops and fold groups.
int run_dstage(double2 *a, int m, const sv_gate *gates, int n, cudaStream_t st) {
  static thread_local DsParams P;
  static thread_local DtParams T;
  if (n < 1 || n > MS_MAX) return fail(SV_EINVAL, "tolerance stage group: %d gates not in [1, %d]", n, MS_MAX);
  if (m < MS_K) return fail(SV_EINVAL, "tolerance stage group: m=%d below %d", m, MS_K);
  int bits[MS_K];
  int rc = ds_slots(gates, n, m, 0, bits);
  if (rc) return rc;
  const int nbytes = (m + 7) / 8;
#if SV_XFORM
  if (nbytes >= 2 && nbytes <= 5) {  // shaped like transform stages: the compiled phase
    static thread_local Xf1Params X;
    for (int inverse = 0; inverse < 2; ++inverse) {
      T.nfold = 0;
      int ng = 0;
      double scale = 1.0;
      if (!match_xform(gates, n, bits, inverse != 0, X.ph, T, &ng, &scale)) continue;
      const int nb = fold_bytes(T, nbytes);
      rc = launch_dtable(T, ng, nb, st, &X.tab);
      if (rc) return rc;
      X.nbytes = nb;
      X.scale = scale;
      for (int k = 0; k < MS_K; ++k) X.bits[k] = bits[k];
      return inverse ? launch_xstage<true>(a, m, X, st) : launch_xstage<false>(a, m, X, st);
    }
  }
#endif
  int ngroups = 0;
  bool has0[DS_MAXG] = {};
  T.nfold = 0;
  DsCompiled c;
  rc = compile_ds(gates, n, bits, P.hdr, DS_MAX, P.q, DS_QMAX, T, &ngroups, has0, c);
  if (rc) return rc;
  const double scale = c.scale;
  P.nops = c.nops;
  P.nbytes = nbytes;
  for (int k = 0; k < MS_K; ++k) P.bits[k] = bits[k];
  rc = launch_dtable(T, ngroups, nbytes, st, &P.tab);
  if (rc) return rc;
  P.nfg = ngroups;
  P.scale = scale;
  P.has0 = 0;
  for (int g = 0; g < ngroups; ++g) P.has0 |= has0[g] ? (1u << g) : 0u;
  const uint64_t ng = 1ull << (m - MS_K);
  static int per_sm[9] = {};  // resident CTAs per SM of k_dstage<NB> (persistent grid)
  constexpr int DS_SMEM = MS_N * 256 * (int)sizeof(double2);  // 64 KiB prefetch slots per CTA
  auto occupancy = [&](auto kern, int nbt) {
    if (!per_sm[nbt]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DS_SMEM);
      int v = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 256, DS_SMEM) != cudaSuccess || v < 1) v = 1;
      per_sm[nbt] = v;
    }
    return per_sm[nbt];
  };
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int per = 1;
  switch (nbytes) {
    case 1: per = occupancy(k_dstage<1>, 1); break;
    case 2: per = occupancy(k_dstage<2>, 2); break;
    case 3: per = occupancy(k_dstage<3>, 3); break;
    case 4: per = occupancy(k_dstage<4>, 4); break;
    case 5: per = occupancy(k_dstage<5>, 5); break;
    case 6: per = occupancy(k_dstage<6>, 6); break;
    case 7: per = occupancy(k_dstage<7>, 7); break;
    default: per = occupancy(k_dstage<8>, 8); break;
  }
  const uint64_t need = grid_for(ng, 256);
  const unsigned grid = (unsigned)std::min<uint64_t>(need, (uint64_t)nsm * per);
  switch (nbytes) {
    case 1: k_dstage<1><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 2: k_dstage<2><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 3: k_dstage<3><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 4: k_dstage<4><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 5: k_dstage<5><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 6: k_dstage<6><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    case 7: k_dstage<7><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
    default: k_dstage<8><<<grid, 256, DS_SMEM, st>>>(a, ng, P); break;
  }
  return after_launch("k_dstage");
}
// ops <= gates + flushes, and every flush follows a fold and precedes a gate (or ends the pass)
static_assert(DS_MAX >= 3 * MS_MAX / 2 + MS_K && DS_QMAX >= 8 * MS_MAX, "k_dstage program capacity");
static_assert(DT_SLOT_BYTES >= (size_t)DS_MAXG * 2 * ((62 + 7) / 8) * 256 * sizeof(double2), "fold-table slot");

// Tolerance-mode low-bit launch (k_dlow): every target in slice bits 0..5 (controls anywhere).
// The tail of a transform on qubits t0..0 (t0 <= 5), exactly: 1 = forward (for t = t0..0: the
// butterfly, then R(t, c) for c = t-1..0), 2 = inverse (for t = 0..t0: R(t, c) for c = 0..t-1,
// then the butterfly), 0 = neither; xq[t] = index of stage t's first gate.
int xtail_shape(const sv_gate *gates, int n, int32_t (&xq)[DL_BITS]) {
  auto is_h = [&](int k, int t) {
    return k < n && gates[k].target == t && gates[k].control < 0 && gate_kind(gates[k].q) == KIND_HSHARE;
  };
  auto is_r = [&](int k, int t, int c) {
    return k < n && gates[k].target == t && gates[k].control == c && gate_kind(gates[k].q) == KIND_PHASE;
  };
  for (int t = 0; t < DL_BITS; ++t) xq[t] = -1;
  if (n < 1 || gates[0].target >= DL_BITS) return 0;
  {  // forward
    int k = 0, t = gates[0].target;
    bool ok = true;
    for (; ok && t >= 0; --t) {
      ok = is_h(k, t);
      if (!ok) break;
      xq[t] = k++;
      for (int c = t - 1; ok && c >= 0; --c, ++k) ok = is_r(k, t, c);
    }
    if (ok && k == n) return 1;
  }
  for (int t = 0; t < DL_BITS; ++t) xq[t] = -1;
  {  // inverse
    int k = 0;
    bool ok = gates[0].target == 0;
    for (int t = 0; ok && t < DL_BITS && k < n; ++t) {
      xq[t] = k;
      for (int c = 0; ok && c < t; ++c, ++k) ok = is_r(k, t, c);
      ok = ok && is_h(k, t);
      ++k;
    }
    if (ok && k == n) return 2;
  }
  for (int t = 0; t < DL_BITS; ++t) xq[t] = -1;
  return 0;
}

int run_dlow(double2 *a, int m, const sv_gate *gates, int n, cudaStream_t st, bool exact = false) {
  static thread_local DlParams P;
  if (m < 11) return fail(SV_EINVAL, "low-bit group: m=%d below 11", m);
  if (n < 1 || n > DL_MAX) return fail(SV_EINVAL, "low-bit group: %d gates not in [1, %d]", n, DL_MAX);
  int nops = 0, ntab = 0, nst = 0, ngate = 0, layout = 0;
  double scale = 1.0;
  bool pending = false;
  double tr[64], ti[64];
  // the pending diagonal run as one stage: its common target (-2: none yet, -1: not one stage)
  // and the product of its phases per control (index 6: uncontrolled)
  int run_t = -2;
  double ur[7], ui[7];
  auto reset = [&]() {
    for (int x = 0; x < 64; ++x) tr[x] = 1.0, ti[x] = 0.0;
    for (int c = 0; c < 7; ++c) ur[c] = 1.0, ui[c] = 0.0;
    run_t = -2;
  };
  // register bits of a slice bit (< 6) in a layout, -1 when it is a lane bit
  auto regbit = [](int lay, int b) { return lay ? (b < 3 ? b : -1) : ((b >= 3 && b < 6) ? b - 3 : -1); };
  auto flush = [&]() {
    if (!pending) return 0;
    if (run_t >= 0 && regbit(layout, run_t) >= 0 && nst < DL_TABMAX) {  // one stage on a register bit
      const int rbt = regbit(layout, run_t), lane0 = layout ? 3 : 0, reg0 = layout ? 0 : 3;
      auto mul = [](double &xr, double &xi, double yr, double yi) {
        const double nr = xr * yr - xi * yi, ni = xr * yi + xi * yr;
        xr = nr, xi = ni;
      };
      for (int v = 0; v < 8; ++v) {
        double fr = ur[6], fi = ui[6];
        for (int i = 0; i < 3; ++i)
          if ((v >> i) & 1) mul(fr, fi, ur[lane0 + i], ui[lane0 + i]);
        P.stl[nst][v] = make_double2(fr, fi);
      }
      int other[2], no = 0;
      for (int b = 0; b < 3; ++b)
        if (b != rbt) other[no++] = reg0 + b;
      for (int k = 0; k < 4; ++k) {
        double fr = 1.0, fi = 0.0;
        for (int i = 0; i < 2; ++i)
          if ((k >> i) & 1) mul(fr, fi, ur[other[i]], ui[other[i]]);
        P.str[nst][k] = make_double2(fr, fi);
      }
      P.hdr[nops++] = (uint64_t)DL_STAGE | ((uint64_t)rbt << 2) | ((uint64_t)nst << 16);
      ++nst;
      pending = false;
      reset();
      return 0;
    }
    if (ntab == DL_TABMAX) return fail(SV_EINVAL, "low-bit group: more than %d diagonal runs", DL_TABMAX);
    for (int x = 0; x < 64; ++x) P.tab[ntab][x] = make_double2(tr[x], ti[x]);
    P.hdr[nops++] = (uint64_t)DL_TABLE | ((uint64_t)ntab << 16);
    ++ntab;
    pending = false;
    reset();
    return 0;
  };
  reset();
  for (int k = 0; k < n; ++k) {
    const sv_gate &g = gates[k];
    if (g.target < 0 || g.target >= DL_BITS) return fail(SV_EINVAL, "low-bit group: target %d >= %d", g.target, DL_BITS);
    const int c = g.control, kind = gate_kind(g.q);
    const bool diag = kind == KIND_DIAG || kind == KIND_PHASE;
    if (!exact && diag && c < DL_BITS) {  // into the block's product table
      for (int x = 0; x < 64; ++x) {
        if (c >= 0 && !((x >> c) & 1)) continue;
        const int o = ((x >> g.target) & 1) ? 6 : 0;
        const double dr = g.q[o], di = g.q[o + 1];
        const double nr = tr[x] * dr - ti[x] * di, ni = tr[x] * di + ti[x] * dr;
        tr[x] = nr;
        ti[x] = ni;
      }
      if (kind == KIND_PHASE && (run_t == -2 || run_t == g.target)) {
        run_t = g.target;
        const int ci = c < 0 ? 6 : c;
        const double nr = ur[ci] * g.q[6] - ui[ci] * g.q[7], ni = ur[ci] * g.q[7] + ui[ci] * g.q[6];
        ur[ci] = nr, ui[ci] = ni;
      } else {
        run_t = -1;
      }
      pending = true;
      continue;
    }
    int rc = flush();
    if (rc) return rc;
    if (regbit(layout, g.target) < 0) {  // bring the target into the registers
      layout ^= 1;
      P.hdr[nops++] = (uint64_t)DL_LAYOUT | ((uint64_t)layout << 16);
    }
    const bool hbf = !exact && kind == KIND_HSHARE && c < 0;
    if (hbf) scale *= g.q[0];
    uint64_t cm = 0, cb = 0;
    if (c >= 0) {
      const int rbc = c < DL_BITS ? regbit(layout, c) : -1;
      cm = rbc >= 0 ? 1 : 2;
      cb = rbc >= 0 ? (uint64_t)rbc : (uint64_t)c;
    }
    P.hdr[nops++] = (uint64_t)DL_GATE | ((uint64_t)regbit(layout, g.target) << 2) |
                    ((uint64_t)(hbf ? KIND_HBF : kind) << 4) | (cm << 8) | (cb << 10) | ((uint64_t)ngate << 16);
    memcpy(P.q[ngate], g.q, sizeof(P.q[0]));
    ++ngate;
  }
  int rc = flush();
  if (rc) return rc;
  P.nops = nops;
  P.ntab = ntab;
  P.nst = nst;
  P.scale = scale;
  // exact mode: the gate list is exactly the stages t0..0 of a transform (or 0..t0 of its inverse)
  P.compiled = exact ? xtail_shape(gates, n, P.xq) : 0;
  if (!P.compiled)
    for (int q = 0; q < DL_BITS; ++q) P.xq[q] = -1;
  const uint64_t nblocks = 1ull << (m - 8);
  static int per[2] = {0, 0}, nsm = 0;
  if (!per[exact]) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int v = 0;
    const cudaError_t e = exact ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_dlow<true>, 256, 0)
                                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_dlow<false>, 256, 0);
    per[exact] = (e != cudaSuccess || v < 1) ? 1 : v;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>(grid_for(nblocks, 8), (uint64_t)nsm * per[exact]);
  if (exact)
    k_dlow<true><<<grid, 256, 0, st>>>(a, nblocks, P);
  else
    k_dlow<false><<<grid, 256, 0, st>>>(a, nblocks, P);
  return after_launch("k_dlow");
}

// Native pass planner: the launch group starting at gates[i], returned as its end.
// Candidate 1, a register-tiled run: targets below L = T-G, or one of up to G
// (TG_BITS) higher slice bits taken in order of appearance (the tile then
// gathers those bits).  Candidate 2, a stage: the run whose targets stay within MS_K = 4
// distinct bits.  Cost model (B200, ms at 2^30 amplitudes, compute overlapping
// HBM): a pass costs max(5, sum of per-gate costs); per gate, tile 1.15
// general / 0.45 diagonal (real 0.75, Hadamard-like 0.55), stage by structure (general 0.9, real 0.55,
// Hadamard-like 0.35, diagonal 0.35, phase 0.18; half that when controlled;
// a stage with a target below bit 3 pays 1.7x for its strided loads).
// The candidate with the lower cost per gate wins (ties: the stage).  A lone
// gate is a single-gate launch.  Pure host code (sv_plan_gates exposes it).
#ifndef SV_PLAN_LOOKAHEAD
#define SV_PLAN_LOOKAHEAD 1  // measured: QFT(30) 74.2 -> 72.2 ms (one tail tile instead of stage + tile), controlled steps -2 %
#endif

double stage_cost(const sv_gate &g, bool tol) {
  static const double c[KIND_COUNT] = {0.9, 0.35, 0.18, 0.55, 0.35};
  const int k = gate_kind(g.q);
  // tolerance mode: a diagonal gate folds into a per-thread factor (one multiply per 16 amplitudes)
  if (tol && (k == KIND_DIAG || k == KIND_PHASE)) return 0.02;
  return c[k] * (g.control >= 0 ? 0.5 : 1.0);
}

// Tolerance mode: the run from i whose targets all lie in slice bits 0..DL_BITS-1 (k_dlow), as
// long as its diagonal runs fit the table budget; its length.
int low_run(int m, const sv_gate *gates, int n, int i, bool tol = true) {
  if (m < 11) return 0;
  int j = i, tabs = 0;
  bool in_diag = false;
  for (; j < n && j - i < DL_MAX; ++j) {
    if (gates[j].target >= DL_BITS) break;
    const int k = gate_kind(gates[j].q);
    const bool d = tol && (k == KIND_DIAG || k == KIND_PHASE) && gates[j].control < DL_BITS;
    if (d && !in_diag) {
      if (tabs == DL_TABMAX) break;
      ++tabs;
    }
    in_diag = d;
  }
  return j - i;
}

// Tolerance mode: the two-phase stage run from i (k_dstage2): up to MS_K distinct targets, then up
// to MS_K others, never returning to the first set; per phase at most MS_MAX gates.  Returns its
// end (i when there is no second phase);
// *split = the first gate of phase 2.  The same scan recovers the split from a planned group.
int stage2_run(int m, const sv_gate *gates, int n, int i, int *split) {
  *split = i;
  if (m < 3 * MS_K + 2) return i;
  int S[2][MS_K], ns[2] = {0, 0}, ph = 0, cnt = 0, j = i;
  auto in = [&](int p, int t) {
    for (int k = 0; k < ns[p]; ++k)
      if (S[p][k] == t) return true;
    return false;
  };
  for (; j < n; ++j) {
    const int t = gates[j].target;
    // slots below bit 4 would push the coalescing lanes off the contiguous low bits (such a pass
    // runs at 1.5-2.3x an ordinary one): those gates are left to a low-bit pass / a stage pass
    if (t < MS_K) break;
    if (ph == 0 && !in(0, t)) {
      if (ns[0] == MS_K) {
        ph = 1;
        *split = j;
        cnt = 0;
      } else {
        S[0][ns[0]++] = t;
      }
    }
    if (ph == 1) {
      if (in(0, t)) break;
      if (!in(1, t)) {
        if (ns[1] == MS_K) break;
        S[1][ns[1]++] = t;
      }
    }
    if (cnt + 1 > MS_MAX) {
      if (ph == 0) return i;
      break;
    }
    ++cnt;
  }
  return ph == 1 ? j : i;
}

int next_group(int m, const sv_gate *gates, int n, int i, int T, int *kind, bool tol = false) {
  const int L = T - TG_BITS;
  auto tile_cost = [&](int k) {
    static const double c[KIND_COUNT] = {1.15, 0.45, 0.45, 0.75, 0.55};
    return c[gate_kind(gates[k].q)];
  };
  auto pass = [](double c) { return c > 5.0 ? c : 5.0; };
  int H[TG_BITS], nh = 0, ja = i;
  double ct = 0.0;
  if (T >= 9) {
    for (; ja < n && ja - i < TILE_MAX_GATES; ++ja) {
      const int tt = gates[ja].target;
      bool in = tt < L;
      for (int k = 0; k < nh && !in; ++k) in = H[k] == tt;
      if (!in) {
        if (nh == TG_BITS) break;
        H[nh++] = tt;
      }
      ct += tile_cost(ja);
    }
  }
  int S[MS_K], ns = 0, jb = i;
  double cs = 0.0;
  if (m >= MS_K + 5) {
    for (; jb < n && jb - i < MS_MAX; ++jb) {
      const int tt = gates[jb].target;
      bool in = false;
      for (int k = 0; k < ns && !in; ++k) in = S[k] == tt;
      if (!in) {
        if (ns == MS_K) break;
        S[ns++] = tt;
      }
      cs += stage_cost(gates[jb], tol);
    }
  }
  const int A = ja - i, B = jb - i;
  int lowest = 64;
  for (int k = 0; k < ns; ++k) lowest = S[k] < lowest ? S[k] : lowest;
  if (lowest < 3) cs = 1.7 * pass(cs);  // slot bits 0..2: 16-B pieces at 128-B strides per load (measured)
  {  // a low-bit run: one k_dlow pass
    const int C = low_run(m, gates, n, i, tol);
    // tolerance mode: when it is at least as long as both other candidates
    if (tol && C >= 2 && C >= A && C >= B) {
      *kind = SV_GROUP_LOW;
      return i + C;
    }
    // exact mode: only a transform tail (forward or inverse), which runs as compiled straight-line
    // code in k_dlow<exact> -- one HBM-bound pass (6 ms at n = 30) where the tile needs 10 ms for the
    // six forward stages and 24 ms for the twelve inverse stages it would gather.  (Any other exact
    // low-bit run goes through the op interpreter at ~0.8 ms per gate: the tile is faster.)
    if (!tol && C >= 2 && (C >= 10 || (C >= A && C >= B))) {
      int32_t xq[DL_BITS];
      if (xtail_shape(gates + i, C, xq)) {
        *kind = SV_GROUP_LOW;
        return i + C;
      }
    }
    // tolerance mode: k_dlow is one HBM-bound pass whatever it carries (diagonal runs are
    // factors), so it also wins against a longer but FP64-heavy tile / stage run per gate --
    // e.g. the first stages of an inverse transform (a 78-gate tile of 12 stages: 24 ms at
    // n = 30; its first six stages as a low-bit pass: 6 ms)
    if (tol && C >= 8) {
      const double per_low = 5.5 / C;
      if ((A <= 1 || per_low <= pass(ct) / A) && (B <= 1 || per_low <= pass(cs) / B)) {
        *kind = SV_GROUP_LOW;
        return i + C;
      }
    }
  }
  if (tol) {
    // a two-phase stage run (eight targets) longer than both: one k_dstage2 pass, when it is
    // mostly diagonal (its folds are what make it cheap; general gates cost the same anywhere)
    int split;
    const int e = stage2_run(m, gates, n, i, &split);
    // longer than the stage run, and longer than the tile run or cheaper per gate than it (a
    // mostly diagonal two-phase pass costs ~7 ms whatever it carries)
    if (e - i > B && (e - i >= A || 7.0 / (e - i) <= pass(ct) / A)) {
      int nd = 0;
      for (int k = i; k < e; ++k) {
        const int kd = gate_kind(gates[k].q);
        nd += kd == KIND_DIAG || kd == KIND_PHASE;
      }
      if (2 * nd >= e - i) {
        *kind = SV_GROUP_STAGE2;
        return e;
      }
    }
  }
  if (A <= 1 && B <= 1) {
    *kind = SV_GROUP_GATES;
    return i + 1;
  }
#if SV_PLAN_LOOKAHEAD
  if (B > 1 && A > B) {  // the tile run covers the stage run and more: vs the stage + one pass for the rest
    double rest = 0.0;
    for (int k = i + B; k < i + A; ++k) rest += tile_cost(k);
    if (pass(ct) <= pass(cs) + pass(rest)) {
      *kind = SV_GROUP_TILE;
      return ja;
    }
  }
#endif
  if (B > 1 && (A <= 1 || pass(cs) / B <= pass(ct) / A)) {
    *kind = SV_GROUP_STAGE;
    return jb;
  }
  *kind = SV_GROUP_TILE;
  return ja;
}

bool stage_gains_from_tolerance(const sv_gate *gates, int n) {
  uint64_t targets = 0;
  for (int k = 0; k < n; ++k) targets |= 1ull << gates[k].target;
  for (int k = 0; k < n; ++k) {
    const int kd = gate_kind(gates[k].q), c = gates[k].control;
    if ((kd == KIND_DIAG || kd == KIND_PHASE) && (c < 0 || !((targets >> c) & 1ull))) return true;
    if (kd == KIND_HSHARE && c < 0) return true;
  }
  return false;
}

int exec_group(double2 *a, int m, int T, int kind, const sv_gate *gates, int n, cudaStream_t st, bool tol = false) {
  if (kind == SV_GROUP_LOW) return run_dlow(a, m, gates, n, st, !tol);
  if (kind == SV_GROUP_STAGE2) {
    if (!tol) return fail(SV_EINVAL, "two-phase stage groups run in the tolerance mode only (SV_FLAG_TOLERANCE)");
    int split;
    if (stage2_run(m, gates, n, 0, &split) != n) return fail(SV_EINVAL, "not a two-phase stage group");
    return run_dstage2(a, m, gates, n, split, st);
  }
  if (kind == SV_GROUP_STAGE) {
    if (n == 1) return launch_gate(a, m, gates[0], st);
    // tolerance mode pays off through folds (diagonal gates controlled from outside the
    // targets) and deferred butterflies; a group with neither runs the exact kernel, which is
    // faster on general gates (5 Haar gates at n = 30: 5.1 vs 10.5 ms) and trivially within the bound
    return tol && stage_gains_from_tolerance(gates, n) ? run_dstage(a, m, gates, n, st)
                                                       : run_mstage(a, m, gates, n, st);
  }
  if (kind == SV_GROUP_TILE && T >= 9 && n > 1) {
    const int L = T - TG_BITS;
    int H[TG_BITS], nh = 0;
    for (int k = 0; k < n; ++k) {
      const int tt = gates[k].target;
      bool in = tt < L;
      for (int q = 0; q < nh && !in; ++q) in = H[q] == tt;
      if (!in) {
        if (nh == TG_BITS) return fail(SV_EINVAL, "tile group: more than %d targets above bit %d", TG_BITS, L - 1);
        H[nh++] = tt;
      }
    }
    for (int b = L; nh < TG_BITS; ++b) {  // pad with the natural block bits
      bool dup = false;
      for (int q = 0; q < nh; ++q) dup |= H[q] == b;
      if (!dup) H[nh++] = b;
    }
    std::sort(H, H + TG_BITS);
    return run_tile(a, m, T, H, gates, n, st);
  }
  for (int k = 0; k < n; ++k) {
    const int rc = launch_gate(a, m, gates[k], st);
    if (rc != SV_OK) return rc;
  }
  return SV_OK;
}

int check_gates(const char *who, int m, const sv_gate *gates, int n, int tmax) {
  for (int i = 0; i < n; ++i) {
    const sv_gate &g = gates[i];
    if (g.target < 0 || g.target >= tmax || g.control < -1 || g.control >= m || g.control == g.target)
      return fail(SV_EINVAL, "%s: gate %d (t=%d, c=%d) invalid for m=%d (targets < %d)", who, i, g.target,
                  g.control, m, tmax);
  }
  return SV_OK;
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

int alloc_base(const void *ptr, uintptr_t *base) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !f)
      return fail(SV_ECUDA, "sv_ipc_handle: cuMemGetAddressRange unavailable");
    fn = (PFN_getAddressRange)f;
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  CUresult r = fn(&b, &sz, (CUdeviceptr)(uintptr_t)ptr);
  if (r != CUDA_SUCCESS) return fail(SV_ECUDA, "sv_ipc_handle: address range lookup failed (%d)", (int)r);
  *base = (uintptr_t)b;
  return SV_OK;
}

}  // namespace

// ======================================================================= C ABI

extern "C" {

int sv_version(void) { return SV_ABI_VERSION; }

const char *sv_last_error(void) { return g_err; }

uint64_t sv_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int sv_apply_single(void *amps, int m, int k, const double *q, void *stream) {
  if (bad_ptr(amps) || !q) return fail(SV_EINVAL, "sv_apply_single: null or misaligned pointer");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_apply_single: m=%d out of range", m);
  if (k < 0 || k >= m) return fail(SV_EINVAL, "sv_apply_single: qubit %d not in [0, %d)", k, m);
  return launch_local<MODE_SINGLE>((double2 *)amps, m, k, 0, load_q(q), (cudaStream_t)stream,
                                   "sv_apply_single");
}

int sv_apply_controlled(void *amps, int m, int c, int t, const double *q, void *stream) {
  if (bad_ptr(amps) || !q) return fail(SV_EINVAL, "sv_apply_controlled: null or misaligned pointer");
  if (m < 2 || m > 62) return fail(SV_EINVAL, "sv_apply_controlled: m=%d out of range", m);
  if (c == t) return fail(SV_EINVAL, "sv_apply_controlled: control and target must differ, both are %d", c);
  if (c < 0 || c >= m || t < 0 || t >= m)
    return fail(SV_EINVAL, "sv_apply_controlled: qubits (%d,%d) not in [0, %d)", c, t, m);
  const GateQ g = load_q(q);
  cudaStream_t st = (cudaStream_t)stream;
  if (c == 0) return launch_local<MODE_PRED>((double2 *)amps, m, t, 0, g, st, "sv_apply_controlled");
  const int tv = t < c ? t : t - 1;
  return launch_local<MODE_CTL>((double2 *)amps, m - 1, tv, c, g, st, "sv_apply_controlled");
}

int sv_apply_fused(void *amps, int m, int l, const sv_gate *gates, int ngates, void *stream) {
  if (bad_ptr(amps) || !gates) return fail(SV_EINVAL, "sv_apply_fused: null or misaligned pointer");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_apply_fused: m=%d out of range", m);
  const int lmax = m < SV_FUSED_MAX_TILE ? m : SV_FUSED_MAX_TILE;
  if (l < 1 || l > lmax) return fail(SV_EINVAL, "sv_apply_fused: block exponent %d not in [1, %d]", l, lmax);
  if (ngates < 1 || ngates > SV_FUSED_MAX_GATES)
    return fail(SV_EINVAL, "sv_apply_fused: %d gates not in [1, %d]", ngates, SV_FUSED_MAX_GATES);
  for (int i = 0; i < ngates; ++i) {
    const sv_gate &g = gates[i];
    if (g.target < 0 || g.target >= l || g.control >= l || g.control < -1 || g.control == g.target)
      return fail(SV_EINVAL, "sv_apply_fused: gate %d (t=%d, c=%d) outside block exponent %d", i, g.target,
                  g.control, l);
  }
  // Tile: 2^12 amplitudes per CTA where the slice allows (64 KiB: two CTAs per
  // SM overlap one tile's HBM traffic with the other's gates), never below l.
  const int T = l > 12 ? l : (m < 12 ? m : 12);
  if (T >= 9) {
    int hb[TG_BITS];  // contiguous 2^T blocks
    for (int k = 0; k < TG_BITS; ++k) hb[k] = T - TG_BITS + k;
    return run_tile((double2 *)amps, m, T, hb, gates, ngates, (cudaStream_t)stream);
  }
  static thread_local FusedParams P;  // 18 KB: keep it off the stack
  P.ngates = ngates;
  P.pad = 0;
  for (int i = 0; i < ngates; ++i) P.g[i] = gates[i];
  return launch_fused((double2 *)amps, m, T, P, (cudaStream_t)stream);
}

int sv_apply_gates_ex(void *amps, int m, const sv_gate *gates, int ngates, int tile, int flags, void *stream) {
  if (bad_ptr(amps) || (!gates && ngates)) return fail(SV_EINVAL, "sv_apply_gates: null or misaligned pointer");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_apply_gates: m=%d out of range", m);
  if (ngates < 0) return fail(SV_EINVAL, "sv_apply_gates: negative gate count");
  if (flags & ~SV_FLAG_TOLERANCE) return fail(SV_EINVAL, "sv_apply_gates: unknown flags %#x", flags);
  int rc = check_gates("sv_apply_gates", m, gates, ngates, m);
  if (rc != SV_OK) return rc;
  const int tmax = m < SV_FUSED_MAX_TILE ? m : SV_FUSED_MAX_TILE;
  const int T = tile > 0 ? tile : tmax;
  if (tile != 0 && (tile < 9 || tile > tmax)) return fail(SV_EINVAL, "sv_apply_gates: tile %d not in [9, %d]", tile, tmax);
  const bool tol = flags & SV_FLAG_TOLERANCE;
  int i = 0;
  while (i < ngates && rc == SV_OK) {
    int kind;
    const int j = next_group(m, gates, ngates, i, T, &kind, tol);
    rc = exec_group((double2 *)amps, m, T, kind, gates + i, j - i, (cudaStream_t)stream, tol);
    i = j;
  }
  return rc;
}

int sv_apply_gates(void *amps, int m, const sv_gate *gates, int ngates, int tile, void *stream) {
  return sv_apply_gates_ex(amps, m, gates, ngates, tile, 0, stream);
}

int sv_plan_gates_ex(int m, const sv_gate *gates, int ngates, int tile, int flags, int32_t *group_end,
                     int32_t *group_kind, int max_groups) {
  if ((!gates && ngates) || !group_end || !group_kind) return fail(SV_EINVAL, "sv_plan_gates: null pointer");
  if (m < 1 || m > 62 || ngates < 0) return fail(SV_EINVAL, "sv_plan_gates: m=%d / ngates=%d invalid", m, ngates);
  if (flags & ~SV_FLAG_TOLERANCE) return fail(SV_EINVAL, "sv_plan_gates: unknown flags %#x", flags);
  int rc = check_gates("sv_plan_gates", m, gates, ngates, m);
  if (rc != SV_OK) return rc;
  const int tmax = m < SV_FUSED_MAX_TILE ? m : SV_FUSED_MAX_TILE;
  if (tile != 0 && (tile < 9 || tile > tmax)) return fail(SV_EINVAL, "sv_plan_gates: tile %d not in [9, %d]", tile, tmax);
  const int T = tile > 0 ? tile : tmax;
  int i = 0, ng = 0;
  while (i < ngates) {
    if (ng == max_groups) return fail(SV_EINVAL, "sv_plan_gates: more than %d groups", max_groups);
    int kind;
    i = next_group(m, gates, ngates, i, T, &kind, flags & SV_FLAG_TOLERANCE);
    group_end[ng] = i;
    group_kind[ng] = kind;
    ++ng;
  }
  return ng;
}

int sv_stage_shape(int m, const sv_gate *gates, int ngates) {
  if (!gates) return fail(SV_EINVAL, "sv_stage_shape: null pointer");
  if (m < 1 || m > 62 || ngates < 1) return fail(SV_EINVAL, "sv_stage_shape: m=%d / ngates=%d invalid", m, ngates);
  int rc = check_gates("sv_stage_shape", m, gates, ngates, m);
  if (rc != SV_OK) return rc;
  static thread_local MsParams P;
  XmParams X;
  int compiled = 0;
  rc = build_mstage(m, gates, ngates, P, X, &compiled);
  return rc != SV_OK ? rc : (!compiled ? SV_SHAPE_INTERPRETED : X.inverse ? SV_SHAPE_INVERSE : SV_SHAPE_FORWARD);
}

int sv_stage2_shape(int m, const sv_gate *gates, int ngates) {
  if (!gates) return fail(SV_EINVAL, "sv_stage2_shape: null pointer");
  if (m < 1 || m > 62 || ngates < 2) return fail(SV_EINVAL, "sv_stage2_shape: m=%d / ngates=%d invalid", m, ngates);
  int rc = check_gates("sv_stage2_shape", m, gates, ngates, m);
  if (rc != SV_OK) return rc;
  int split;
  if (stage2_run(m, gates, ngates, 0, &split) != ngates) return fail(SV_EINVAL, "sv_stage2_shape: not a two-phase stage group");
  int s1[MS_K], s2[MS_K], lb[MS_K];
  rc = stage2_slots(m, gates, ngates, split, s1, s2, lb);
  if (rc) return rc;
  static thread_local Xf2Params X;
  static thread_local DtParams T;
  int ng = 0;
  double scale = 1.0;
  return stage2_shape(m, gates, ngates, split, s1, s2, X, T, &ng, &scale);
}

int sv_plan_gates(int m, const sv_gate *gates, int ngates, int tile, int32_t *group_end, int32_t *group_kind,
                  int max_groups) {
  return sv_plan_gates_ex(m, gates, ngates, tile, 0, group_end, group_kind, max_groups);
}

int sv_apply_group_ex(void *amps, int m, int kind, const sv_gate *gates, int ngates, int tile, int flags,
                      void *stream) {
  if (bad_ptr(amps) || !gates) return fail(SV_EINVAL, "sv_apply_group: null or misaligned pointer");
  if (m < 1 || m > 62 || ngates < 1) return fail(SV_EINVAL, "sv_apply_group: m=%d / ngates=%d invalid", m, ngates);
  if (flags & ~SV_FLAG_TOLERANCE) return fail(SV_EINVAL, "sv_apply_group: unknown flags %#x", flags);
  int rc = check_gates("sv_apply_group", m, gates, ngates, m);
  if (rc != SV_OK) return rc;
  const int tmax = m < SV_FUSED_MAX_TILE ? m : SV_FUSED_MAX_TILE;
  if (tile != 0 && (tile < 9 || tile > tmax)) return fail(SV_EINVAL, "sv_apply_group: tile %d not in [9, %d]", tile, tmax);
  if (kind < SV_GROUP_GATES || kind > SV_GROUP_STAGE2) return fail(SV_EINVAL, "sv_apply_group: kind %d", kind);
  return exec_group((double2 *)amps, m, tile > 0 ? tile : tmax, kind, gates, ngates, (cudaStream_t)stream,
                    flags & SV_FLAG_TOLERANCE);
}

int sv_apply_group(void *amps, int m, int kind, const sv_gate *gates, int ngates, int tile, void *stream) {
  return sv_apply_group_ex(amps, m, kind, gates, ngates, tile, 0, stream);
}

int sv_exchange_stage(void *mine, void *theirs, int m, int own_is_zero, const sv_gate *gates, int ngates,
                      void *stream) {
  if (bad_ptr(mine) || bad_ptr(theirs) || !gates)
    return fail(SV_EINVAL, "sv_exchange_stage: null or misaligned pointer");
  if (mine == theirs) return fail(SV_EINVAL, "sv_exchange_stage: partner slice aliases the local slice");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_exchange_stage: m=%d out of range", m);
  if (ngates < 1 || ngates > STAGE_MAX_GATES)
    return fail(SV_EINVAL, "sv_exchange_stage: %d gates not in [1, %d]", ngates, STAGE_MAX_GATES);
  static thread_local StageParams P;
  P.ngates = ngates;
  for (int i = 0; i < ngates; ++i) {
    if (gates[i].control < -1 || gates[i].control >= m)
      return fail(SV_EINVAL, "sv_exchange_stage: gate %d control %d is not a local qubit", i, gates[i].control);
    P.g[i].cmask = gates[i].control >= 0 ? (1ull << gates[i].control) : 0ull;
    P.g[i].kind = classify_kind(gates[i].q);
    memcpy(P.g[i].q, gates[i].q, sizeof(P.g[i].q));
  }
  const uint64_t half = 1ull << (m - 1);
  const unsigned grid = grid_for(half, BLK * SUNROLL);
  if (stage_sig(P) == 1)
    k_exchange_stage<1><<<grid, BLK, 0, (cudaStream_t)stream>>>((double2 *)mine, (double2 *)theirs, half,
                                                                own_is_zero ? 0 : half, own_is_zero ? 1 : 0, P);
  else
    k_exchange_stage<0><<<grid, BLK, 0, (cudaStream_t)stream>>>((double2 *)mine, (double2 *)theirs, half,
                                                                own_is_zero ? 0 : half, own_is_zero ? 1 : 0, P);
  return after_launch("sv_exchange_stage");
}

int sv_swap_global(void *mine, void *theirs, int m, int own_is_zero, int l, void *stream) {
  if (bad_ptr(mine) || bad_ptr(theirs)) return fail(SV_EINVAL, "sv_swap_global: null or misaligned pointer");
  if (mine == theirs) return fail(SV_EINVAL, "sv_swap_global: partner slice aliases the local slice");
  if (m < 2 || m > 62) return fail(SV_EINVAL, "sv_swap_global: m=%d out of range", m);
  if (l < 0 || l >= m) return fail(SV_EINVAL, "sv_swap_global: qubit %d not local (m=%d)", l, m);
  const uint64_t quarter = 1ull << (m - 2);  // each side swaps half of the 2^(m-1) pairs
  k_swap_global<<<grid_for(quarter, BLK * UNROLL), BLK, 0, (cudaStream_t)stream>>>(
      (double2 *)mine, (double2 *)theirs, quarter, own_is_zero ? 0 : quarter, l, own_is_zero ? 0 : 1);
  return after_launch("sv_swap_global");
}

int sv_exchange(void *mine, void *theirs, int m, int own_is_zero, int c_local, const double *q, void *stream) {
  if (bad_ptr(mine) || bad_ptr(theirs) || !q) return fail(SV_EINVAL, "sv_exchange: null or misaligned pointer");
  if (mine == theirs) return fail(SV_EINVAL, "sv_exchange: partner slice aliases the local slice");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_exchange: m=%d out of range", m);
  if (c_local < -1 || c_local >= m) return fail(SV_EINVAL, "sv_exchange: control %d not local (m=%d)", c_local, m);
  const uint64_t half = 1ull << (m - 1);
  const uint64_t base = own_is_zero ? 0 : half;
  uint64_t count;
  int cmap = c_local;
  if (c_local < 0) {
    count = half;
  } else if (c_local == m - 1) {  // the half-selecting bit: all of the second half, none of the first
    count = own_is_zero ? 0 : half;
    cmap = -1;
  } else {
    count = half >> 1;
  }
  if (count == 0) return SV_OK;
  k_exchange<<<grid_for(count, BLK * UNROLL), BLK, 0, (cudaStream_t)stream>>>(
      (double2 *)mine, (double2 *)theirs, count, base, cmap, own_is_zero ? 1 : 0, load_q(q));
  return after_launch("sv_exchange");
}

int diag_check(const char *who, void *amps, int m, int c_local, const double *q) {
  if (bad_ptr(amps) || !q) return fail(SV_EINVAL, "%s: null or misaligned pointer", who);
  if (m < 1 || m > 62) return fail(SV_EINVAL, "%s: m=%d out of range", who, m);
  if (c_local < -1 || c_local >= m) return fail(SV_EINVAL, "%s: control %d not local (m=%d)", who, c_local, m);
  if (!(q[2] == 0.0 && q[3] == 0.0 && q[4] == 0.0 && q[5] == 0.0))
    return fail(SV_EINVAL, "%s: gate is not diagonal (q12 and q21 must be exactly zero)", who);
  return SV_OK;
}

int sv_diag_global(void *amps, int m, int own_is_zero, int c_local, const double *q, void *signs, int *flag,
                   void *stream) {
  int rc = diag_check("sv_diag_global", amps, m, c_local, q);
  if (rc != SV_OK) return rc;
  if (!signs || !flag) return fail(SV_EINVAL, "sv_diag_global: null sign map or flag");
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(SV_ECUDA, "sv_diag_global: %s", cudaGetErrorString(e));
  const double dr = own_is_zero ? q[0] : q[6], di = own_is_zero ? q[1] : q[7];
  k_diag_global<<<fill_grid(1ull << m), BLK, 0, (cudaStream_t)stream>>>((double2 *)amps, 1ull << m, c_local, dr, di,
                                                                        (uint32_t *)signs, flag);
  return after_launch("sv_diag_global");
}

int sv_diag_fix(void *amps, int m, int own_is_zero, int c_local, const double *q, const void *partner_signs,
                const int *flag, void *stream) {
  int rc = diag_check("sv_diag_fix", amps, m, c_local, q);
  if (rc != SV_OK) return rc;
  if (!partner_signs || !flag) return fail(SV_EINVAL, "sv_diag_fix: null sign map or flag");
  const double zr = own_is_zero ? q[2] : q[4], zi = own_is_zero ? q[3] : q[5];
  k_diag_fix<<<fill_grid(1ull << m), BLK, 0, (cudaStream_t)stream>>>((double2 *)amps, 1ull << m, c_local, zr, zi,
                                                                     (const uint32_t *)partner_signs, flag);
  return after_launch("sv_diag_fix");
}

int sv_exchange_chunk(void *mine, void *buf, int m, int own_is_zero, int c_local, const double *q, uint64_t j0,
                      uint64_t count_j, void *stream) {
  if (bad_ptr(mine) || bad_ptr(buf) || !q) return fail(SV_EINVAL, "sv_exchange_chunk: null or misaligned pointer");
  if (m < 1 || m > 62) return fail(SV_EINVAL, "sv_exchange_chunk: m=%d out of range", m);
  if (c_local < -1 || c_local >= m - 1)
    return fail(SV_EINVAL, "sv_exchange_chunk: control %d not an interior local bit (m=%d)", c_local, m);
  const uint64_t half = 1ull << (m - 1), lo = own_is_zero ? 0 : half;
  if (count_j == 0) return SV_OK;
  if (j0 < lo || j0 + count_j > lo + half) return fail(SV_EINVAL, "sv_exchange_chunk: range outside own half");
  const uint64_t align = c_local >= 0 ? (2ull << c_local) : 1ull;
  if (j0 % align || count_j % align) return fail(SV_EINVAL, "sv_exchange_chunk: range not aligned to 2^(c+1)");
  const uint64_t count = c_local >= 0 ? count_j >> 1 : count_j;
  // k_exchange addresses theirs[j]: shift the chunk buffer so that buf[0] is element j0
  double2 *theirs = (double2 *)buf - j0;
  k_exchange<<<grid_for(count, BLK * UNROLL), BLK, 0, (cudaStream_t)stream>>>(
      (double2 *)mine, theirs, count, j0, c_local, own_is_zero ? 1 : 0, load_q(q));
  return after_launch("sv_exchange_chunk");
}

int sv_pair_update(void *mine, void *theirs, uint64_t count, int own_is_zero, const double *q, void *stream) {
  if (bad_ptr(mine) || bad_ptr(theirs) || !q) return fail(SV_EINVAL, "sv_pair_update: null or misaligned pointer");
  if (mine == theirs) return fail(SV_EINVAL, "sv_pair_update: the two chunks alias");
  if (count == 0) return SV_OK;
  k_exchange<<<grid_for(count, BLK * UNROLL), BLK, 0, (cudaStream_t)stream>>>(
      (double2 *)mine, (double2 *)theirs, count, 0, -1, own_is_zero ? 1 : 0, load_q(q));
  return after_launch("sv_pair_update");
}

int sv_norm_sq(const void *amps, int m, int qubit, double *scratch, void *stream) {
  if (bad_ptr(amps) || !scratch) return fail(SV_EINVAL, "sv_norm_sq: null or misaligned pointer");
  if (m < 0 || m > 62) return fail(SV_EINVAL, "sv_norm_sq: m=%d out of range", m);
  if (qubit < -1 || qubit >= m) return fail(SV_EINVAL, "sv_norm_sq: qubit %d not local (m=%d)", qubit, m);
  cudaStream_t st = (cudaStream_t)stream;
  k_norm_partial<<<NORM_BLOCKS, BLK, 0, st>>>((const double2 *)amps, 1ull << m, qubit, scratch);
  k_norm_final<<<1, BLK, 0, st>>>(scratch);
  return after_launch("sv_norm_sq", 2);
}

int sv_max_abs_diff(const void *a, const void *b, int m, double *scratch, void *stream) {
  if (bad_ptr(a) || bad_ptr(b) || !scratch) return fail(SV_EINVAL, "sv_max_abs_diff: null or misaligned pointer");
  if (m < 0 || m > 62) return fail(SV_EINVAL, "sv_max_abs_diff: m=%d out of range", m);
  cudaStream_t st = (cudaStream_t)stream;
  k_maxdiff_partial<<<NORM_BLOCKS, BLK, 0, st>>>((const double2 *)a, (const double2 *)b, 1ull << m, scratch);
  k_max_final<<<1, BLK, 0, st>>>(scratch);
  return after_launch("sv_max_abs_diff", 2);
}

int sv_init_random(void *amps, int m, uint64_t seed, uint64_t rank, void *stream) {
  if (bad_ptr(amps)) return fail(SV_EINVAL, "sv_init_random: null or misaligned pointer");
  if (m < 0 || m > 62) return fail(SV_EINVAL, "sv_init_random: m=%d out of range", m);
  const uint64_t n = 1ull << m;
  k_init_random<<<grid_for(n, BLK), BLK, 0, (cudaStream_t)stream>>>((double2 *)amps, n, rank << m, seed);
  return after_launch("sv_init_random");
}

int sv_scale(void *amps, int m, double s, void *stream) {
  if (bad_ptr(amps)) return fail(SV_EINVAL, "sv_scale: null or misaligned pointer");
  if (m < 0 || m > 62) return fail(SV_EINVAL, "sv_scale: m=%d out of range", m);
  const uint64_t n = 1ull << m;
  k_scale<<<fill_grid(n), BLK, 0, (cudaStream_t)stream>>>((double2 *)amps, n, s);
  return after_launch("sv_scale");
}

int sv_init_basis(void *amps, int m, int64_t local, void *stream) {
  if (bad_ptr(amps)) return fail(SV_EINVAL, "sv_init_basis: null or misaligned pointer");
  if (m < 0 || m > 62) return fail(SV_EINVAL, "sv_init_basis: m=%d out of range", m);
  const uint64_t n = 1ull << m;
  if (local >= (int64_t)n) return fail(SV_EINVAL, "sv_init_basis: index %lld outside slice", (long long)local);
  k_basis<<<fill_grid(n), BLK, 0, (cudaStream_t)stream>>>((double2 *)amps, n, local);
  return after_launch("sv_init_basis");
}

int sv_copy(void *dst, const void *src, uint64_t nbytes, void *stream) {
  if (!dst || !src) return fail(SV_EINVAL, "sv_copy: null pointer");
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)nbytes, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(SV_ECUDA, "sv_copy: %s", cudaGetErrorString(e));
  return SV_OK;
}

int sv_ipc_handle(const void *ptr, void *handle_out, uint64_t *offset_out) {
  if (!ptr || !handle_out || !offset_out) return fail(SV_EINVAL, "sv_ipc_handle: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  uintptr_t base = 0;
  int rc = alloc_base(ptr, &base);
  if (rc != SV_OK) return rc;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
  if (e != cudaSuccess) return fail(SV_ECUDA, "sv_ipc_handle: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((uintptr_t)ptr - base);
  return SV_OK;
}

int sv_ipc_open(const void *handle, uint64_t offset, void **ptr_out) {
  if (!handle || !ptr_out) return fail(SV_EINVAL, "sv_ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void *p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SV_ECUDA, "sv_ipc_open: %s", cudaGetErrorString(e));
  *ptr_out = (void *)((uintptr_t)p + offset);
  return SV_OK;
}

int sv_ipc_close(void *ptr, uint64_t offset) {
  if (!ptr) return fail(SV_EINVAL, "sv_ipc_close: null pointer");
  cudaError_t e = cudaIpcCloseMemHandle((void *)((uintptr_t)ptr - offset));
  if (e != cudaSuccess) return fail(SV_ECUDA, "sv_ipc_close: %s", cudaGetErrorString(e));
  return SV_OK;
}

}  // extern "C"
