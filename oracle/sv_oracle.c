/*
 * sv_oracle.c -- CPU restatement of the reference's gate arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, as the checker or as the timed
 * CPU baseline.  Parity is pinned: tests/test_oracle_golden.py compares it
 * bit-for-bit against vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/svsim).
 *
 * Arithmetic (the part that decides bitwise parity)
 * -------------------------------------------------
 * The reference evaluates every pair update with numpy ufuncs
 * (pkg/src/svsim/kernels.py:120-131):
 *
 *     new0 = mix(a0, a1, q11, q12);  new1 = mix(a0, a1, q21, q22)
 *     mix(a0, a1, r0, r1):  out = r0*a0 ; out += r1*a1
 *
 * numpy 2.x's SIMD complex multiply (scalar * array) rounds as
 *
 *     re = fma(r.re, a.re, -(a.im * r.im))
 *     im = fma(r.re, a.im,  (a.re * r.im))
 *
 * (probed in this container: numpy 2.3.5, AVX512/FMA3 dispatch, bit-exact on
 * every k and view shape the kernels use), followed by an exact-per-component
 * complex add.  This file reproduces that rounding sequence with explicit
 * fma() and -ffp-contract=off, so its results equal the reference's bit for
 * bit; the CUDA kernels use the same sequence (__fma_rn / __dmul_rn).
 *
 * Index maps follow the reference's strided views:
 *   single      kernels.py:174-176  pairs (i, i + 2^k), bit k of i clear
 *   controlled  kernels.py:179-184  pairs with bit c set, bit t in {0,1}
 *   block run   kernels.py:225-240 + fusion.py:124-135  gates in order per
 *               contiguous 2^l block
 *   exchange    distributed.py:187-202 (_pair_kernel), :293-311, :341-422
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  double re, im;
} c128;

typedef struct {
  int32_t target;
  int32_t control; /* -1: no control */
  double q[8];     /* q11re q11im q12re q12im q21re q21im q22re q22im */
} or_gate;

/* numpy complex multiply of scalar r by element a (see header). */
static inline c128 cmul(double rr, double ri, c128 a) {
  c128 o;
  o.re = fma(rr, a.re, -(a.im * ri));
  o.im = fma(rr, a.im, a.re * ri);
  return o;
}

/* mix() of kernels.py:120-124: r0*a0 then += r1*a1. */
static inline c128 mix(c128 a0, c128 a1, double r0r, double r0i, double r1r, double r1i) {
  c128 x = cmul(r0r, r0i, a0);
  c128 y = cmul(r1r, r1i, a1);
  c128 o;
  o.re = x.re + y.re;
  o.im = x.im + y.im;
  return o;
}

static inline void pair_update(c128 *p0, c128 *p1, const double *q) {
  c128 a0 = *p0, a1 = *p1;
  c128 n0 = mix(a0, a1, q[0], q[1], q[2], q[3]);
  c128 n1 = mix(a0, a1, q[4], q[5], q[6], q[7]);
  *p0 = n0;
  *p1 = n1;
}

static inline uint64_t insert_zero(uint64_t x, int b) {
  uint64_t lo = x & ((1ull << b) - 1);
  return ((x >> b) << (b + 1)) | lo;
}

static int clamp_threads(int threads) { return threads < 1 ? 1 : threads; }

/* kernels.py:187-189 apply_single_raw */
void or_apply_single(double *amps_d, int m, int k, const double *q, int threads) {
  c128 *amps = (c128 *)amps_d;
  int64_t npairs = (int64_t)1 << (m - 1);
  uint64_t stride = 1ull << k;
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t p = 0; p < npairs; ++p) {
    uint64_t i0 = insert_zero((uint64_t)p, k);
    pair_update(&amps[i0], &amps[i0 | stride], q);
  }
}

/* kernels.py:192-196 apply_controlled_raw */
void or_apply_controlled(double *amps_d, int m, int c, int t, const double *q, int threads) {
  c128 *amps = (c128 *)amps_d;
  int lo = c < t ? c : t, hi = c < t ? t : c;
  int64_t npairs = (int64_t)1 << (m - 2);
  uint64_t cbit = 1ull << c, tbit = 1ull << t;
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t p = 0; p < npairs; ++p) {
    uint64_t i0 = insert_zero(insert_zero((uint64_t)p, lo), hi) | cbit;
    pair_update(&amps[i0], &amps[i0 | tbit], q);
  }
}

static void block_apply_gate(c128 *blk, int b, const or_gate *g) {
  if (g->control < 0) {
    uint64_t npairs = 1ull << (b - 1), stride = 1ull << g->target;
    for (uint64_t p = 0; p < npairs; ++p) {
      uint64_t i0 = insert_zero(p, g->target);
      pair_update(&blk[i0], &blk[i0 | stride], g->q);
    }
  } else {
    int c = g->control, t = g->target;
    int lo = c < t ? c : t, hi = c < t ? t : c;
    uint64_t npairs = 1ull << (b - 2);
    for (uint64_t p = 0; p < npairs; ++p) {
      uint64_t i0 = insert_zero(insert_zero(p, lo), hi) | (1ull << c);
      pair_update(&blk[i0], &blk[i0 | (1ull << t)], g->q);
    }
  }
}

/* fusion.py:124-135 FusedBlockRun: every 2^l block gets apply_block(gates). */
void or_apply_block_run(double *amps_d, int m, int l, const or_gate *gates, int ngates,
                        int threads) {
  c128 *amps = (c128 *)amps_d;
  int64_t nblocks = (int64_t)1 << (m - l);
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t blk = 0; blk < nblocks; ++blk) {
    c128 *base = amps + ((uint64_t)blk << l);
    for (int g = 0; g < ngates; ++g) block_apply_gate(base, l, &gates[g]);
  }
}

/*
 * One rank's share of a half exchange (distributed.py:187-202, :293-311,
 * :404-422), with the partner's slice addressed directly instead of through
 * messages.  The computing rank owns half `own_is_zero ? 0 : 1` of the pair
 * space; for every local index j of that half (restricted to local bit c set
 * when c_local >= 0) it reads mine[j] and theirs[j], keeps one output and
 * writes the other back into theirs[j], with the same operand order as the
 * reference's _pair_kernel.
 */
void or_exchange(double *mine_d, double *theirs_d, int m, int own_is_zero, int c_local,
                 const double *q, int threads) {
  c128 *mine = (c128 *)mine_d, *theirs = (c128 *)theirs_d;
  uint64_t half = 1ull << (m - 1);
  uint64_t base = own_is_zero ? 0 : half;
  int64_t count;
  if (c_local < 0) {
    count = (int64_t)half;
  } else if (c_local == m - 1) {
    count = own_is_zero ? 0 : (int64_t)half;
  } else {
    count = (int64_t)(half >> 1);
  }
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t p = 0; p < count; ++p) {
    uint64_t j;
    if (c_local < 0 || c_local == m - 1)
      j = base + (uint64_t)p;
    else
      j = base + (insert_zero((uint64_t)p, c_local) | (1ull << c_local));
    c128 a_m = mine[j], a_t = theirs[j], keep, ret;
    if (own_is_zero) {
      keep = mix(a_m, a_t, q[0], q[1], q[2], q[3]);
      ret = mix(a_m, a_t, q[4], q[5], q[6], q[7]);
    } else {
      keep = mix(a_t, a_m, q[4], q[5], q[6], q[7]);
      ret = mix(a_t, a_m, q[0], q[1], q[2], q[3]);
    }
    mine[j] = keep;
    theirs[j] = ret;
  }
}

/* The same update restricted to local indices j0 .. j0+count-1 of the computing
 * half, with the partner's elements staged contiguously in buf (buf[0] = element
 * j0): the NCCL data plane's chunk step (distributed.py:257-287). */
void or_exchange_chunk(double *mine_d, double *buf_d, int m, int own_is_zero, int c_local, const double *q,
                       int64_t j0, int64_t count) {
  c128 *mine = (c128 *)mine_d, *buf = (c128 *)buf_d;
  (void)m;
  for (int64_t j = j0; j < j0 + count; ++j) {
    if (c_local >= 0 && !(((uint64_t)j >> c_local) & 1)) continue;
    c128 a_m = mine[j], a_t = buf[j - j0], keep, ret;
    if (own_is_zero) {
      keep = mix(a_m, a_t, q[0], q[1], q[2], q[3]);
      ret = mix(a_m, a_t, q[4], q[5], q[6], q[7]);
    } else {
      keep = mix(a_t, a_m, q[4], q[5], q[6], q[7]);
      ret = mix(a_t, a_m, q[0], q[1], q[2], q[3]);
    }
    mine[j] = keep;
    buf[j - j0] = ret;
  }
}

/* Sum of |a|^2 over the slice, or over bit `qubit` = 1 when qubit >= 0
 * (core.py:147-167).  Reduction order differs from numpy's pairwise sum, so
 * this is compared within tolerance, never bitwise. */
double or_norm_sq(const double *amps_d, int m, int qubit, int threads) {
  const c128 *amps = (const c128 *)amps_d;
  int64_t n = (int64_t)1 << m;
  double acc = 0.0;
  (void)threads;
#pragma omp parallel for schedule(static) reduction(+ : acc) num_threads(clamp_threads(threads))
  for (int64_t i = 0; i < n; ++i) {
    if (qubit >= 0 && !(((uint64_t)i >> qubit) & 1)) continue;
    acc += amps[i].re * amps[i].re + amps[i].im * amps[i].im;
  }
  return acc;
}

/* Deterministic, cheap fill for CPU-baseline timing buffers (values are not
 * a parity input; they only need to be finite and normalised-ish). */
void or_fill_phase(double *amps_d, int m, int threads) {
  c128 *amps = (c128 *)amps_d;
  int64_t n = (int64_t)1 << m;
  double s = 1.0 / sqrt((double)n);
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t i = 0; i < n; ++i) {
    double ph = (double)(i & 1023) * (6.283185307179586 / 1024.0);
    amps[i].re = s * cos(ph);
    amps[i].im = s * sin(ph);
  }
}

/* The seeded state of the GPU arm (sv_init_random: Philox4x32-10 with the global
 * index as counter, Box-Muller), unnormalised, for the CPU reference arm's input.
 * libm's log/sincos may differ from CUDA's in the last ulp: same distribution and
 * seed, not a parity vector. */
static void philox4x32(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

void or_fill_philox(double *amps_d, int m, uint64_t gbase, uint64_t seed, int threads) {
  c128 *amps = (c128 *)amps_d;
  int64_t n = (int64_t)1 << m;
#pragma omp parallel for schedule(static) num_threads(clamp_threads(threads))
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t g = gbase + (uint64_t)i;
    uint32_t c[4] = {(uint32_t)g, (uint32_t)(g >> 32), 0x51u, 0x7u};
    philox4x32(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t b1 = ((uint64_t)c[0] << 32) | c[1], b2 = ((uint64_t)c[2] << 32) | c[3];
    const double u1 = ((double)(b1 >> 11) + 1.0) * 0x1.0p-53, u2 = (double)(b2 >> 11) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    amps[i].re = rad * cos(6.283185307179586 * u2);
    amps[i].im = rad * sin(6.283185307179586 * u2);
  }
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
