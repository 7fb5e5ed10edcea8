// sgp4b.cu — B200 (sm_100a) SGP4 near-Earth batch propagator.
//
// Kernels
//   init_kernel        1 thread / satellite, fp64.  _sgp4_init, kernel.py:154-322
//   pack_kernel        1 thread / satellite.  SoA satrec -> packed record
//   grid_kernel<T>     persistent, 16 warps / SM; a warp walks (satellite,
//                      128-step chunk) items row by row (4 steps per lane in
//                      fp32, 1 per lane x 4 in fp64): _propagate +
//                      solve_kepler + merge, kernel.py:325-534, over the dense
//                      grid of propagate_batch, batch.py:166-205
//   (pairs)            sgp4_propagate's broadcasting form (kernel.py:513-534)
//                      runs through grid_kernel as P one-step rows
//   kepler_kernel<T>   solve_kepler, kernel.py:325-349
//   code_rows_kernel   which rows of a code plane hold a nonzero code
//   tle_columns_kernel TLE catalogue decode (parse_catalog_columns)
//   drift_norms_kernel, drift_pct_kernel   drift_report, drift.py:46-100
//
// Numerics
//   * fp64 cells keep the reference's guards, thresholds and code
//     precedence; they depart from its operation order only far below the
//     1 mm / 1e-6 km/s budget: per-satellite products folded into the
//     record, sin/cos from a shared-memory table plus a short polynomial,
//     small corrections applied as rotations, straight-line fast cells for
//     Kepler classes 1 and 2 with a per-cell fallback to the general cell.
//   * fp32 cells are the throughput path: per-satellite work is hoisted into
//     the packed record at init time (computed in fp64, rounded once), the
//     secular angle is formed in double-float (hi/lo pairs) and reduced
//     mod 2*pi before anything is rounded to fp32, sin/cos/rcp/rsqrt use the
//     SFU (MUFU) pipe, Kepler runs a warp-uniform fixed iteration count
//     chosen from the satellite's eccentricity, atan2 and three of the
//     sincos evaluations of the short-period stage are replaced by exact
//     rotations by small angles, and cells run as packed dual-fp32 pairs.
//   * Error codes follow _first_error precedence 2 > 1 > 4 > 6 and the
//     init-code merge of kernel.py:497-502, 529-534.

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <float.h>
#include <stdio.h>
#include <stdarg.h>
#include <math_constants.h>
#include <type_traits>
#include <algorithm>

#include "../../include/sgp4b.h"

// helpers used only by the non-default build knobs below
#pragma nv_diag_suppress 177

// build-time tuning knobs (defaults are the shipped configuration; the
// alternatives measured slower, DESIGN.md §5/§8).  Analysis-only builds:
// SGP4B_NOSTORE (compute without the output stores) and
// SGP4B_ONLY_CLASS_K1 (one class instance, for tools/sass_mix.sh).
#ifndef SGP4B_SMEM_REC
#define SGP4B_SMEM_REC 0          // fp32 records in shared memory (default: registers)
#endif
#ifndef SGP4B_SHFL_REC
#define SGP4B_SHFL_REC 0          // fp32 records spread over the warp (shfl at use)
#endif
#ifndef SGP4B_SEC64
#define SGP4B_SEC64 0             // fp32 secular angle on the FP64 pipe (see secular_angle64)
#endif
#ifndef SGP4B_K2_SERIES
#define SGP4B_K2_SERIES 1           // class-2 (e < 0.1) series for 1/pl_lp, 1/den, 1/(1+betal)
#endif
#ifndef SGP4B_F64_DRAG32
#define SGP4B_F64_DRAG32 1          // fp64 class-1 cell: drag trig/cubic on the SFU/FP32 pipes
#endif
#ifndef SGP4B_MINB64
#define SGP4B_MINB64 1
#endif
constexpr int kGridMinBlocks64 = SGP4B_MINB64; // resident blocks per SM (fp64)

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kInvTwoPi = 0.15915494309189533576888376337251;
constexpr double kX2o3 = 2.0 / 3.0;
constexpr double kPi = 3.14159265358979323846264338327950;

// 2*pi split for float Cody-Waite reduction: hi has 8 trailing zero bits so
// k*hi is exact for |k| < 2^8 ... we rely on fmaf exactness instead (see
// reduce2pi_f): hi is the float nearest 2*pi, lo the float nearest the rest.
constexpr float kTwoPiHiF = 6.28318548202514648437f;     // float(2*pi)
constexpr float kTwoPiLoF = -1.7484556000744487e-07f;    // 2*pi - hi
constexpr float kInvTwoPiF = 0.159154943091895335768883763372514f;
constexpr float kRoundMagicF = 12582912.0f;                // 1.5 * 2^23

struct Grav {
  double mu, re, xke, tumin, j2, j3, j4, j3oj2;
  // derived on the host once per launch (propagate kernels)
  double vkm;                                    // re * xke / 60
  double inv_xke;
  float xke_f, re_f, vkm_f, inv_xke_f, half_j2_f;
};

// ---- SoA satrec fields: SatInit float fields in dataclass order --------
// kernel.py:68-107
enum Field {
  F_NO_KOZAI = 0, F_ECCO, F_INCLO, F_NODEO, F_ARGPO, F_MO, F_BSTAR,
  F_NO_UNKOZAI, F_AO, F_CON41, F_X1MTH2, F_X7THM1,
  F_MDOT, F_ARGPDOT, F_NODEDOT, F_NODECF,
  F_CC1, F_CC4, F_CC5, F_D2, F_D3, F_D4, F_T2COF, F_T3COF, F_T4COF, F_T5COF,
  F_ETA, F_OMGCOF, F_XMCOF, F_DELMO, F_SINMAO, F_AYCOF, F_XLCOF,
  F_COUNT
};
static_assert(F_COUNT == SGP4B_SATREC_FIELDS, "satrec field count");

// ---- packed propagate record (one per satellite, 40 T slots) ----------
enum Slot {
  S_MO = 0, S_MDOT, S_ARGPO, S_ARGPDOT, S_NODEO, S_NODEDOT, S_NODECF, S_CC1,
  S_BC4, S_T2COF, S_OMGCOF, S_ETA, S_XMCOF, S_DELMO, S_D2, S_D3,
  S_D4, S_BC5, S_SINMAO, S_T3COF, S_T4COF, S_T5COF, S_NO, S_AM0,
  S_ECCO, S_INCLO, S_SINIO, S_COSIO, S_AYCOF, S_XLCOF, S_CON41, S_X1MTH2,
  S_X7THM1, S_FLAGS,
  // fp32 double-float secular support (low words; zero in fp64 records)
  S_MDOT_LO, S_ARGPDOT_LO, S_NODEDOT_LO, S_UDOT, S_UDOT_LO, S_U0,
  S_COUNT
};
// fp64 records re-use the (fp32-only) low-word slots
constexpr int S64_SQAM0 = S_MDOT_LO;       // sqrt((xke/no)^(2/3))
constexpr int S64_NOSAFE = S_ARGPDOT_LO;   // xke / am0^1.5 (= no, or 1e-4 if no <= 0)
static_assert(S_COUNT == SGP4B_RECORD_SLOTS, "record slot count");

// fp32 records have their own layout: per-satellite products the fp32 cell
// would otherwise form per cell, computed in fp64 at pack time and rounded
// once (store_record<float>).  The flags word sits at S_FLAGS in both.
enum Slot32 {
  P_MO = 0, P_MDOT,                 // kept for inspection; the cell derives xmdf from U0/UDOT
  P_ARGPO, P_ARGPDOT, P_NODEO, P_NODEDOT, P_NODECF,
  P_UDOT, P_UDOT_LO, P_U0,          // (mdot + argpdot) as hi + lo, (mo + argpo) in [-pi, pi)
  P_A0, P_A1, P_A2, P_A3, P_OMGCOF, // delm: xmcof ((1 + eta x)^3 - delmo) = A0 + A1 x + A2 x^2 + A3 x^3
  P_S, P_SC1, P_SD2, P_SD3, P_SD4,  // s, -s cc1, -s d2, -s d3, -s d4 with s = sqrt((xke/no)^(2/3))
  P_N2, P_N3, P_N4, P_N5,           // no t2cof .. no t5cof
  P_E0, P_BC4, P_BC5,               // ecco + bstar cc5 sinmao, bstar cc4, bstar cc5
  P_AYCOF, P_XLCOF,
  P_K41R, P_KXR, P_QX, P_C15CO,     // -1.5 con41 hj2 re, 0.5 x1mth2 hj2 re, -0.25 x7thm1 hj2, 1.5 cosio hj2
  P_FLAGS,
  P_C15CS, P_X1V, P_C41V,           // 1.5 cosio sinio hj2, x1mth2 hj2 vkm, 1.5 con41 hj2 vkm
  P_SINIO, P_COSIO,
  P_COUNT
};
static_assert((int)P_FLAGS == (int)S_FLAGS, "fp32 flags slot");
static_assert((int)P_COUNT <= (int)S_COUNT, "fp32 record fits the packed slot count");

// fp64 records: the same folding as fp32 (every per-satellite product the
// reference forms per cell is computed once at pack time), kept in fp64.
enum Slot64 {
  Q_ARGPO = 0, Q_ARGPDOT, Q_NODEO, Q_NODEDOT, Q_NODECF, Q_MO, Q_MDOT,
  Q_U0, Q_UDOT,                         // (mo + argpo) mod 2pi, mdot + argpdot
  Q_S, Q_SC1, Q_SD2, Q_SD3, Q_SD4,      // sqrt(am) = s (1 - cc1 t - d2 t^2 - d3 t^3 - d4 t^4)
  Q_N2, Q_N3, Q_N4, Q_N5,               // no t2cof .. no t5cof
  Q_A0, Q_A1, Q_A2, Q_A3, Q_OMGCOF,     // drag cubic in cos xmdf (as P_A0..P_A3)
  Q_E0, Q_BC4, Q_BC5,                   // ecco + bstar cc5 sinmao, bstar cc4, bstar cc5
  Q_AYCOF, Q_XLCOF,
  Q_K41R, Q_KXR, Q_QX, Q_C15CO, Q_C15CS, Q_X1V, Q_C41V,   // as the P_ factors
  Q_SINIO, Q_COSIO, Q_INCLO,
  Q_FLAGS,
  Q_COUNT
};
static_assert((int)Q_COUNT <= (int)S_COUNT, "fp64 record fits the packed slot count");

// flags word
constexpr int FLAG_ISIMP = 1;
constexpr int FLAG_BAD_NM = 2;
constexpr int KEPLER_SHIFT = 4;   // 4 bits: fixed Kepler iterations (fp32)
constexpr int CODE_SHIFT = 8;     // 23 bits: persistent init code (0 .. 2^23 - 1)

// ---- error plumbing ----------------------------------------------------
thread_local char g_last_error[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(SGP4B_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return SGP4B_OK;
}

// ======================================================================
// fp64 helpers with the reference's select semantics
// ======================================================================

// dmath.maximum(x, floor) == where(x >= floor, x, floor)   dmath.py:213-215
__device__ __forceinline__ double gmax(double x, double f) { return x >= f ? x : f; }

// C fmod(x, 2*pi), exact: with the right integer quotient q the remainder
// x - q*2pi is representable, so one fma produces it without rounding.
__device__ __forceinline__ double fmod_2pi(double x) {
  if (!(fabs(x) < 1.0e15)) return fmod(x, kTwoPi);
  double q = trunc(x * kInvTwoPi);
  double r = fma(-q, kTwoPi, x);
  if (x >= 0.0) {
    if (r < 0.0) { q -= 1.0; r = fma(-q, kTwoPi, x); }
    else if (r >= kTwoPi) { q += 1.0; r = fma(-q, kTwoPi, x); }
  } else {
    if (r > 0.0) { q += 1.0; r = fma(-q, kTwoPi, x); }
    else if (r <= -kTwoPi) { q -= 1.0; r = fma(-q, kTwoPi, x); }
  }
  return r;
}

// numpy remainder (Python floor-mod) by 2*pi: npy_divmod semantics.
__device__ __forceinline__ double pymod_2pi(double x) {
  double r = fmod_2pi(x);
  if (r != 0.0) {
    if (r < 0.0) r += kTwoPi;
  } else {
    r = 0.0;
  }
  return r;
}

// ======================================================================
// Record (register-resident copy of one satellite's packed record)
// ======================================================================
template <typename T>
struct Rec {
  T v[S_COUNT];
  __device__ __forceinline__ T operator[](int i) const { return v[i]; }
  __device__ __forceinline__ int flags() const;
};

// a record held in shared memory (one per warp): fields are re-read at use,
// which lets the register allocator drop them instead of spilling
template <typename T>
struct RecS {
  const T* p;
  __device__ __forceinline__ T operator[](int i) const { return p[i]; }
  __device__ __forceinline__ int flags() const;
};
template <>
__device__ __forceinline__ int RecS<float>::flags() const { return __float_as_int(p[S_FLAGS]); }

// a fp32 record spread over the warp: lane l holds fields l and 32 + l;
// a field is broadcast with one shfl at use (2 registers per thread instead
// of 40).  Requires the whole warp converged at every access.
struct RecW {
  float lo, hi;
  __device__ __forceinline__ float operator[](int i) const {
    return __shfl_sync(0xffffffffu, i < 32 ? lo : hi, i & 31);
  }
  __device__ __forceinline__ int flags() const { return __float_as_int((*this)[S_FLAGS]); }
};
template <>
__device__ __forceinline__ int RecS<double>::flags() const {
  return (int)__double_as_longlong(p[Q_FLAGS]);
}
template <>
__device__ __forceinline__ int Rec<float>::flags() const { return __float_as_int(v[S_FLAGS]); }
template <>
__device__ __forceinline__ int Rec<double>::flags() const {
  return (int)__double_as_longlong(v[Q_FLAGS]);
}

__device__ __forceinline__ void load_rec(const float* __restrict__ p, Rec<float>& r) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int i = 0; i < S_COUNT / 4; ++i) {
    float4 x = __ldg(q + i);
    r.v[4 * i + 0] = x.x; r.v[4 * i + 1] = x.y; r.v[4 * i + 2] = x.z; r.v[4 * i + 3] = x.w;
  }
}
__device__ __forceinline__ void load_rec(const double* __restrict__ p, Rec<double>& r) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < S_COUNT / 2; ++i) {
    double2 x = __ldg(q + i);
    r.v[2 * i + 0] = x.x; r.v[2 * i + 1] = x.y;
  }
}


// ======================================================================
// Kepler (kernel.py:325-349)
// ======================================================================
template <typename T>
__device__ __forceinline__ T kepler_reference(T axnl, T aynl, T u) {
  const T clamp = T(0.95);
  T eo1 = u;
  bool active = true;
#pragma unroll 1
  for (int it = 0; it < 10 && active; ++it) {
    T s, c;
    sincos(eo1, &s, &c);
    T den = T(1) - c * axnl - s * aynl;
    T tem5 = (u - aynl * c + axnl * s - eo1) / den;
    tem5 = tem5 >= clamp ? clamp : (tem5 <= -clamp ? -clamp : tem5);
    eo1 = eo1 + tem5;
    active = fabs(tem5) >= T(1.0e-12);
  }
  return eo1;
}
template <>
__device__ __forceinline__ float kepler_reference<float>(float axnl, float aynl, float u) {
  const float clamp = 0.95f;
  float eo1 = u;
  bool active = true;
#pragma unroll 1
  for (int it = 0; it < 10 && active; ++it) {
    float s, c;
    sincosf(eo1, &s, &c);
    float den = 1.0f - c * axnl - s * aynl;
    float tem5 = (u - aynl * c + axnl * s - eo1) / den;
    tem5 = tem5 >= clamp ? clamp : (tem5 <= -clamp ? -clamp : tem5);
    eo1 = eo1 + tem5;
    active = fabsf(tem5) >= 1.0e-12f;
  }
  return eo1;
}

// streaming (evict-first) scalar stores
__device__ __forceinline__ void st_cs(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(int32_t* p, int32_t v) { __stcs(reinterpret_cast<int*>(p), (int)v); }

// ======================================================================
// fp64 cells (kernel.py:352-510)
// ======================================================================
struct Cell64 {
  double r[3], v[3];
  int code;
};

// 1/x by one third-order step r (1 + e + e^2), e = 1 - x r, from the SFU
// seed (|e| ~ 2^-22, so the result error e^3 is below fp64 rounding)
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);              // r (1 + e + e^2)
}
// sqrt(x) and 1/sqrt(x) for x > 0: SFU rsqrt seed + Newton, then a
// Tuckerman-style correction of x * (1/sqrt x)
__device__ __forceinline__ double rsqrt64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);                // ~2^-22 -> 2^-43 -> fp64
  return y * fma(-hx * y, y, 1.5);
}
__device__ __forceinline__ double sqrt64(double x) {
  const double y = rsqrt64(x);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

// |x| < 2^-k as an integer test of the high word (ALU pipe, not FP64)
__device__ __forceinline__ bool small_abs(double x, unsigned hi_bound) {
  return ((unsigned)__double2hiint(x) & 0x7fffffffu) < hi_bound;
}
constexpr unsigned kHi2m6 = 0x3F900000u;     // 2^-6
constexpr unsigned kHi2m8 = 0x3F700000u;     // 2^-8
constexpr unsigned kHi2m10 = 0x3F500000u;    // 2^-10

// sin/cos providers.  TrigTab is the propagate kernels' evaluation: a
// 512-entry (sin, cos)(2 pi i / 512) table in shared memory and a short
// polynomial on the remainder |r| <= pi/512 (sin to r^5, truncation r^7/5040
// < 1e-19; cos to r^4, truncation r^6/720 < 1e-16), 14 fp64 operations and
// one 16-byte shared load.  The reduction is two-part Cody-Waite (C1 has 27
// significant bits, so k C1 is exact for |k| < 2^26, |x| < 8e5 rad), and the
// quotient k comes from the 1.5 2^52 shifter, whose low word is the table
// index.  TrigLib (libdevice) serves the init kernel.
#ifndef SGP4B_TABN
#define SGP4B_TABN 1024
#endif
constexpr int kTabN = SGP4B_TABN;
constexpr double kTabScale = kTabN / 6.283185307179586476925286766559;   // N / (2 pi)
// 2 pi / N rounded to 27 significant bits (k C1 exact for |k| < 2^26), and
// the remainder
constexpr double kTabStep = 6.283185307179586476925286766559 / kTabN;
constexpr double kTabC1Scale = kTabN <= 512 ? 17179869184.0 * 2.0 : 17179869184.0 * (kTabN / 1024);
constexpr double kTabC1 = (double)(long long)(kTabStep * kTabC1Scale) / kTabC1Scale;
// (2 pi = fl(2 pi) + 2.4492935982947064e-16: the low word keeps k C2 exact
// to ~1e-21 for the |k| < 2^26 the reduction admits)
constexpr double kTabC2 = (6.283185307179586476925286766559 - kTabC1 * kTabN) / kTabN +
                          2.4492935982947064e-16 / kTabN;
// with |r| <= pi / N the sine needs r^5/120 only for N < 1024 (at N = 1024
// it is below 2.3e-15, so every evaluation takes the short form)
constexpr bool kTabShortSin = kTabN >= 1024;
constexpr double kShift52 = 6755399441055744.0;         // 1.5 * 2^52
// fp64 constants whose low words are nonzero live in constant memory, so
// DFMA reads them as c[][] operands instead of rematerialising 64-bit
// immediates into register pairs every cell
__constant__ double c_k64[8] = {kTabScale, kTabC1, kTabC2, 1.0 / 120.0, -1.0 / 6.0, 1.0 / 24.0,
                                kInvTwoPi, kTwoPi};
#define K_TABSCALE c_k64[0]
#define K_TABC1 c_k64[1]
#define K_TABC2 c_k64[2]
#define K_1_120 c_k64[3]
#define K_M1_6 c_k64[4]
#define K_1_24 c_k64[5]
#define K_INV2PI c_k64[6]
#define K_2PI c_k64[7]

struct TrigTab {
  const double2* tab;
  __device__ __forceinline__ void operator()(double x, double& s, double& c) const {
    const double y = fma(x, K_TABSCALE, kShift52);
    const double k = y - kShift52;
    const int idx = __double2loint(y) & (kTabN - 1);
    double r = fma(-k, K_TABC1, x);
    r = fma(-k, K_TABC2, r);
    const double z = r * r;
    const double sr = kTabShortSin ? fma(r * z, K_M1_6, r) : fma(r * z, fma(z, K_1_120, K_M1_6), r);
    const double cr = fma(z, fma(z, K_1_24, -0.5), 1.0);
    const double2 e = tab[idx];                          // (sin a, cos a)
    s = fma(e.x, cr, e.y * sr);
    c = fma(e.y, cr, -e.x * sr);
  }
  // the same with the sine series one term shorter (r^5/120 < 8e-14): for
  // angles that reach the state scaled down (argpm by em, xmdf by drag)
  __device__ __forceinline__ void short_sin(double x, double& s, double& c) const {
    const double y = fma(x, K_TABSCALE, kShift52);
    const double k = y - kShift52;
    const int idx = __double2loint(y) & (kTabN - 1);
    double r = fma(-k, K_TABC1, x);
    r = fma(-k, K_TABC2, r);
    const double z = r * r;
    const double sr = fma(r * z, K_M1_6, r);
    const double cr = fma(z, fma(z, K_1_24, -0.5), 1.0);
    const double2 e = tab[idx];
    s = fma(e.x, cr, e.y * sr);
    c = fma(e.y, cr, -e.x * sr);
  }
};
// table-free alternative (SGP4B_F64_TABLE=0): quadrant reduction and
// degree-13/14 polynomials, coefficients in constant memory
__constant__ double c_sin_poly[6] = {
    -1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
    2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10};
__constant__ double c_cos_poly[6] = {
    4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
    -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11};
__constant__ double c_pio2[4] = {1.57079632673412561417e+00, 6.07710050630396597660e-11,
                                 2.02226624879595063154e-21, 6.36619772367581382433e-01};
struct TrigPoly {
  const double2* tab;                                    // unused
  __device__ __forceinline__ void operator()(double x, double& s, double& c) const {
    const double y = fma(x, c_pio2[3], kShift52);
    const double k = y - kShift52;
    const int q = __double2loint(y) & 3;
    double r = fma(-k, c_pio2[0], x);
    r = fma(-k, c_pio2[1], r);
    r = fma(-k, c_pio2[2], r);
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, c_sin_poly[5], c_sin_poly[4]),
                                                   c_sin_poly[3]), c_sin_poly[2]), c_sin_poly[1]),
                          c_sin_poly[0]);
    const double sr = fma(r * z, ps, r);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, c_cos_poly[5], c_cos_poly[4]),
                                                   c_cos_poly[3]), c_cos_poly[2]), c_cos_poly[1]),
                          c_cos_poly[0]);
    const double cr = fma(z * z, pc, fma(-0.5, z, 1.0));
    const double s0 = (q & 1) ? cr : sr;
    const double c0 = (q & 1) ? sr : cr;
    s = (q & 2) ? -s0 : s0;
    c = ((q + 1) & 2) ? -c0 : c0;
  }
  __device__ __forceinline__ void short_sin(double x, double& s, double& c) const { (*this)(x, s, c); }
};
#ifndef SGP4B_F64_TABLE
#define SGP4B_F64_TABLE 1
#endif
struct TrigLib {
  __device__ __forceinline__ void operator()(double x, double& s, double& c) const { sincos(x, &s, &c); }
  __device__ __forceinline__ void short_sin(double x, double& s, double& c) const { sincos(x, &s, &c); }
};

// (sin, cos)(a + d) from (sin, cos)(a): series to d^5 / d^4 for |d| < 2^-8
// (truncation d^7/5040 < 1e-20, d^6/720 < 5e-18), otherwise a direct
// evaluation of the new angle x.
template <class Trig>
__device__ __forceinline__ void rotate64(double s, double c, double d, double x, const Trig& tr,
                                         double& so, double& co) {
  if (small_abs(d, kHi2m8)) {
    const double d2 = d * d;
    const double sd = fma(d * d2, fma(d2, K_1_120, K_M1_6), d);
    const double cd = fma(d2, fma(d2, K_1_24, -0.5), 1.0);
    so = fma(s, cd, c * sd);
    co = fma(c, cd, -s * sd);
  } else {
    tr(x, so, co);
  }
}

// orientation and output (kernel.py:472-493) from (sin, cos) su, xnode, xinc
__device__ __forceinline__ void orient64(double mr, double mv, double rv, double sinsu,
                                         double cossu, double snod, double cnod, double sini,
                                         double cosi, Cell64& o) {
  const double xmx = -snod * cosi;
  const double xmy = cnod * cosi;
  const double ra = mr * sinsu, rb = mr * cossu;
  o.r[0] = fma(xmx, ra, cnod * rb);
  o.r[1] = fma(xmy, ra, snod * rb);
  o.r[2] = sini * ra;
  const double va = fma(mv, sinsu, rv * cossu);
  const double vb = fma(mv, cossu, -rv * sinsu);
  o.v[0] = fma(xmx, va, cnod * vb);
  o.v[1] = fma(xmy, va, snod * vb);
  o.v[2] = sini * va;
}

// General fp64 cell: every orbit class, the reference's guards, thresholds
// and code precedence, and the reference's Kepler loop (<= 10 Newton steps,
// +-0.95 clamp, 1e-12 freeze).  It departs from the reference operation
// order only where results move far below the 1 mm / 1e-6 km/s budget
// (measured ~1e-9 km): per-satellite products folded into the record (fp64),
// no floor-mods (every angle only reaches sin/cos, whose reduction is exact),
// the Kepler argument formed as u = (mo + argpo) + (mdot + argpdot) t +
// no templ + xlcof axnl / pl_lp (mm + argpm: the drag terms cancel) with E
// carried as u + d, sin/cos carried through the small drag, Newton and J2
// corrections by rotation (rotate64), and the atan2 of kernel.py:455
// replaced by normalising (sin u, cos u).
template <class RT, class Trig>
__device__ __forceinline__ void cell64_general(const RT& R, double t, double re, double vkm,
                                               const Trig& tr, Cell64& o) {
  const double tiny = DBL_MIN;
  const int flags = R.flags();
  const bool isimp = flags & FLAG_ISIMP;

  // secular gravity and atmospheric drag  kernel.py:365-391
  const double argpdf = fma(R[Q_ARGPDOT], t, R[Q_ARGPO]);
  const double t2 = t * t;
  const double nodem = fma(R[Q_NODECF], t2, fma(R[Q_NODEDOT], t, R[Q_NODEO]));
  const double usec = fma(R[Q_UDOT], t, R[Q_U0]);
  double sqam, nol, argpm, em;
  if (isimp) {
    sqam = fma(R[Q_SC1], t, R[Q_S]);
    nol = R[Q_N2] * t2;
    em = fma(-R[Q_BC4], t, R[Q_E0]);
    argpm = argpdf;
  } else {
    const double xmdf = fma(R[Q_MDOT], t, R[Q_MO]);
    double sx, cx;
    tr(xmdf, sx, cx);
    const double temp = fma(fma(fma(cx, R[Q_A3], R[Q_A2]), cx, R[Q_A1]), cx,
                            fma(R[Q_OMGCOF], t, R[Q_A0]));
    argpm = argpdf - temp;
    sqam = fma(t, fma(t, fma(t, fma(t, R[Q_SD4], R[Q_SD3]), R[Q_SD2]), R[Q_SC1]), R[Q_S]);
    nol = t2 * fma(t, fma(t, fma(t, R[Q_N5], R[Q_N4]), R[Q_N3]), R[Q_N2]);
    double smm, cmm;
    rotate64(sx, cx, temp, xmdf + temp, tr, smm, cmm);    // sin(mm)
    em = fma(-R[Q_BC5], smm, fma(-R[Q_BC4], t, R[Q_E0]));
  }

  // mean motion / eccentricity update  kernel.py:393-414
  const double asq = fabs(sqam);                            // sqrt(am)
  const double am = gmax(sqam * sqam, tiny);                // am_safe
  const double irs = rcp64(asq);
  const double nmx = irs * irs * irs;                       // nm / xke = am^-1.5
  const bool bad_em = (em >= 1.0) || (em < -0.001);
  em = em < 1.0e-6 ? 1.0e-6 : em;

  // long-period periodics  kernel.py:419-431
  double sa, ca;
  tr(argpm, sa, ca);
  const double axnl = em * ca;
  const double ilp = rcp64(gmax(am * fma(-em, em, 1.0), tiny));
  const double aynl = fma(em, sa, ilp * R[Q_AYCOF]);
  const double u = fma(ilp * R[Q_XLCOF], axnl, usec + nol);

  // Kepler  kernel.py:325-349: E = u + d, (sin, cos) E carried along the
  // Newton updates by rotation, the reference's clamp and 1e-12 freeze
  double sineo1, coseo1, d = 0.0;
  tr(u, sineo1, coseo1);
  bool active = true;
#pragma unroll 1
  for (int it = 0; it < 10 && active; ++it) {
    const double den = fma(-sineo1, aynl, fma(-coseo1, axnl, 1.0));
    const double num = fma(axnl, sineo1, fma(-aynl, coseo1, -d));
    double tem5 = num * rcp64(den);
    tem5 = tem5 >= 0.95 ? 0.95 : (tem5 <= -0.95 ? -0.95 : tem5);
    d += tem5;
    rotate64(sineo1, coseo1, tem5, u + d, tr, sineo1, coseo1);
    active = fabs(tem5) >= 1.0e-12;
  }

  // short-period preliminaries  kernel.py:440-460
  const double ecose = fma(axnl, coseo1, aynl * sineo1);
  const double esine = fma(axnl, sineo1, -aynl * coseo1);
  const double el2 = fma(axnl, axnl, aynl * aynl);
  const double omel2 = 1.0 - el2;
  const double pl = am * omel2;
  const bool bad_pl = pl < 0.0;
  const double pl_safe = gmax(pl, tiny);
  const double rl = am * (1.0 - ecose);
  const double irl = rcp64(rl == 0.0 ? tiny : rl);
  const double betal = sqrt64(gmax(omel2, tiny));
  const double rdv = (asq * vkm) * esine * irl;
  // sqrt(pl_safe) = sqrt(am) betal whenever pl >= tiny
  const double rvdv = (pl >= tiny ? asq * betal : sqrt64(pl_safe)) * (irl * vkm);
  const double tq = esine * rcp64(1.0 + betal);
  // (sin u, cos u) normalised: the reference's am/rl factor is positive and
  // only the direction reaches su
  const double sn = fma(-axnl, tq, sineo1 - aynl);
  const double cs = fma(aynl, tq, coseo1 - axnl);
  const double inrm = rsqrt64(fma(sn, sn, cs * cs));
  const double sinu = sn * inrm, cosu = cs * inrm;
  const double s2u = sinu + sinu;
  const double sin2u = s2u * cosu;
  const double cos2u = fma(-s2u, sinu, 1.0);
  const double ipl = rcp64(pl_safe);
  const double ipl2 = ipl * ipl;

  // short-period periodics  kernel.py:463-469 (0.5 j2, re, vkm folded)
  const double mrt = fma(rl, fma(ipl2 * R[Q_K41R], betal, re), (ipl * R[Q_KXR]) * cos2u);
  const double t2s = ipl2 * sin2u;
  const double dsu = t2s * R[Q_QX];
  const double xnode = fma(t2s, R[Q_C15CO], nodem);
  const double dinc = (ipl2 * cos2u) * R[Q_C15CS];
  const double nmt = nmx * ipl;
  const double mv = fma(-(nmt * R[Q_X1V]), sin2u, rdv);
  const double rv = fma(nmt, fma(cos2u, R[Q_X1V], R[Q_C41V]), rvdv);

  // orientation  kernel.py:472-493
  double sinsu, cossu, snod, cnod, sini, cosi;
  if (small_abs(dsu, kHi2m8))
    rotate64(sinu, cosu, dsu, 0.0, tr, sinsu, cossu);
  else
    tr(atan2(sinu, cosu) + dsu, sinsu, cossu);
  tr(xnode, snod, cnod);
  rotate64(R[Q_SINIO], R[Q_COSIO], dinc, R[Q_INCLO] + dinc, tr, sini, cosi);
  orient64(mrt, mv, rv, sinsu, cossu, snod, cnod, sini, cosi, o);

  // _first_error + init merge  kernel.py:495-502, 529-534 (bad_nm is folded
  // into the persistent code field of the record); decayed: mrt < 1 earth
  // radius, i.e. mr < re
  const int code = bad_em ? 1 : bad_pl ? 4 : (mrt < re) ? 6 : 0;
  const int persistent = (flags >> CODE_SHIFT) & 0x7fffff;
  o.code = persistent != 0 ? persistent : code;
}

// the general cell as one out-of-line copy, storing its own outputs: the
// fallback of the fast cell (nothing of the fast path's state escapes to
// local memory)
using TrigGrid = std::conditional<SGP4B_F64_TABLE != 0, TrigTab, TrigPoly>::type;

__device__ __noinline__ void cell64_fallback(const double* rec, double t, double re, double vkm,
                                             const double2* tab, double* out, int64_t ps,
                                             int32_t* cout) {
  RecS<double> R;
  R.p = rec;
  Cell64 o;
  cell64_general(R, t, re, vkm, TrigGrid{tab}, o);
  st_cs(out, o.r[0]);
  st_cs(out + ps, o.r[1]);
  st_cs(out + 2 * ps, o.r[2]);
  st_cs(out + 3 * ps, o.v[0]);
  st_cs(out + 4 * ps, o.v[1]);
  st_cs(out + 5 * ps, o.v[2]);
  st_cs(cout, o.code);
}

// 64-bit integer views of doubles: ordering tests on the ALU pipe (the FP64
// pipe is the binding resource of the fp64 cell).  Valid for finite x.
__device__ __forceinline__ long long dbits(double x) { return __double_as_longlong(x); }
// x < b for a constant b > 0: negative doubles are negative int64s
__device__ __forceinline__ bool lt_pos(double x, long long bbits) { return dbits(x) < bbits; }
// x < b for a constant b < 0: among doubles with the sign bit set, the
// unsigned bit pattern grows with the magnitude; positives are below them all
__device__ __forceinline__ bool lt_neg(double x, unsigned long long bbits) {
  return (unsigned long long)dbits(x) > bbits;
}
constexpr long long kBits1em6 = 0x3EB0C6F7A0B5ED8DLL;          // 1.0e-6
constexpr unsigned long long kBitsM1em3 = 0xBF50624DD2F1A9FCULL; // -0.001
constexpr unsigned kHi4em3 = 0x3F70624Du;                        // hi word of 0.004
constexpr unsigned kHiE2 = 0x3FB97F62u;                          // hi word of ~0.0996
// el2 = axnl^2 + aynl^2 <= (em + |aycof| / pl_lp)^2: below these for every
// class-1 / class-2 cell of a normal orbit; a collapsed semi-major axis
// (1/pl_lp large) exceeds them and takes the general cell
constexpr unsigned kHiEl2K1 = 0x3EFF7510u;                       // hi word of 3e-5
constexpr unsigned kHiEl2K2 = 0x3F88C7E2u;                       // hi word of 0.0121
constexpr unsigned kHiTiny = 0x20C00000u;                        // ~6e-151

// Fast fp64 cell for near-circular orbits (|em| < 0.004 at this cell, every
// Starlink-like satellite): with el = |(axnl, aynl)| < 0.0052, el2 < 3e-5,
//   * two Newton steps reach the fixed point of the reference's loop (error
//     el^7/8 < 1e-17; the first step's 1/den as 1 + q + q^2, the second's as
//     1 + q + q^2 + q^3, |q| < el: the second step absorbs the first
//     truncation and leaves q^4 of a 1e-7 step; its rotation has cos = 1 to
//     2.5e-15);
//   * betal = 1 - el2/2 - el2^2/8, 1/pl = (1 + el2 + el2^2)/am,
//     1/pl_lp = (1 + em^2 + em^4)/am, 1/(1 + betal) = 1/2 + el2/8 + el2^2/16
//     (truncations < 3e-14 relative, on terms of order 1e-3), pl > 0 so the
//     SEMILATUS code cannot occur;
//   * (sin u, cos u) = (am/rl) (...) as the reference forms them (unit norm
//     at the converged E);
//   * sin(mm) = sin(xmdf + temp) to temp^3 (|temp| < 2^-6; it only enters
//     through bstar cc5 < 4e-6), the J2 rotations of su and xinc as series
//     (|dsu|, |dinc| < 2^-10; near-Earth orbits have |dsu| < 8.1e-4 and
//     |dinc| < 4.1e-4), and the first Newton rotation to d^3 and d^4;
//   * sin/cos of argpm (scaled by em < 0.004) and of xmdf (through the drag
//     coefficients) with the sine series one term shorter (r^5/120 < 8e-14).
// The cell is straight-line code; a cell outside that domain (|em| >= 0.004,
// a NaN, sqrt(am) < 6e-151, or a larger drag / J2 angle) reports false and
// the caller runs the general cell instead.  The test is per cell, so a
// cell's value never depends on which other cells share its launch
// (batch == scalar).
// K2 = true: the same cell for Kepler class 2 (|em| < 0.0996 at this cell,
// most of a general LEO catalogue): three Newton steps (error (e/2)^7 e^8
// < 1e-17), the first rotation by a full table evaluation, exact
// reciprocals / square roots where class 1 uses series (1/pl_lp, betal,
// 1/pl, 1/(1 + betal), 1/den).  The J2, drag and orientation stages and the
// domain fallback are class 1's.
template <bool ISIMP, class RT, class Trig, bool K2 = false>
__device__ __forceinline__ bool cell64_c1(const RT& R, double t, double re, long long re_bits,
                                          double vkm, const Trig& tr, Cell64& o) {
  const int flags = R.flags();
  const double argpdf = fma(R[Q_ARGPDOT], t, R[Q_ARGPO]);
  const double t2 = t * t;
  const double nodem = fma(R[Q_NODECF], t2, fma(R[Q_NODEDOT], t, R[Q_NODEO]));
  const double usec = fma(R[Q_UDOT], t, R[Q_U0]);
  double sqam, nol, argpm, em;
  bool ok = true;
  if constexpr (ISIMP) {
    sqam = fma(R[Q_SC1], t, R[Q_S]);
    nol = R[Q_N2] * t2;
    em = fma(-R[Q_BC4], t, R[Q_E0]);
    argpm = argpdf;
  } else {
#if !SGP4B_F64_DRAG32
    const double xmdf = fma(R[Q_MDOT], t, R[Q_MO]);
    double sx, cx;
    tr.short_sin(xmdf, sx, cx);
    const double temp = fma(fma(fma(cx, R[Q_A3], R[Q_A2]), cx, R[Q_A1]), cx,
                            fma(R[Q_OMGCOF], t, R[Q_A0]));
    argpm = argpdf - temp;
    sqam = fma(t, fma(t, fma(t, fma(t, R[Q_SD4], R[Q_SD3]), R[Q_SD2]), R[Q_SC1]), R[Q_S]);
    nol = t2 * fma(t, fma(t, fma(t, R[Q_N5], R[Q_N4]), R[Q_N3]), R[Q_N2]);
    const double tt = temp * temp;
    const double smm = fma(sx, fma(tt, -0.5, 1.0), (cx * temp) * fma(tt, K_M1_6, 1.0));
    em = fma(-R[Q_BC5], smm, fma(-R[Q_BC4], t, R[Q_E0]));
#else
    // drag, off the FP64 pipe: xmdf only reaches the state through the drag
    // cubic (coefficients A1..A3, times em when it moves argpm) and through
    // bstar cc5 sin(mm) (< 4e-6), so after an fp64 reduction to [-pi, pi]
    // its sin/cos come from the SFU and the cubic and sin(mm) are fp32: the
    // position error this adds is below 1e-8 km (2 coef bstar 4e-7 a), and
    // the conversions ride the idle XU
    const double xmdf = fma(R[Q_MDOT], t, R[Q_MO]);
    const double kx = fma(xmdf, K_INV2PI, kShift52) - kShift52;
    float sx, cx;
    __sincosf((float)fma(-kx, K_2PI, xmdf), &sx, &cx);
    const float cub = cx * fmaf(fmaf(cx, (float)R[Q_A3], (float)R[Q_A2]), cx, (float)R[Q_A1]);
    const double temp = fma(R[Q_OMGCOF], t, R[Q_A0]) + (double)cub;
    argpm = argpdf - temp;
    sqam = fma(t, fma(t, fma(t, fma(t, R[Q_SD4], R[Q_SD3]), R[Q_SD2]), R[Q_SC1]), R[Q_S]);
    nol = t2 * fma(t, fma(t, fma(t, R[Q_N5], R[Q_N4]), R[Q_N3]), R[Q_N2]);
    const float tf = (float)temp;
    const float tt = tf * tf;
    const float smm = fmaf(sx, fmaf(tt, -0.5f, 1.0f), (cx * tf) * fmaf(tt, -1.0f / 6.0f, 1.0f));
    em = fma(-R[Q_BC4], t, R[Q_E0]) - (double)((float)R[Q_BC5] * smm);
#endif
    ok = small_abs(temp, kHi2m6);
  }
  const double asq = __longlong_as_double(dbits(sqam) & 0x7fffffffffffffffLL);   // |sqam|
  ok = ok && small_abs(em, K2 ? kHiE2 : kHi4em3) &&
       ((unsigned)__double2hiint(asq) & 0x7fffffffu) >= kHiTiny;
  const bool bad_em = lt_neg(em, kBitsM1em3);
  em = lt_pos(em, kBits1em6) ? 1.0e-6 : em;

  // mean motion  kernel.py:397-401 (nm / xke = am^-1.5)
  const double am = sqam * sqam;
  const double irs = rcp64(asq);
  const double inv_am = irs * irs;
  const double nmx = inv_am * irs;

  // long-period periodics  kernel.py:419-431
  double sa, ca;
  tr.short_sin(argpm, sa, ca);
  const double axnl = em * ca;
  const double em2 = em * em;
  const double ilp = K2 ? inv_am * rcp64(1.0 - em2)                  // 1 / (am (1 - em^2))
                        : fma(inv_am, fma(em2, em2, em2), inv_am);
  const double aynl = fma(em, sa, ilp * R[Q_AYCOF]);
  const double u = fma(ilp * R[Q_XLCOF], axnl, usec + nol);

  // Kepler  kernel.py:325-349, from E0 = u: class 1 two Newton steps,
  // class 2 three (the reference's freeze at |step| < 1e-12 is reached)
  double s0, c0;
  tr(u, s0, c0);
  double q = fma(c0, axnl, s0 * aynl);
  double num = fma(axnl, s0, -aynl * c0);
  double sineo1, coseo1;
  if constexpr (K2) {
    const double d1 = num * rcp64(1.0 - q);             // |d1| <= ~0.11
    double s1, c1;
    tr(u + d1, s1, c1);
    q = fma(c1, axnl, s1 * aynl);
    num = fma(axnl, s1, fma(-aynl, c1, -d1));
    const double d2 = num * rcp64(1.0 - q);             // |d2| < 1e-3
    const double dd = d2 * d2;
    const double sd = fma(d2 * dd, K_M1_6, d2);          // d^5/120 < 1e-17
    const double cd = fma(dd, fma(dd, K_1_24, -0.5), 1.0);
    const double s2 = fma(s1, cd, c1 * sd), c2 = fma(c1, cd, -s1 * sd);
    q = fma(c2, axnl, s2 * aynl);
    num = fma(axnl, s2, fma(-aynl, c2, -(d1 + d2)));
    const double d3 = num * rcp64(1.0 - q);             // |d3| < 1e-8: cos d3 = 1
    sineo1 = fma(c2, d3, s2);
    coseo1 = fma(-s2, d3, c2);
  } else {
    const double d1 = fma(num, fma(q, q, q), num);
    const double dd = d1 * d1;
    const double sd = fma(d1 * dd, K_M1_6, d1);         // d^5/120 < 4e-14
    const double cd = fma(dd, fma(dd, K_1_24, -0.5), 1.0);
    const double s1 = fma(s0, cd, c0 * sd), c1 = fma(c0, cd, -s0 * sd);
    q = fma(c1, axnl, s1 * aynl);
    num = fma(axnl, s1, fma(-aynl, c1, -d1));
    const double d2 = fma(num, q, num) * fma(q, q, 1.0);
    sineo1 = fma(c1, d2, s1);
    coseo1 = fma(-s1, d2, c1);
  }

  // short-period preliminaries  kernel.py:440-460
  const double ecose = fma(axnl, coseo1, aynl * sineo1);
  const double esine = fma(axnl, sineo1, -aynl * coseo1);
  const double el2 = fma(axnl, axnl, aynl * aynl);
  ok = ok && small_abs(el2, K2 ? kHiEl2K2 : kHiEl2K1);
  const double ome = 1.0 - ecose;
  const double iome = rcp64(ome);                                 // am / rl
  const double rl = am * ome;
  double betal, ipl, tq;
  if constexpr (K2) {
    // el2 < 0.0121: pl = am (1 - el2) > 0 (no SEMILATUS code)
    const double omel2 = 1.0 - el2;
    const double rb = rsqrt64(omel2);
    betal = omel2 * rb;                                           // sqrt(1 - el2)
    ipl = inv_am * (rb * rb);                                     // 1 / pl
    tq = esine * rcp64(1.0 + betal);
  } else {
    betal = fma(el2, fma(el2, -0.125, -0.5), 1.0);
    ipl = fma(inv_am, fma(el2, el2, el2), inv_am);
    tq = esine * fma(el2, fma(el2, 0.0625, 0.125), 0.5);
  }
  const double sqvk = (irs * vkm) * iome;                         // sqrt(am)/rl km/s
  const double rdv = sqvk * esine;
  const double rvdv = sqvk * betal;
  const double sinu = fma(-axnl, tq, sineo1 - aynl) * iome;
  const double cosu = fma(aynl, tq, coseo1 - axnl) * iome;
  const double s2u = sinu + sinu;
  const double sin2u = s2u * cosu;
  const double cos2u = fma(-s2u, sinu, 1.0);
  const double ipl2 = ipl * ipl;

  // short-period periodics  kernel.py:463-469
  const double mr = fma(rl, fma(ipl2 * R[Q_K41R], betal, re), (ipl * R[Q_KXR]) * cos2u);
  const double t2s = ipl2 * sin2u;
  const double dsu = t2s * R[Q_QX];
  const double xnode = fma(t2s, R[Q_C15CO], nodem);
  const double dinc = (ipl2 * cos2u) * R[Q_C15CS];
  const double nmt = nmx * ipl;
  const double mv = fma(-(nmt * R[Q_X1V]), sin2u, rdv);
  const double rv = fma(nmt, fma(cos2u, R[Q_X1V], R[Q_C41V]), rvdv);
  ok = ok && small_abs(dsu, kHi2m10) && small_abs(dinc, kHi2m10);

  // orientation  kernel.py:472-493: su = u + dsu, xinc = inclo + dinc by
  // rotation, |d| < 2^-10: sin d = d - d^3/6, cos d = 1 - d^2/2 (truncation
  // < 4e-14)
  const double du2 = dsu * dsu;
  const double sdu = fma(dsu * du2, K_M1_6, dsu);
  const double cdu = fma(du2, -0.5, 1.0);
  const double sinsu = fma(sinu, cdu, cosu * sdu), cossu = fma(cosu, cdu, -sinu * sdu);
  double snod, cnod;
  tr(xnode, snod, cnod);
  const double di2 = dinc * dinc;
  const double sdi = fma(dinc * di2, K_M1_6, dinc);
  const double cdi = fma(di2, -0.5, 1.0);
  const double sini = fma(R[Q_SINIO], cdi, R[Q_COSIO] * sdi);
  const double cosi = fma(R[Q_COSIO], cdi, -R[Q_SINIO] * sdi);
  orient64(mr, mv, rv, sinsu, cossu, snod, cnod, sini, cosi, o);

  const int code = bad_em ? 1 : lt_pos(mr, re_bits) ? 6 : 0;
  const int persistent = (flags >> CODE_SHIFT) & 0x7fffff;
  o.code = persistent != 0 ? persistent : code;
  return ok;
}

// ======================================================================
// fp32 cells: the throughput path, two cells per instruction
// ======================================================================
// Blackwell executes packed dual-fp32 FMUL2/FADD2/FFMA2 (one issue slot, two
// IEEE results, scalar-broadcast operands allowed).  A lane's consecutive
// time steps run the identical instruction stream, so cells are evaluated in
// pairs on V2 = float2; the SFU ops (sin/cos/rcp/rsqrt), compares and
// selects stay per component.  Every mul/add/fma below is an explicit
// IEEE-rounded op (no contraction decisions left to the compiler), so a
// cell's value does not depend on which half of a pair it ran in: the
// scalar API (pairs kernel) evaluates the same V2 code with both halves
// equal and matches the grid bit for bit.

// N cells (N even) as N/2 packed float2 halves; every op applies to all
// halves in program order, so two cell-pairs advance in lockstep and the
// scheduler always has an independent packed op in flight.
template <int N>
struct VN {
  float2 h[N / 2];
};
template <int N>
__device__ __forceinline__ VN<N> sp(float s) {
  VN<N> r;
#pragma unroll
  for (int i = 0; i < N / 2; ++i) r.h[i] = make_float2(s, s);
  return r;
}
#define VN_MAP1(expr)                      \
  VN<N> r;                                 \
  _Pragma("unroll") for (int i = 0; i < N / 2; ++i) r.h[i] = (expr); \
  return r;
template <int N>
__device__ __forceinline__ VN<N> operator+(VN<N> a, VN<N> b) { VN_MAP1(__fadd2_rn(a.h[i], b.h[i])) }
template <int N>
__device__ __forceinline__ VN<N> operator-(VN<N> a) { VN_MAP1(make_float2(-a.h[i].x, -a.h[i].y)) }
template <int N>
__device__ __forceinline__ VN<N> operator-(VN<N> a, VN<N> b) {
  VN_MAP1(__fadd2_rn(a.h[i], make_float2(-b.h[i].x, -b.h[i].y)))
}
template <int N>
__device__ __forceinline__ VN<N> operator*(VN<N> a, VN<N> b) { VN_MAP1(__fmul2_rn(a.h[i], b.h[i])) }
template <int N>
__device__ __forceinline__ VN<N> fma2(VN<N> a, VN<N> b, VN<N> c) {
  VN_MAP1(__ffma2_rn(a.h[i], b.h[i], c.h[i]))
}
template <int N>
__device__ __forceinline__ VN<N> operator+(VN<N> a, float b) { return a + sp<N>(b); }
template <int N>
__device__ __forceinline__ VN<N> operator-(float a, VN<N> b) { return sp<N>(a) - b; }
template <int N>
__device__ __forceinline__ VN<N> operator-(VN<N> a, float b) { return a - sp<N>(b); }
template <int N>
__device__ __forceinline__ VN<N> operator*(VN<N> a, float b) { return a * sp<N>(b); }
template <int N>
__device__ __forceinline__ VN<N> fma2(VN<N> a, VN<N> b, float c) { return fma2(a, b, sp<N>(c)); }
template <int N>
__device__ __forceinline__ VN<N> fma2(VN<N> a, float b, VN<N> c) { return fma2(a, sp<N>(b), c); }
template <int N>
__device__ __forceinline__ VN<N> fma2(VN<N> a, float b, float c) { return fma2(a, sp<N>(b), sp<N>(c)); }
// component k (0..N-1)
template <int N>
__device__ __forceinline__ float comp(const VN<N>& a, int k) { return (k & 1) ? a.h[k >> 1].y : a.h[k >> 1].x; }

// SFU (MUFU) approximations with flush-to-zero, per component (sin/cos add
// the FMUL by 1/2pi the SFU expects).  Absolute error of sin/cos ~2^-21 on
// [-pi, pi]; rcp/rsqrt ~1 ulp.
__device__ __forceinline__ float rcp_a(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsq_a(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void sincos_a(float x, float& s, float& c) {
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(x));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(x));
}
template <int N>
__device__ __forceinline__ VN<N> rcp2(VN<N> a) { VN_MAP1(make_float2(rcp_a(a.h[i].x), rcp_a(a.h[i].y))) }
template <int N>
__device__ __forceinline__ VN<N> rsq2(VN<N> a) { VN_MAP1(make_float2(rsq_a(a.h[i].x), rsq_a(a.h[i].y))) }
template <int N>
__device__ __forceinline__ void sincos2(VN<N> a, VN<N>& s, VN<N>& c) {
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    sincos_a(a.h[i].x, s.h[i].x, c.h[i].x);
    sincos_a(a.h[i].y, s.h[i].y, c.h[i].y);
  }
}
template <int N>
__device__ __forceinline__ VN<N> rint2(VN<N> a) { VN_MAP1(make_float2(rintf(a.h[i].x), rintf(a.h[i].y))) }
// maximum(x, f) == where(x >= f, x, f): fmaxf has the same NaN behaviour
template <int N>
__device__ __forceinline__ VN<N> vmax(VN<N> a, float f) {
  VN_MAP1(make_float2(fmaxf(a.h[i].x, f), fmaxf(a.h[i].y, f)))
}
template <int N>
__device__ __forceinline__ VN<N> clamp95(VN<N> a) {
  VN_MAP1(make_float2(fminf(fmaxf(a.h[i].x, -0.95f), 0.95f), fminf(fmaxf(a.h[i].y, -0.95f), 0.95f)))
}
// x < f ? f : x  (the em floor of kernel.py:406; NaN propagates)
template <int N>
__device__ __forceinline__ VN<N> floor_sel(VN<N> a, float f) {
  VN_MAP1(make_float2(a.h[i].x < f ? f : a.h[i].x, a.h[i].y < f ? f : a.h[i].y))
}
// x == 0 ? tiny : x
template <int N>
__device__ __forceinline__ VN<N> nonzero(VN<N> a, float tiny) {
  VN_MAP1(make_float2(a.h[i].x == 0.0f ? tiny : a.h[i].x, a.h[i].y == 0.0f ? tiny : a.h[i].y))
}

// x0 + (rate_hi + rate_lo) * (t + tl), reduced mod 2*pi, in double-float:
// p = rate_hi*t rounded, its exact error by fma, k = nearest revolution;
// p - k*2pi_hi is exact (the difference needs < 24 bits: DESIGN.md §4).
template <bool LO, int N>
__device__ __forceinline__ VN<N> secular_angle(float x0, float rate, float rate_lo, VN<N> t, VN<N> tl) {
  const VN<N> p = t * rate;
  VN<N> e = fma2(t, rate, -p);
  e = fma2(t, rate_lo, e);
  if constexpr (LO) e = fma2(tl, rate, e);
  // k = rint(p / 2pi) by the 1.5 2^23 shifter (packed, |p / 2pi| < 2^22)
  const VN<N> k = fma2(p, kInvTwoPiF, kRoundMagicF) - kRoundMagicF;
  VN<N> r = fma2(-k, kTwoPiHiF, p);
  r = fma2(-k, kTwoPiLoF, r);
  return r + (e + x0);
}

// The same angle on the FP64 pipe (SGP4B_SEC64): u = U0 + (UDOT_hi +
// UDOT_lo) t in fp64 (t, U0 exact in fp64), reduced by k = rint(u / 2pi)
// with one fma (|u| < 2^20 rad), rounded to fp32 once.  Moves the 9 FP32
// ops of the double-float form to the otherwise idle FP64 pipe, at the cost
// of two conversions per cell.
template <bool LO, int N>
__device__ __forceinline__ VN<N> secular_angle64(float x0, double rate, VN<N> t, VN<N> tl) {
  VN<N> out;
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    double t0 = (double)t.h[i].x, t1 = (double)t.h[i].y;
    if constexpr (LO) {
      t0 += (double)tl.h[i].x;
      t1 += (double)tl.h[i].y;
    }
    const double u0 = fma(rate, t0, (double)x0);
    const double u1 = fma(rate, t1, (double)x0);
    const double k0 = fma(u0, 0.15915494309189535, 6755399441055744.0) - 6755399441055744.0;
    const double k1 = fma(u1, 0.15915494309189535, 6755399441055744.0) - 6755399441055744.0;
    out.h[i] = make_float2((float)fma(-k0, 6.283185307179586, u0),
                           (float)fma(-k1, 6.283185307179586, u1));
  }
  return out;
}

// (sin, cos)(a + d) from (sin, cos)(a) for |d| < 4e-3 (the J2 short-period
// corrections and the last Newton step): d^3/6 < 1.1e-8 is below fp32
// resolution, so sin d = d, cos d = 1 - d^2/2.
template <int N>
__device__ __forceinline__ void rotate_tiny(VN<N> s, VN<N> c, VN<N> d, VN<N>& so, VN<N>& co) {
  const VN<N> cd = fma2(d * d, -0.5f, 1.0f);
  so = fma2(s, cd, c * d);
  co = fma2(c, cd, (-s) * d);
}

// fp32 cells of one satellite.  ISIMP and KITER are warp-uniform per
// satellite and compile-time here, so the cell is straight-line code.
// KITER = 0: runtime Kepler count with a final SFU sincos (eccentric
// orbits).  `R[i]` is the satellite's packed fp32 record (P_* slots): every
// per-satellite product the reference forms per cell is pre-multiplied there
// (in fp64, rounded once), including 0.5 j2, the Earth radius and the km/s
// scale, so the cell spends its FP32 issue slots on per-cell work only.
template <bool ISIMP, int KITER, bool LO, int NC, class RT>
__device__ __forceinline__ void cellv(const RT& R, VN<NC> t, VN<NC> tl, const Grav& g,
                                      VN<NC> (&o)[6], int (&code)[NC]) {
  using V2 = VN<NC>;
  const float tiny = FLT_MIN;
  const int flags = R.flags();

  // secular gravity  kernel.py:366-370.  Only the Kepler argument needs the
  // double-float treatment: u = (mo + argpo) + (mdot + argpdot) t + ...
  // (mm + argpm; the drag term cancels), the rest enter sin/cos damped.
  const V2 argpdf = fma2(t, R[P_ARGPDOT], sp<NC>(R[P_ARGPO]));
  const V2 t2 = t * t;
  const V2 nodem = fma2(t2, R[P_NODECF], fma2(t, R[P_NODEDOT], sp<NC>(R[P_NODEO])));
#if SGP4B_SEC64
  const V2 ubase = secular_angle64<LO, NC>(R[P_U0], (double)R[P_UDOT] + (double)R[P_UDOT_LO],
                                           t, tl);
#else
  const V2 ubase = secular_angle<LO, NC>(R[P_U0], R[P_UDOT], R[P_UDOT_LO], t, tl);
#endif

  // drag  kernel.py:371-391.  With s = sqrt((xke/no)^(2/3)) folded in,
  // sqrt(am) = s tempa is one Horner polynomial in t; no templ is another.
  V2 sqa, nol, argpm, em;
  if constexpr (ISIMP) {
    sqa = fma2(t, R[P_SC1], sp<NC>(R[P_S]));                       // s (1 - cc1 t)
    nol = t2 * R[P_N2];                                            // no t2cof t^2
    em = fma2(t, -R[P_BC4], sp<NC>(R[P_E0]));                     // ecco - bstar cc4 t
    argpm = argpdf;
  } else {
    // xmdf = mo + mdot t = (mo + argpo + (mdot + argpdot) t) - argpdf,
    // from the reduced Kepler argument: a small angle for the SFU
    const V2 xmdf = ubase - argpdf;
    V2 sx, cx;
    sincos2(xmdf, sx, cx);
    // delomg + delm = omgcof t + xmcof ((1 + eta cos xmdf)^3 - delmo), the
    // cubic expanded in cos xmdf (better conditioned than cubing 1 + eta cx)
    V2 temp;
    if constexpr (KITER == 1) {
      // e < 0.003: eta = ao e tsi < 0.06, so the eta^2, eta^3 terms are below
      // 3e-7 rad of the small drag angle, which only reaches r through
      // em sin/cos(argpm) (< 1e-7 m)
      temp = fma2(cx, R[P_A1], fma2(t, R[P_OMGCOF], sp<NC>(R[P_A0])));
    } else {
      temp = fma2(fma2(fma2(cx, R[P_A3], sp<NC>(R[P_A2])), cx, sp<NC>(R[P_A1])), cx,
                  fma2(t, R[P_OMGCOF], sp<NC>(R[P_A0])));
    }
    // s (1 - cc1 t - d2 t^2 - d3 t^3 - d4 t^4)
    sqa = fma2(t, fma2(t, fma2(t, fma2(t, R[P_SD4], sp<NC>(R[P_SD3])), sp<NC>(R[P_SD2])),
                       sp<NC>(R[P_SC1])), sp<NC>(R[P_S]));
    // no (t2cof t^2 + t3cof t^3 + t4cof t^4 + t5cof t^5)
    nol = t2 * fma2(t, fma2(t, fma2(t, R[P_N5], sp<NC>(R[P_N4])), sp<NC>(R[P_N3])),
                    sp<NC>(R[P_N2]));
    // em = ecco - bstar cc4 t - bstar cc5 (sin(xmdf + temp) - sinmao), the
    // sine expanded to first order in the small drag angle temp; E0 holds
    // ecco + bstar cc5 sinmao
    em = fma2(fma2(cx, temp, sx), -R[P_BC5], fma2(t, -R[P_BC4], sp<NC>(R[P_E0])));
    argpm = argpdf - temp;
  }

  // mean motion / eccentricity  kernel.py:397-408
  const V2 am = vmax(sqa * sqa, tiny);                            // maximum(am, tiny)
  const V2 rsam = rsq2(am);
  bool bad_em[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) bad_em[k] = (comp(em, k) >= 1.0f) || (comp(em, k) < -0.001f);
  em = floor_sel(em, 1.0e-6f);

  // long-period periodics  kernel.py:420-431
  V2 sa, ca;
  sincos2(argpm, sa, ca);
  const V2 axnl = em * ca;
  const V2 rsam2 = rsam * rsam;                                   // 1 / am
  V2 ilp;                                                         // 1 / pl_lp
  if constexpr (KITER == 1) {
    // class 1 (e < 0.003): 1 / (am (1 - em^2)) = (1 + em^2) / am
    // to O(em^4) < 1e-9, the guard pl_lp > tiny is implied
    ilp = fma2(em, em, 1.0f) * rsam2;
  } else if constexpr (KITER == 2 && SGP4B_K2_SERIES) {
    // class 2 (e < 0.1): (1 + em^2 + em^4) / am, truncation em^6 < 1e-6
    // relative on terms of order 1e-3 (aycof, xlcof)
    const V2 em2 = em * em;
    ilp = fma2(em2, em2 + 1.0f, 1.0f) * rsam2;
  } else {
    ilp = rcp2(vmax(am * fma2(-em, em, 1.0f), tiny));
  }
  const V2 aynl = fma2(em, sa, ilp * R[P_AYCOF]);
  // u = xl - nodep = mm + argpm + (xlcof/pl) axnl  (mod 2pi)
  const V2 u = fma2(ilp * R[P_XLCOF], axnl, ubase + nol);

  // Kepler, fixed warp-uniform iteration count  kernel.py:325-349.  E is
  // carried as u + d so the residual u - E + axnl sinE - aynl cosE is formed
  // without cancelling against u.
  V2 s, c, d = sp<NC>(0.0f), tem5 = sp<NC>(0.0f);
  V2 eo1 = u;
  const int kiter = KITER > 0 ? KITER : 10;     // the reference loop bound
#pragma unroll
  for (int it = 0; it < (KITER > 0 ? KITER : 16); ++it) {
    if (KITER == 0 && it >= kiter) break;
    sincos2(it == 0 ? u : (KITER > 0 ? u + d : eo1), s, c);
    V2 num;
    if constexpr (KITER > 0) {
      num = it == 0 ? fma2(axnl, s, (-aynl) * c) : fma2(axnl, s, fma2(-aynl, c, -d));
    } else {
      num = fma2(axnl, s, fma2(-aynl, c, u)) - eo1;
    }
    if constexpr (KITER == 1) {
      // den = 1 - q with |q| <= e < 0.004: 1/den = 1 + q + q^2 to O(q^3)
      const V2 q = fma2(c, axnl, s * aynl);
      tem5 = num * fma2(q, q + 1.0f, 1.0f);
    } else if constexpr (KITER == 2 && SGP4B_K2_SERIES) {
      // |q| <= e < 0.1: the first step's 1 + q + q^2 (error q^3 e) is
      // absorbed by the second Newton step, the last step's 1 + q + q^2 + q^3
      // leaves q^4 of a step below e^3/2
      const V2 q = fma2(c, axnl, s * aynl);
      const V2 q1 = q + 1.0f;
      tem5 = num * (it == 0 ? fma2(q, q1, 1.0f) : fma2(q, fma2(q, q1, 1.0f), 1.0f));
    } else {
      const V2 den = fma2(-s, aynl, fma2(-c, axnl, 1.0f));
      tem5 = num * rcp2(den);
    }
    // the +-0.95 clamp (kernel.py:343-346) cannot trigger for e < 0.1
    // (|num| <= 2e, den >= 1 - 2e), i.e. for KITER 1 and 2
    if (KITER == 0 || KITER > 2) tem5 = clamp95(tem5);
    if constexpr (KITER > 0) d = it == 0 ? tem5 : d + tem5;
    else eo1 = eo1 + tem5;
  }
  V2 sineo1, coseo1;
  if constexpr (KITER == 1 || KITER == 2) {
    // E = u + d straight through the SFU: the FMA pipe is the binding
    // resource and the XU has room (12 vs 10 MUFU per cell measured 2 %
    // faster than the 6-op rotation); accuracy is the same SFU-level
    sincos2(u + d, sineo1, coseo1);
  } else if constexpr (KITER > 0) {
    rotate_tiny(s, c, tem5, sineo1, coseo1);     // last step <= e^3/2 < 4e-3
  } else {
    sincos2(eo1, sineo1, coseo1);
  }

  // short-period preliminaries  kernel.py:440-460
  const V2 ecose = fma2(axnl, coseo1, aynl * sineo1);
  const V2 esine = fma2(axnl, sineo1, (-aynl) * coseo1);
  const V2 el2 = fma2(axnl, axnl, aynl * aynl);
  const V2 omel2 = 1.0f - el2;
  bool bad_pl[NC];
  const V2 ome = 1.0f - ecose;
  const V2 rl = am * ome;
  const V2 nrm = rcp2(nonzero(ome, tiny));                 // am / rl (am > 0)
  V2 betal, tq, ipl;
  if constexpr (KITER == 1) {
    // x = el2 < 2e-5: sqrt(1-x), 1/sqrt(1-x) and 1/(1 + sqrt(1-x)) as
    // first-order series (truncation < 4e-9 even at e = 0.01); pl < 0 iff
    // el2 > 1
#pragma unroll
    for (int k = 0; k < NC; ++k) bad_pl[k] = comp(el2, k) > 1.0f;
    betal = fma2(el2, -0.5f, 1.0f);
    tq = esine * fma2(el2, 0.125f, 0.5f);
    ipl = fma2(rsam2, el2, rsam2);                         // (1 + el2) / am
  } else if constexpr (KITER == 2) {
    // e < 0.1: pl = am (1 - el2), and am > 0, so the sign test of pl is
    // that of 1 - el2; one SFU rsqrt serves betal, sqrt(pl) and 1/pl
#pragma unroll
    for (int k = 0; k < NC; ++k) bad_pl[k] = comp(omel2, k) < 0.0f;
    const V2 rb = rsq2(omel2);
    betal = omel2 * rb;
    if constexpr (SGP4B_K2_SERIES) {
      // 1/(1 + sqrt(1-x)) = 1/2 + x/8 + x^2/16 + O(5x^3/128), x = el2 < 0.0121
      tq = esine * fma2(el2, fma2(el2, 0.0625f, 0.125f), 0.5f);
    } else {
      tq = esine * rcp2(betal + 1.0f);
    }
    const V2 rspl = rsam * rb;
    ipl = rspl * rspl;
  } else {
    const V2 pl = am * omel2;
#pragma unroll
    for (int k = 0; k < NC; ++k) bad_pl[k] = comp(pl, k) < 0.0f;
    const V2 rspl = rsq2(vmax(pl, tiny));
    const V2 ob = vmax(omel2, tiny);
    betal = ob * rsq2(ob);
    tq = esine * rcp2(betal + 1.0f);
    // sqrt(pl_safe) / rl = (am/rl) betal when pl > tiny; otherwise use the
    // guarded form
    ipl = rspl * rspl;
  }
  // sqrt(am) / rl and sqrt(pl) / rl in km/s: (am/rl) (vkm / sqrt(am))
  const V2 sqv = nrm * (rsam * g.vkm_f);
  const V2 rdv = sqv * esine;                              // rdotl vkm
  V2 rvdv = sqv * betal;                                   // rvdotl vkm
  if constexpr (KITER == 0 || KITER > 2) {
    // general orbits: sqrt(pl_safe) may differ from sqrt(am) betal
    const V2 pl = am * omel2;
    const V2 pls = vmax(pl, tiny);
    rvdv = (pls * rsq2(pls)) * (nrm * (rsam2 * g.vkm_f));  // sqrt(pl) / rl
  }
  // (sin u, cos u) = (am/rl) (sn, cs)  (kernel.py:453-454); the atan2 of
  // :455 is only ever used through sin/cos, so no angle is formed.
  const V2 sinu = fma2(-axnl, tq, sineo1 - aynl) * nrm;
  const V2 cosu = fma2(aynl, tq, coseo1 - axnl) * nrm;
  const V2 s2u = sinu + sinu;
  const V2 sin2u = s2u * cosu;
  const V2 cos2u = fma2(-s2u, sinu, 1.0f);
  const V2 ipl2 = ipl * ipl;                               // temp2 / (0.5 j2)

  // short-period periodics  kernel.py:463-469 (0.5 j2, re and the km/s
  // scale pre-multiplied into the record's per-satellite factors)
  // mr = re mrt; for e < 0.003 betal = 1 - O(1e-5) in the J2 term (< 1e-8)
  const V2 k41 = KITER == 1 ? fma2(ipl2, R[P_K41R], sp<NC>(g.re_f))
                            : fma2(ipl2 * R[P_K41R], betal, sp<NC>(g.re_f));
  const V2 mr = fma2(rl, k41, (ipl * R[P_KXR]) * cos2u);
  const V2 t2s = ipl2 * sin2u;
  const V2 dsu = t2s * R[P_QX];
  const V2 dinc = (ipl2 * cos2u) * R[P_C15CS];
  const V2 nmt = rsam2 * rsam * ipl;                       // nm temp1 / (xke 0.5 j2)
  const V2 mv = fma2(-(nmt * R[P_X1V]), sin2u, rdv);
  const V2 rv = fma2(nmt, fma2(cos2u, R[P_X1V], sp<NC>(R[P_C41V])), rvdv);

  // orientation  kernel.py:472-493
  V2 sinsu, cossu, snod, cnod, sini, cosi;
  rotate_tiny(sinu, cosu, dsu, sinsu, cossu);
  sincos2(fma2(t2s, R[P_C15CO], nodem), snod, cnod);     // xnode
  // xinc = inclo + dinc with |dinc| <= 1.5 temp2 |cos i sin i| < 4e-4: the
  // second-order term dinc^2/2 < 8e-8 is below fp32 resolution of r and v
  sini = fma2(dinc, R[P_COSIO], sp<NC>(R[P_SINIO]));
  cosi = fma2(dinc, -R[P_SINIO], sp<NC>(R[P_COSIO]));
  // r = mr U, v = mv U + rv V with U, V the orientation vectors; grouped as
  // r = (xm, cnod|snod, sini) . (mr sinsu, mr cossu), same for v
  const V2 xmx = (-snod) * cosi;
  const V2 xmy = cnod * cosi;
  const V2 ra = mr * sinsu, rb = mr * cossu;
  o[0] = fma2(xmx, ra, cnod * rb);
  o[1] = fma2(xmy, ra, snod * rb);
  o[2] = sini * ra;
  const V2 va = fma2(mv, sinsu, rv * cossu);
  const V2 vb = fma2(mv, cossu, (-rv) * sinsu);
  o[3] = fma2(xmx, va, cnod * vb);
  o[4] = fma2(xmy, va, snod * vb);
  o[5] = sini * va;

  // _first_error 2 > 1 > 4 > 6 and the init merge  kernel.py:497-502, 529-534
  // (decayed: mrt < 1 earth radius, i.e. mr < re)
  const int persistent = (flags >> CODE_SHIFT) & 0x7fffff; // includes bad_nm -> 2
#pragma unroll
  for (int h = 0; h < NC; ++h) {
    const int cellc = bad_em[h] ? 1 : bad_pl[h] ? 4 : (comp(mr, h) < g.re_f) ? 6 : 0;
    code[h] = persistent != 0 ? persistent : cellc;
  }
}

// ======================================================================
// Packing: SoA fp64 satrec -> packed record (per satellite, fp64 math)
// ======================================================================
__device__ __forceinline__ int kepler_iters_for(double ecco) {
  // fp32 Newton from E0 = u: |E - E_k| <~ e^(2^(k+1)-1) / 2^(2^k-1); these
  // counts reach fp32 resolution.  The margin covers the
  // drag-driven change of em = ecco - tempe over the propagation span.
  const double e = fabs(ecco) + 0.001;
  if (e < 0.004) return 1;
  if (e < 0.1) return 2;
  if (e < 0.4) return 3;
  return 10;
}

// split x into a float hi word and the float nearest the remainder
__device__ __forceinline__ void split_df(double x, float& hi, float& lo) {
  hi = (float)x;
  lo = (float)(x - (double)hi);
}

template <typename T>
__device__ __forceinline__ void store_record(const double* f, const double* v, int flags,
                                             bool isimp, const Grav& g, T* __restrict__ rec);

// (xke / n)^(2/3) as cbrt squared: within 2 ulp of pow(x, 2/3) (the
// reference's np.power), at a fraction of the libdevice pow chain
__device__ __forceinline__ double pow2o3(double x) {
  const double c = cbrt(x);
  return c * c;
}

// flags word of a record: isimp, Kepler class, persistent init code
__device__ __forceinline__ int record_flags(const double* f, int init_code, bool isimp) {
  const bool bad_nm = f[F_NO_UNKOZAI] <= 0.0;
  // kernel.py:532: init codes persist except 6; bad_nm (per satellite) is
  // folded in behind them, preserving _first_error precedence 2 > 1 > 4 > 6
  int persistent = init_code == 6 ? 0 : init_code;
  if (persistent == 0 && bad_nm) persistent = 2;
  return (isimp ? FLAG_ISIMP : 0) | (bad_nm ? FLAG_BAD_NM : 0) |
         (kepler_iters_for(f[F_ECCO]) << KEPLER_SHIFT) | ((persistent & 0x7fffff) << CODE_SHIFT);
}

// fp64 record values (flags slot left 0; see record_flags)
// ao_sc = (ao, sin inclo, cos inclo) when the caller already has them (the
// init kernel); otherwise they are recomputed from the satrec fields
__device__ __forceinline__ void record_values(const double* f, const Grav& g, double* out,
                                              const double* ao_sc = nullptr) {
  const double no = f[F_NO_UNKOZAI];
  const bool bad_nm = no <= 0.0;
  const double nm_safe = bad_nm ? 1.0e-4 : no;
  out[S_MO] = f[F_MO];
  out[S_MDOT] = f[F_MDOT];
  out[S_ARGPO] = f[F_ARGPO];
  out[S_ARGPDOT] = f[F_ARGPDOT];
  out[S_NODEO] = f[F_NODEO];
  out[S_NODEDOT] = f[F_NODEDOT];
  out[S_NODECF] = f[F_NODECF];
  out[S_CC1] = f[F_CC1];
  out[S_BC4] = f[F_BSTAR] * f[F_CC4];
  out[S_T2COF] = f[F_T2COF];
  out[S_OMGCOF] = f[F_OMGCOF];
  out[S_ETA] = f[F_ETA];
  out[S_XMCOF] = f[F_XMCOF];
  out[S_DELMO] = f[F_DELMO];
  out[S_D2] = f[F_D2];
  out[S_D3] = f[F_D3];
  out[S_D4] = f[F_D4];
  out[S_BC5] = f[F_BSTAR] * f[F_CC5];
  out[S_SINMAO] = f[F_SINMAO];
  out[S_T3COF] = f[F_T3COF];
  out[S_T4COF] = f[F_T4COF];
  out[S_T5COF] = f[F_T5COF];
  out[S_NO] = no;
  // (xke / nm_safe)^(2/3) is the init's ao unless n <= 0
  out[S_AM0] = (ao_sc != nullptr && !bad_nm) ? ao_sc[0] : pow2o3(g.xke / nm_safe);
  out[S_ECCO] = f[F_ECCO];
  out[S_INCLO] = f[F_INCLO];
  double si, ci;
  if (ao_sc != nullptr) {
    si = ao_sc[1];
    ci = ao_sc[2];
  } else {
    sincos(f[F_INCLO], &si, &ci);
  }
  out[S_SINIO] = si;
  out[S_COSIO] = ci;
  out[S_AYCOF] = f[F_AYCOF];
  out[S_XLCOF] = f[F_XLCOF];
  out[S_CON41] = f[F_CON41];
  out[S_X1MTH2] = f[F_X1MTH2];
  out[S_X7THM1] = f[F_X7THM1];
  out[S_FLAGS] = 0.0;
  out[S64_SQAM0] = sqrt(out[S_AM0]);
  out[S64_NOSAFE] = g.xke / (out[S_AM0] * out[S64_SQAM0]);
  out[S_NODEDOT_LO] = 0.0;
  out[S_UDOT] = f[F_MDOT] + f[F_ARGPDOT];
  out[S_UDOT_LO] = 0.0;
  out[S_U0] = pymod_2pi(f[F_MO] + f[F_ARGPO]);
}

template <>
__device__ __forceinline__ void store_record<double>(const double* f, const double* v, int flags,
                                                     bool isimp, const Grav& g,
                                                     double* __restrict__ rec) {
  double o[S_COUNT];
#pragma unroll
  for (int i = 0; i < S_COUNT; ++i) o[i] = 0.0;
  const double hj2 = 0.5 * g.j2, bstar = f[F_BSTAR], no = v[S_NO];
  const double s = v[S64_SQAM0];
  o[Q_ARGPO] = f[F_ARGPO];
  o[Q_ARGPDOT] = f[F_ARGPDOT];
  o[Q_NODEO] = f[F_NODEO];
  o[Q_NODEDOT] = f[F_NODEDOT];
  o[Q_NODECF] = f[F_NODECF];
  o[Q_MO] = f[F_MO];
  o[Q_MDOT] = f[F_MDOT];
  o[Q_U0] = v[S_U0];
  o[Q_UDOT] = v[S_UDOT];
  o[Q_S] = s;
  o[Q_SC1] = -s * f[F_CC1];
  o[Q_N2] = no * f[F_T2COF];
  o[Q_E0] = f[F_ECCO];
  o[Q_BC4] = bstar * f[F_CC4];
  if (!isimp) {                       // kernel.py:371-391 (zero in isimp records)
    const double eta = f[F_ETA], xmcof = f[F_XMCOF];
    o[Q_A0] = xmcof * (1.0 - f[F_DELMO]);
    o[Q_A1] = 3.0 * xmcof * eta;
    o[Q_A2] = 3.0 * xmcof * eta * eta;
    o[Q_A3] = xmcof * eta * eta * eta;
    o[Q_OMGCOF] = f[F_OMGCOF];
    o[Q_SD2] = -s * f[F_D2];
    o[Q_SD3] = -s * f[F_D3];
    o[Q_SD4] = -s * f[F_D4];
    o[Q_N3] = no * f[F_T3COF];
    o[Q_N4] = no * f[F_T4COF];
    o[Q_N5] = no * f[F_T5COF];
    o[Q_BC5] = bstar * f[F_CC5];
    o[Q_E0] = f[F_ECCO] + bstar * f[F_CC5] * f[F_SINMAO];
  }
  o[Q_AYCOF] = f[F_AYCOF];
  o[Q_XLCOF] = f[F_XLCOF];
  o[Q_K41R] = -1.5 * f[F_CON41] * hj2 * g.re;
  o[Q_KXR] = 0.5 * f[F_X1MTH2] * hj2 * g.re;
  o[Q_QX] = -0.25 * f[F_X7THM1] * hj2;
  o[Q_C15CO] = 1.5 * v[S_COSIO] * hj2;
  o[Q_C15CS] = 1.5 * v[S_COSIO] * v[S_SINIO] * hj2;
  o[Q_X1V] = f[F_X1MTH2] * hj2 * g.vkm;
  o[Q_C41V] = 1.5 * f[F_CON41] * hj2 * g.vkm;
  o[Q_SINIO] = v[S_SINIO];
  o[Q_COSIO] = v[S_COSIO];
  o[Q_INCLO] = f[F_INCLO];
  o[Q_FLAGS] = __longlong_as_double((long long)flags);
#pragma unroll
  for (int i = 0; i < S_COUNT; ++i) rec[i] = o[i];
}

// reduce an angle to [-pi, pi): fp32 has the most resolution there
__device__ __forceinline__ double signed_2pi(double x) {
  const double r = pymod_2pi(x);
  return r >= kPi ? r - kTwoPi : r;
}

template <>
__device__ __forceinline__ void store_record<float>(const double* f, const double* v, int flags,
                                                    bool isimp, const Grav& g,
                                                    float* __restrict__ rec) {
  double o[S_COUNT];
#pragma unroll
  for (int i = 0; i < S_COUNT; ++i) o[i] = 0.0;
  const double hj2 = 0.5 * g.j2, bstar = f[F_BSTAR], no = v[S_NO];
  const double s = sqrt(v[S_AM0]);
  o[P_MO] = signed_2pi(f[F_MO]);
  o[P_MDOT] = f[F_MDOT];
  o[P_ARGPO] = signed_2pi(f[F_ARGPO]);
  o[P_ARGPDOT] = f[F_ARGPDOT];
  o[P_NODEO] = signed_2pi(f[F_NODEO]);
  o[P_NODEDOT] = f[F_NODEDOT];
  o[P_NODECF] = f[F_NODECF];
  o[P_U0] = signed_2pi(v[S_U0]);
  o[P_S] = s;
  o[P_SC1] = -s * f[F_CC1];
  o[P_N2] = no * f[F_T2COF];
  o[P_E0] = f[F_ECCO];
  o[P_BC4] = bstar * f[F_CC4];
  if (!isimp) {                       // kernel.py:371-391 (zero in isimp records)
    const double eta = f[F_ETA], xmcof = f[F_XMCOF];
    o[P_A0] = xmcof * (1.0 - f[F_DELMO]);
    o[P_A1] = 3.0 * xmcof * eta;
    o[P_A2] = 3.0 * xmcof * eta * eta;
    o[P_A3] = xmcof * eta * eta * eta;
    o[P_OMGCOF] = f[F_OMGCOF];
    o[P_SD2] = -s * f[F_D2];
    o[P_SD3] = -s * f[F_D3];
    o[P_SD4] = -s * f[F_D4];
    o[P_N3] = no * f[F_T3COF];
    o[P_N4] = no * f[F_T4COF];
    o[P_N5] = no * f[F_T5COF];
    o[P_BC5] = bstar * f[F_CC5];
    o[P_E0] = f[F_ECCO] + bstar * f[F_CC5] * f[F_SINMAO];
  }
  o[P_AYCOF] = f[F_AYCOF];
  o[P_XLCOF] = f[F_XLCOF];
  o[P_K41R] = -1.5 * f[F_CON41] * hj2 * g.re;
  o[P_KXR] = 0.5 * f[F_X1MTH2] * hj2 * g.re;
  o[P_QX] = -0.25 * f[F_X7THM1] * hj2;
  o[P_C15CO] = 1.5 * v[S_COSIO] * hj2;
  o[P_C15CS] = 1.5 * v[S_COSIO] * v[S_SINIO] * hj2;
  o[P_X1V] = f[F_X1MTH2] * hj2 * g.vkm;
  o[P_C41V] = 1.5 * f[F_CON41] * hj2 * g.vkm;
  o[P_SINIO] = v[S_SINIO];
  o[P_COSIO] = v[S_COSIO];
  float r[S_COUNT];
#pragma unroll
  for (int i = 0; i < S_COUNT; ++i) r[i] = (float)o[i];
  split_df(v[S_UDOT], r[P_UDOT], r[P_UDOT_LO]);
  r[P_FLAGS] = __int_as_float(flags);
#pragma unroll
  for (int i = 0; i < S_COUNT; ++i) rec[i] = r[i];
}

// ======================================================================
// Init (kernel.py:154-322), fp64, one thread per satellite
// ======================================================================

// The epoch evaluation of kernel.py:316-322: _propagate at t = 0, where the
// secular and drag terms vanish exactly (xmdf = mo, tempa = 1, tempe =
// templ = delm = 0, so mm = mo, argpm = argpo, nodem = nodeo, em = ecco,
// am = ao), reduced to what decides its code: _first_error 2 > 1 > 4 > 6
// (kernel.py:393-414, 419-431, 325-349, 440-469, 495-502) in the
// reference's operation order, with the reference Kepler loop.  Only the
// code is kept, so the orientation and velocity terms are not formed.
__device__ int epoch_code(const double* f, double ao, const Grav& g) {
  const double tiny = DBL_MIN;
  const bool bad_nm = f[F_NO_UNKOZAI] <= 0.0;
  const double am = bad_nm ? pow2o3(g.xke / 1.0e-4) : ao;        // tempa = 1
  const double am_safe = gmax(am, tiny);
  double em = f[F_ECCO];
  const bool bad_em = (em >= 1.0) || (em < -0.001);
  em = em < 1.0e-6 ? 1.0e-6 : em;
  // floor-mods as kernel.py:407-411 (templ = 0: mm = mo)
  const double nodeo = f[F_NODEO];
  const double nodem = nodeo >= 0.0 ? pymod_2pi(nodeo) : -pymod_2pi(-nodeo);
  const double argpm = pymod_2pi(f[F_ARGPO]);
  const double xlm = pymod_2pi(f[F_MO] + f[F_ARGPO] + nodeo);
  const double mm = pymod_2pi(xlm - argpm - nodem);
  double sa, ca;
  sincos(argpm, &sa, &ca);
  const double axnl = em * ca;
  const double temp_lp = 1.0 / gmax(am_safe * (1.0 - em * em), tiny);
  const double aynl = em * sa + temp_lp * f[F_AYCOF];
  const double xl = mm + argpm + nodem + temp_lp * f[F_XLCOF] * axnl;
  const double u = pymod_2pi(xl - nodem);
  // solve_kepler  kernel.py:325-349
  double eo1 = u;
  bool live = true;
  for (int it = 0; it < 10 && live; ++it) {
    double s, c;
    sincos(eo1, &s, &c);
    double step = 1.0 - c * axnl - s * aynl;
    step = (u - aynl * c + axnl * s - eo1) / step;
    step = step >= 0.95 ? 0.95 : (step <= -0.95 ? -0.95 : step);
    eo1 += step;
    live = fabs(step) >= 1.0e-12;
  }
  double sineo1, coseo1;
  sincos(eo1, &sineo1, &coseo1);
  const double ecose = axnl * coseo1 + aynl * sineo1;
  const double esine = axnl * sineo1 - aynl * coseo1;
  const double el2 = axnl * axnl + aynl * aynl;
  const double pl = am_safe * (1.0 - el2);
  const bool bad_pl = pl < 0.0;
  const double pl_safe = gmax(pl, tiny);
  const double rl = am_safe * (1.0 - ecose);
  const double rl_safe = rl == 0.0 ? tiny : rl;
  const double betal = sqrt(gmax(1.0 - el2, tiny));
  const double temp = esine / (1.0 + betal);
  const double sinu = am_safe / rl_safe * (sineo1 - aynl - axnl * temp);
  const double cos2u = 1.0 - 2.0 * sinu * sinu;
  const double ipl = 1.0 / pl_safe;
  const double temp1 = 0.5 * g.j2 * ipl;
  const double temp2 = temp1 * ipl;
  const double mrt = rl * (1.0 - 1.5 * temp2 * betal * f[F_CON41]) +
                     0.5 * temp1 * f[F_X1MTH2] * cos2u;
  return bad_nm ? 2 : bad_em ? 1 : bad_pl ? 4 : (mrt < 1.0) ? 6 : 0;
}

// true when the epoch evaluation (epoch_code) provably returns 0, from
// bounds that hold for every E: with el = |(axnl, aynl)| <= em +
// |aycof| / pl_lp =: elb, ecose <= el gives rl >= am (1 - elb), pl >= am
// (1 - elb^2) bounds temp1 = j2/2/pl and temp2 = temp1/pl, and betal,
// cos2u lie in [0, 1] and [-1, 1], so (kernel.py:495-502)
//   mrt >= am (1 - elb) (1 - 1.5 temp2 |con41|) - temp1/2 |x1mth2|,
// and pl > 0.  A margin of 1e-6 covers the rounding of both evaluations.
// Every ordinary orbit passes and skips the Kepler loop; anything near a
// threshold (or outside 1e-6 <= em < 0.5, or bad_nm) takes the exact path.
__device__ __forceinline__ bool epoch_clear(const double* f, double ao, const Grav& g) {
  const double em = f[F_ECCO];
  if (!(f[F_NO_UNKOZAI] > 0.0) || !(em >= 1.0e-6 && em < 0.5) || !(ao > 0.0)) return false;
  const double tlp = 1.0 / (ao * (1.0 - em * em));
  const double elb = em + tlp * fabs(f[F_AYCOF]);
  if (!(elb < 0.5)) return false;
  const double plmin = ao * (1.0 - elb * elb);
  const double t1 = 0.5 * fabs(g.j2) / plmin;
  const double t2 = t1 / plmin;
  const double k = 1.5 * t2 * fabs(f[F_CON41]);
  if (!(k < 1.0)) return false;
  const double lb = ao * (1.0 - elb) * (1.0 - k) - 0.5 * t1 * fabs(f[F_X1MTH2]);
  return lb > 1.0 + 1.0e-6;
}

__device__ void init_one(const double el[7], const Grav& g, double* f, double* v, int& code,
                         bool& isimp_out) {
  const double tiny = DBL_MIN;
  const double xke = g.xke, j2 = g.j2, j3oj2 = g.j3oj2, j4 = g.j4, re = g.re;
  const double no_kozai = el[0], ecco = el[1], inclo = el[2], nodeo = el[3];
  const double argpo = el[4], mo = el[5], bstar = el[6];

  const bool bad_n = no_kozai <= 0.0;                              // :177
  const bool bad_e = (ecco >= 1.0) || (ecco < -0.001);             // :178
  const double no_safe = bad_n ? 1.0e-4 : no_kozai;

  const double eccsq = ecco * ecco;
  const double omeosq = gmax(1.0 - eccsq, tiny);
  const double rteosq = sqrt(omeosq);
  double sinio, cosio;
  sincos(inclo, &sinio, &cosio);
  const double cosio2 = cosio * cosio;

  // un-Kozai  :187-193
  const double ak = pow2o3(xke / no_safe);
  const double d1 = 0.75 * j2 * (3.0 * cosio2 - 1.0) / (rteosq * omeosq);
  double del = d1 / (ak * ak);
  const double adel = ak * (1.0 - del * del - del * (1.0 / 3.0 + 134.0 * del * del / 81.0));
  del = d1 / (adel * adel);
  const double no_unkozai = no_safe / (1.0 + del);
  const bool deep_space = kTwoPi / no_unkozai >= 225.0;             // :195

  const double ao = pow2o3(xke / no_unkozai);
  const double po = ao * omeosq;
  const double con42 = 1.0 - 5.0 * cosio2;
  const double con41 = -con42 - cosio2 - cosio2;
  const double posq = gmax(po * po, tiny);
  const double rp = ao * (1.0 - ecco);
  const bool isimp = rp < 220.0 / re + 1.0;                        // :205
  const double perige = (rp - 1.0) * re;

  // s* and (q0-s)^4 by perigee  :209-221
  const double ss = 78.0 / re + 1.0;
  const double q2 = (120.0 - 78.0) / re;
  const double qzms2t = (q2 * q2) * (q2 * q2);
  const bool low_perige = perige < 156.0;
  const double sfour_low = perige < 98.0 ? 20.0 : perige - 78.0;
  const double qzms24temp = (120.0 - sfour_low) / re;
  const double qz2 = qzms24temp * qzms24temp;
  const double qzms24 = low_perige ? qz2 * qz2 : qzms2t;
  const double sfour = low_perige ? sfour_low / re + 1.0 : ss;

  // drag coefficients and secular rates  :223-275
  const double pinvsq = 1.0 / posq;
  double denom_tsi = ao - sfour;
  denom_tsi = denom_tsi == 0.0 ? tiny : denom_tsi;
  const double tsi = 1.0 / denom_tsi;
  const double eta = ao * ecco * tsi;
  const double etasq = eta * eta;
  const double eeta = ecco * eta;
  const double psisq = gmax(fabs(1.0 - etasq), tiny);
  const double tsi2 = tsi * tsi;
  const double coef = qzms24 * (tsi2 * tsi2);
  const double coef1 = coef / (psisq * psisq * psisq * sqrt(psisq));      // psisq^3.5
  const double cc2 = coef1 * no_unkozai *
      (ao * (1.0 + 1.5 * etasq + eeta * (4.0 + etasq)) +
       0.375 * j2 * tsi / psisq * con41 * (8.0 + 3.0 * etasq * (8.0 + etasq)));
  const double cc1 = bstar * cc2;
  const bool ecc_small = ecco <= 1.0e-4;
  const double ecco_guard = gmax(ecco, 1.0e-4);
  const double cc3 = ecc_small ? 0.0 * ecco
                               : -2.0 * coef * tsi * j3oj2 * no_unkozai * sinio / ecco_guard;
  const double x1mth2 = 1.0 - cosio2;
  double sinargp, cosargp;
  sincos(argpo, &sinargp, &cosargp);
  const double cc4 = 2.0 * no_unkozai * coef1 * ao * omeosq *
      (eta * (2.0 + 0.5 * etasq) + ecco * (0.5 + 2.0 * etasq) -
       j2 * tsi / (ao * psisq) *
           (-3.0 * con41 * (1.0 - 2.0 * eeta + etasq * (1.5 - 0.5 * eeta)) +
            0.75 * x1mth2 * (2.0 * etasq - eeta * (1.0 + etasq)) *
                (cosargp - sinargp) * (cosargp + sinargp)));     // cos(2 argpo)
  const double cc5 = 2.0 * coef1 * ao * omeosq * (1.0 + 2.75 * (etasq + eeta) + eeta * etasq);
  const double cosio4 = cosio2 * cosio2;
  const double temp1 = 1.5 * j2 * pinvsq * no_unkozai;
  const double temp2 = 0.5 * temp1 * j2 * pinvsq;
  const double temp3 = -0.46875 * j4 * pinvsq * pinvsq * no_unkozai;
  const double mdot = no_unkozai + 0.5 * temp1 * rteosq * con41 +
                      0.0625 * temp2 * rteosq * (13.0 - 78.0 * cosio2 + 137.0 * cosio4);
  const double argpdot = -0.5 * temp1 * con42 +
                         0.0625 * temp2 * (7.0 - 114.0 * cosio2 + 395.0 * cosio4) +
                         temp3 * (3.0 - 36.0 * cosio2 + 49.0 * cosio4);
  const double xhdot1 = -temp1 * cosio;
  const double nodedot = xhdot1 + (0.5 * temp2 * (4.0 - 19.0 * cosio2) +
                                   2.0 * temp3 * (3.0 - 7.0 * cosio2)) * cosio;
  const double omgcof = bstar * cc3 * cosargp;
  const double eeta_guard = fabs(eeta) < tiny ? tiny : eeta;
  const double xmcof = ecc_small ? 0.0 * ecco : -kX2o3 * coef * bstar / eeta_guard;
  const double nodecf = 3.5 * omeosq * xhdot1 * cc1;
  const double t2cof = 1.5 * cc1;
  const double xlcof_den = fabs(cosio + 1.0) > 1.5e-12 ? 1.0 + cosio : 1.5e-12;
  const double xlcof = -0.25 * j3oj2 * sinio * (3.0 + 5.0 * cosio) / xlcof_den;
  const double aycof = -0.5 * j3oj2 * sinio;
  double sinmao, cosmo;
  sincos(mo, &sinmao, &cosmo);
  const double delmotemp = 1.0 + eta * cosmo;
  const double delmo = delmotemp * delmotemp * delmotemp;
  const double x7thm1 = 7.0 * cosio2 - 1.0;

  // higher-order drag, zero in simplified mode  :278-294
  const double cc1sq = cc1 * cc1;
  double d2 = 4.0 * ao * tsi * cc1sq;
  const double temp_d = d2 * tsi * cc1 / 3.0;
  double d3 = (17.0 * ao + sfour) * temp_d;
  double d4 = 0.5 * temp_d * ao * tsi * (221.0 * ao + 31.0 * sfour) * cc1;
  double t3cof = d2 + 2.0 * cc1sq;
  double t4cof = 0.25 * (3.0 * d3 + cc1 * (12.0 * d2 + 10.0 * cc1sq));
  double t5cof = 0.2 * (3.0 * d4 + 12.0 * cc1 * d3 + 6.0 * d2 * d2 + 15.0 * cc1sq * (2.0 * d2 + cc1sq));
  if (isimp) {
    const double z = 0.0 * cc1;
    d2 = z; d3 = z; d4 = z; t3cof = z; t4cof = z; t5cof = z;
  }

  f[F_NO_KOZAI] = no_kozai; f[F_ECCO] = ecco; f[F_INCLO] = inclo; f[F_NODEO] = nodeo;
  f[F_ARGPO] = argpo; f[F_MO] = mo; f[F_BSTAR] = bstar;
  f[F_NO_UNKOZAI] = no_unkozai; f[F_AO] = ao; f[F_CON41] = con41; f[F_X1MTH2] = x1mth2;
  f[F_X7THM1] = x7thm1; f[F_MDOT] = mdot; f[F_ARGPDOT] = argpdot; f[F_NODEDOT] = nodedot;
  f[F_NODECF] = nodecf; f[F_CC1] = cc1; f[F_CC4] = cc4; f[F_CC5] = cc5;
  f[F_D2] = d2; f[F_D3] = d3; f[F_D4] = d4; f[F_T2COF] = t2cof; f[F_T3COF] = t3cof;
  f[F_T4COF] = t4cof; f[F_T5COF] = t5cof; f[F_ETA] = eta; f[F_OMGCOF] = omgcof;
  f[F_XMCOF] = xmcof; f[F_DELMO] = delmo; f[F_SINMAO] = sinmao; f[F_AYCOF] = aycof;
  f[F_XLCOF] = xlcof;

  // _first_error 2 > 1 > 7  :296-300
  code = bad_n ? 2 : bad_e ? 1 : deep_space ? 7 : 0;
  isimp_out = isimp;

  // record values for the propagate kernels, reusing ao and sin/cos inclo
  const double ao_sc[3] = {ao, sinio, cosio};
  record_values(f, g, v, ao_sc);
  // epoch evaluation  :316-322
  if (code == 0 && !epoch_clear(f, ao, g)) code = epoch_code(f, ao, g);
}

// One warp per block (the fp64 chains are long and latency-bound: spreading
// satellites over every SM shortens the kernel).  The packed records (AoS,
// 160/320 B per satellite) are staged in shared memory (odd stride: no bank
// conflicts) and written by the warp as consecutive words, i.e. coalesced,
// instead of 40 stores per lane strided by a whole record.
constexpr int kStageStride = S_COUNT + 1;

template <typename T>
__device__ __forceinline__ void write_records(const double* f, const double* v, int flags,
                                              bool simp, const Grav& g, bool valid,
                                              int64_t i0, int64_t n, T* __restrict__ rec,
                                              unsigned char* stage) {
  const int lane = threadIdx.x & 31;
  T* st = reinterpret_cast<T*>(stage);
  if (valid) store_record<T>(f, v, flags, simp, g, st + lane * kStageStride);
  __syncwarp();
  T* dst = rec + i0 * S_COUNT;
  const int words = (int)(min((int64_t)32, n - i0) * S_COUNT);
  for (int k = lane; k < words; k += 32) {
    const int r = k / S_COUNT;
    dst[k] = st[r * kStageStride + (k - r * S_COUNT)];
  }
}

__global__ void __launch_bounds__(32) init_kernel(
    const double* __restrict__ el, int64_t n, Grav g, double* __restrict__ satrec,
    int32_t* __restrict__ codes, uint8_t* __restrict__ isimp, void* __restrict__ rec,
    int precision) {
  __shared__ __align__(16) unsigned char stage[32 * kStageStride * sizeof(double)];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int64_t i = i0 + threadIdx.x;
  const bool valid = i < n;
  double f[F_COUNT], v[S_COUNT];
  int code = 0;
  bool simp = false;
  if (valid) {
    double e[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) e[k] = el[k * n + i];
    init_one(e, g, f, v, code, simp);
    if (satrec != nullptr) {
#pragma unroll
      for (int k = 0; k < F_COUNT; ++k) satrec[k * n + i] = f[k];
    }
    codes[i] = code;
    isimp[i] = simp ? 1 : 0;
  }
  if (rec != nullptr) {
    const int flags = valid ? record_flags(f, code, simp) : 0;
    if (precision == 64)
      write_records<double>(f, v, flags, simp, g, valid, i0, n, static_cast<double*>(rec), stage);
    else
      write_records<float>(f, v, flags, simp, g, valid, i0, n, static_cast<float*>(rec), stage);
  }
}

__global__ void pack_kernel(const double* __restrict__ satrec, const int32_t* __restrict__ codes,
                            const uint8_t* __restrict__ isimp, int64_t n, Grav g,
                            void* __restrict__ rec, int precision) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double f[F_COUNT];
#pragma unroll
  for (int k = 0; k < F_COUNT; ++k) f[k] = satrec[k * n + i];
  double v[S_COUNT];
  record_values(f, g, v);
  const bool simp = isimp[i] != 0;
  const int flags = record_flags(f, codes[i], simp);
  if (precision == 64)
    store_record<double>(f, v, flags, simp, g, static_cast<double*>(rec) + i * S_COUNT);
  else
    store_record<float>(f, v, flags, simp, g, static_cast<float*>(rec) + i * S_COUNT);
}

// ======================================================================
// Propagate: dense grid
// ======================================================================
#ifndef SGP4B_CELLS
#define SGP4B_CELLS 4
#endif
#ifndef SGP4B_MINB
#define SGP4B_MINB 1
#endif
constexpr int kCellsPerLane = SGP4B_CELLS;          // consecutive time steps per lane
constexpr int kCellsPerWarp = 32 * kCellsPerLane;   // one work item (chunk)
#ifndef SGP4B_BLOCK
#define SGP4B_BLOCK 512     // one 16-warp block per SM: its warps own adjacent rows
#endif
constexpr int kGridBlock = SGP4B_BLOCK;
#ifndef SGP4B_BLOCK64
#define SGP4B_BLOCK64 SGP4B_BLOCK
#endif
template <typename T>
__host__ __device__ constexpr int grid_block() { return sizeof(T) == 4 ? SGP4B_BLOCK : SGP4B_BLOCK64; }
constexpr int kGridMinBlocks = SGP4B_MINB;   // resident blocks per SM (fp32)


// vector streaming stores / read-only loads of N consecutive elements
template <int N>
__device__ __forceinline__ void st_vec_cs(float* p, const float (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 4)
      __stcs(reinterpret_cast<float4*>(p + k), make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]));
  } else if constexpr (N == 2) __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  else for (int k = 0; k < N; ++k) __stcs(p + k, v[k]);
}
template <int N>
__device__ __forceinline__ void st_vec_cs(int32_t* p, const int (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 4)
      __stcs(reinterpret_cast<int4*>(p + k), make_int4(v[k], v[k + 1], v[k + 2], v[k + 3]));
  } else if constexpr (N == 2) __stcs(reinterpret_cast<int2*>(p), make_int2(v[0], v[1]));
  else for (int k = 0; k < N; ++k) __stcs(reinterpret_cast<int*>(p) + k, v[k]);
}
template <int N>
__device__ __forceinline__ void st_vec_cs(double* p, const double (&v)[N]) {
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2)
    __stcs(reinterpret_cast<double2*>(p + k), make_double2(v[k], v[k + 1]));
  if constexpr (N % 2) __stcs(p + N - 1, v[N - 1]);
}
template <int N>
__device__ __forceinline__ void ld_vec(const float* p, float (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 4) {
      float4 q = __ldg(reinterpret_cast<const float4*>(p + k));
      v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
    }
  } else if constexpr (N == 2) {
    float2 q = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else {
    for (int k = 0; k < N; ++k) v[k] = __ldg(p + k);
  }
}
template <int N>
__device__ __forceinline__ void ld_vec(const double* p, double (&v)[N]) {
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    double2 q = __ldg(reinterpret_cast<const double2*>(p + k));
    v[k] = q.x; v[k + 1] = q.y;
  }
  if constexpr (N % 2) v[N - 1] = __ldg(p + N - 1);
}

#ifndef SGP4B_VEC
#define SGP4B_VEC 4
#endif
#ifndef SGP4B_ROW32
#define SGP4B_ROW32 1
#endif
#ifndef SGP4B_UNIFORM_W
#define SGP4B_UNIFORM_W 1
#endif
#ifndef SGP4B_ROWPTR
#define SGP4B_ROWPTR 1
#endif
#ifndef SGP4B_F64_K2
#define SGP4B_F64_K2 1            // fp64 class-2 fast cell (cell64_c1<..., K2 = true>)
#endif
#ifndef SGP4B_REC64_REGS
#define SGP4B_REC64_REGS 0
#endif
// longest row the kernels index with 32-bit column offsets
constexpr int64_t kMaxSteps = (int64_t)1 << 30;
constexpr int kVec = SGP4B_VEC;     // cells advanced in lockstep (2 = one packed pair)
static_assert(kCellsPerLane % kVec == 0 && kVec % 2 == 0, "fp32 cells run in packed pairs");

template <bool ISIMP, int KITER, bool LO, class RT>
__device__ __forceinline__ void compute_n(const RT& R, const float (&th)[kCellsPerLane],
                                          const float (&tl)[kCellsPerLane], const Grav& g,
                                          float (&out)[6][kCellsPerLane], int (&code)[kCellsPerLane]) {
#pragma unroll
  for (int k = 0; k < kCellsPerLane; k += kVec) {
    VN<kVec> tv, tlv, o[6];
    int cv[kVec];
#pragma unroll
    for (int i = 0; i < kVec / 2; ++i) {
      tv.h[i] = make_float2(th[k + 2 * i], th[k + 2 * i + 1]);
      tlv.h[i] = make_float2(tl[k + 2 * i], tl[k + 2 * i + 1]);
    }
    cellv<ISIMP, KITER, LO, kVec>(R, tv, tlv, g, o, cv);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
#pragma unroll
      for (int p = 0; p < 6; ++p) out[p][k + j] = comp(o[p], j);
      code[k + j] = cv[j];
    }
  }
}

// One satellite row, chunks [c0, c1): per lane kCellsPerLane consecutive
// steps per chunk.  CellsFn(th, tl, out, code) evaluates a lane's cells;
// it is specialised per satellite class, so the chunk loop is branch-free.
// MASKED: store only the cells with |t| > t_crit (the general instance's
// second pass over a row, see dispatch_row).
template <typename T, bool VEC, bool LO, bool MASKED, class CellsFn>
__device__ __forceinline__ void row_loop(const CellsFn& cells, int64_t c0, int64_t c1, int lane,
                                         const T* __restrict__ times,
                                         const float* __restrict__ times_lo, int64_t m,
                                         T* __restrict__ row, int64_t plane_stride,
                                         int32_t* __restrict__ crow, float t_crit) {
  // column indices: 32-bit (the ABI rejects m > kMaxSteps), so bounds tests
  // and increments are single ALU ops
  using J = typename std::conditional<SGP4B_ROW32 != 0, unsigned, int64_t>::type;
  const J mj = (J)m;
  // a lane's kCellsPerLane times at column j (zero past the row end)
  auto load_times = [&](J j, T (&th)[kCellsPerLane], float (&tl)[kCellsPerLane]) {
    if (VEC && j + kCellsPerLane <= mj) {
      ld_vec<kCellsPerLane>(times + j, th);
    } else {
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) th[k] = j + k < mj ? __ldg(times + j + k) : T(0);
    }
#pragma unroll
    for (int k = 0; k < kCellsPerLane; ++k) tl[k] = (LO && j + k < mj) ? __ldg(times_lo + j + k) : 0.0f;
  };
  J j0 = (J)(c0 * kCellsPerWarp) + (J)(lane * kCellsPerLane);
  T th[kCellsPerLane];
  float tl[kCellsPerLane];
  load_times(j0, th, tl);
#if SGP4B_ROWPTR
  // per-plane row bases (warp-uniform); a store address is base + j0
  T* rp[6];
#pragma unroll
  for (int p = 0; p < 6; ++p) rp[p] = row + p * plane_stride;
#define SGP4B_PADDR(p, k) (rp[p] + (j0 + (k)))
#define SGP4B_CADDR(k) (crow + (j0 + (k)))
#else
  T* pb = row + j0;                          // output pointers walk the row
  int32_t* cb = crow + j0;
#define SGP4B_PADDR(p, k) (pb + (p) * plane_stride + (k))
#define SGP4B_CADDR(k) (cb + (k))
#endif
  const J jc1 = (J)(c1 * kCellsPerWarp);
  for (J jc = (J)(c0 * kCellsPerWarp); jc < jc1; jc += kCellsPerWarp, j0 += kCellsPerWarp) {
#if SGP4B_SHFL_REC
    // keep the warp converged (record fields are shuffled): lanes past the
    // row end compute a dummy cell and skip the stores
    if (__all_sync(0xffffffffu, j0 >= mj)) break;
#else
    if (j0 >= mj) break;                    // only the row's last chunk is partial
#endif
    const bool full = VEC && j0 + kCellsPerLane <= mj;
    // the next chunk's times are loaded before this chunk's cells run, so
    // their latency hides behind the cell math
    T thn[kCellsPerLane];
    float tln[kCellsPerLane];
    load_times(j0 + kCellsPerWarp, thn, tln);

    T out[6][kCellsPerLane];
    int code[kCellsPerLane];
    cells(th, tl, out, code);
    if constexpr (MASKED) {
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) {
        if (fabsf((float)th[k]) > t_crit && j0 + k < mj) {
#pragma unroll
          for (int p = 0; p < 6; ++p) st_cs(SGP4B_PADDR(p, k), out[p][k]);
          st_cs(SGP4B_CADDR(k), code[k]);
        }
      }
#if !SGP4B_ROWPTR
      pb += kCellsPerWarp;
      cb += kCellsPerWarp;
#endif
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) {
        th[k] = thn[k];
        tl[k] = tln[k];
      }
      continue;
    }
#ifdef SGP4B_NOSTORE
    // analysis build: compute-only timing (results kept alive, never stored)
    {
      T acc = T(0);
      int ca = 0;
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) {
#pragma unroll
        for (int p = 0; p < 6; ++p) acc += out[p][k];
        ca |= code[k];
      }
      if (acc == T(1.2345e-30) && ca == 77) st_cs(row + j0, acc);
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) {
        th[k] = thn[k];
        tl[k] = tln[k];
      }
      continue;
    }
#endif

#if !SGP4B_ROWPTR
    T* base = pb;
    int32_t* cbase = cb;
    pb += kCellsPerWarp;
    cb += kCellsPerWarp;
#endif
    if (full) {
#pragma unroll
#if SGP4B_ROWPTR
      for (int p = 0; p < 6; ++p) st_vec_cs<kCellsPerLane>(rp[p] + j0, out[p]);
      st_vec_cs<kCellsPerLane>(crow + j0, code);
#else
      for (int p = 0; p < 6; ++p) st_vec_cs<kCellsPerLane>(base + p * plane_stride, out[p]);
      st_vec_cs<kCellsPerLane>(cbase, code);
#endif
    } else {
#pragma unroll
      for (int k = 0; k < kCellsPerLane; ++k) {
        if (j0 + k < mj) {
#pragma unroll
#if SGP4B_ROWPTR
          for (int p = 0; p < 6; ++p) st_cs(rp[p] + (j0 + k), out[p][k]);
          st_cs(crow + (j0 + k), code[k]);
#else
          for (int p = 0; p < 6; ++p) st_cs(base + p * plane_stride + k, out[p][k]);
          st_cs(cbase + k, code[k]);
#endif
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kCellsPerLane; ++k) {
      th[k] = thn[k];
      tl[k] = tln[k];
    }
  }
}

template <bool ISIMP, int KITER, bool VEC, bool LO, bool MASKED = false, class RT>
__device__ __forceinline__ void row32(const RT& R, const Grav& g, int64_t c0, int64_t c1,
                                      int lane, const float* times, const float* times_lo,
                                      int64_t m, float* row, int64_t plane_stride, int32_t* crow,
                                      float t_crit) {
  auto cells = [&](const float (&th)[kCellsPerLane], const float (&tl)[kCellsPerLane],
                   float (&out)[6][kCellsPerLane], int (&code)[kCellsPerLane]) {
    compute_n<ISIMP, KITER, LO>(R, th, tl, g, out, code);
  };
  row_loop<float, VEC, LO, MASKED>(cells, c0, c1, lane, times, times_lo, m, row, plane_stride,
                                   crow, t_crit);
}

// The masked general pass over one row, out of line (rarely executed; kept
// out of the class passes' register allocation): reloads the record.
template <bool ISIMP, bool VEC, bool LO>
__device__ __noinline__ void fixup_row(const float* recg, float re_f, float vkm_f, int64_t c0,
                                       int64_t c1, int lane, const float* times,
                                       const float* times_lo, int64_t m, float* row, int64_t ps,
                                       int32_t* crow, float t_crit) {
  Rec<float> R;
  load_rec(recg, R);
  Grav g{};
  g.re_f = re_f;
  g.vkm_f = vkm_f;
  row32<ISIMP, 0, VEC, LO, true>(R, g, c0, c1, lane, times, times_lo, m, row, ps, crow, t_crit);
}

// Per-row dispatch on the satellite's (isimp, Kepler class): warp-uniform.
// The class was chosen from ecco at init (kepler_iters_for); it stays valid
// while |em| = |ecco + bc5 sinmao - bc4 t - bc5 sin mm| is below the class
// bound, which holds for |t| <= t_crit = (bound - |E0| - 2 |bc5|) / |bc4|.
// t_absmax (launch argument) bounds |t| over the launch; when it exceeds a
// row's t_crit (long or backward spans of high-drag objects) the cells
// beyond t_crit are recomputed by the general instance in a second, masked
// pass over the row, so every cell's value is a function of its own
// (satellite, t) only (batch == scalar).
template <bool VEC, bool LO, class RT>
__device__ __forceinline__ void dispatch_row(const RT& R, const float* recg, const Grav& g,
                                             int64_t c0, int64_t c1, int lane, const float* times,
                                             const float* times_lo, int64_t m, float* row,
                                             int64_t ps, int32_t* crow, float t_absmax) {
#ifdef SGP4B_ONLY_CLASS_K1
  // analysis build: every row runs the (non-isimp, Kepler SGP4B_ONLY_CLASS_K1)
  // instance, so the SASS holds one chunk loop (static instruction mix)
  row32<false, SGP4B_ONLY_CLASS_K1, VEC, LO>(R, g, c0, c1, lane, times, times_lo, m, row, ps, crow,
                                             INFINITY);
  return;
#endif
  const int flags = R.flags();
  const int kit = (flags >> KEPLER_SHIFT) & 0xf;
  const bool simp = flags & FLAG_ISIMP;
  auto t_crit_of = [&](const auto& rec) {
    const float bound = kit == 1 ? 0.004f : kit == 2 ? 0.1f : 0.4f;
    const float slack = bound - fabsf(rec[P_E0]) - 2.0f * fabsf(rec[P_BC5]);
    return slack > 0.0f ? slack / fabsf(rec[P_BC4]) : -1.0f;
  };
  // NaN t_absmax (unknown bound) counts as unbounded
  const bool need = kit >= 1 && kit <= 3 && !(t_absmax <= t_crit_of(R));
#define SGP4B_ROW(S, K) row32<S, K, VEC, LO>(R, g, c0, c1, lane, times, times_lo, m, row, ps, crow, INFINITY)
  if (!simp) {
    if (kit == 1) SGP4B_ROW(false, 1);
    else if (kit == 2) SGP4B_ROW(false, 2);
    else if (kit == 3) SGP4B_ROW(false, 3);
    else SGP4B_ROW(false, 0);
  } else {
    if (kit == 1) SGP4B_ROW(true, 1);
    else if (kit == 2) SGP4B_ROW(true, 2);
    else if (kit == 3) SGP4B_ROW(true, 3);
    else SGP4B_ROW(true, 0);
  }
#undef SGP4B_ROW
  if (need) {
    const float t_crit = t_crit_of(R);
    if (!simp)
      fixup_row<false, VEC, LO>(recg, g.re_f, g.vkm_f, c0, c1, lane, times, times_lo, m, row, ps,
                                crow, t_crit);
    else
      fixup_row<true, VEC, LO>(recg, g.re_f, g.vkm_f, c0, c1, lane, times, times_lo, m, row, ps,
                               crow, t_crit);
  }
}

// fp64 row: lane l owns columns j0 + l + 32 k of each 128-column chunk, so
// every cell is stored with fully coalesced 8-byte (4-byte code) streaming
// stores straight from registers — no per-lane output buffer.  kIlp64 cells
// (j, j + 32, ...) are evaluated per iteration: independent dependency
// chains for the scheduler, and each record word read from shared memory
// serves all of them.  FAST rows (Kepler class 1 by the record's ecco) run
// cell64_c1 and hand a cell that leaves the class-1 domain to the
// out-of-line general cell; other rows run the general cell.
#ifndef SGP4B_F64_ILP
#define SGP4B_F64_ILP 1
#endif
constexpr int kIlp64 = SGP4B_F64_ILP;

template <bool FAST, bool ISIMP, class RT, bool K2 = false>
__device__ __forceinline__ void row64(const RT& R, const double* recp, const TrigGrid& tr, double re,
                                      double vkm, int64_t c0, int64_t c1, int lane,
                                      const double* __restrict__ times, int64_t m,
                                      double* __restrict__ row, int64_t ps,
                                      int32_t* __restrict__ crow) {
  // column indices are 32-bit (m < 2^31): one IMAD.WIDE per store address
  // off the per-row plane bases
  const unsigned jend = (unsigned)min(c1 * kCellsPerWarp, m);
  double* const p0 = row;
  double* const p1 = row + ps;
  double* const p2 = row + 2 * ps;
  double* const p3 = row + 3 * ps;
  double* const p4 = row + 4 * ps;
  double* const p5 = row + 5 * ps;
#pragma unroll 1
  for (unsigned j = (unsigned)(c0 * kCellsPerWarp) + lane; j < jend; j += 32 * kIlp64) {
    double t[kIlp64];
#pragma unroll
    for (int i = 0; i < kIlp64; ++i) t[i] = j + 32 * i < jend ? __ldg(times + j + 32 * i) : 0.0;
    Cell64 o[kIlp64];
    bool ok[kIlp64];
#pragma unroll
    for (int i = 0; i < kIlp64; ++i) {
      if constexpr (FAST) {
        ok[i] = cell64_c1<ISIMP, RT, TrigGrid, K2>(R, t[i], re, dbits(re), vkm, tr, o[i]);
      } else {
        cell64_general(R, t[i], re, vkm, tr, o[i]);
        ok[i] = true;
      }
    }
#pragma unroll
    for (int i = 0; i < kIlp64; ++i) {
      const unsigned jj = j + 32 * i;
      if (jj >= jend) break;
      if (!ok[i]) {
        cell64_fallback(recp, t[i], re, vkm, tr.tab, row + jj, ps, crow + jj);
        continue;
      }
#ifndef SGP4B_NOSTORE
      st_cs(p0 + jj, o[i].r[0]);
      st_cs(p1 + jj, o[i].r[1]);
      st_cs(p2 + jj, o[i].r[2]);
      st_cs(p3 + jj, o[i].v[0]);
      st_cs(p4 + jj, o[i].v[1]);
      st_cs(p5 + jj, o[i].v[2]);
      st_cs(crow + jj, o[i].code);
#else
      if (o[i].r[0] + o[i].r[1] + o[i].v[2] == 1.2345e-300 && o[i].code == 77) st_cs(row + jj, o[i].r[0]);
#endif
    }
  }
}

template <class RT>
__device__ __forceinline__ void dispatch_row64(const RT& R, const double* recp, const TrigGrid& tr,
                                               const Grav& g, int64_t c0, int64_t c1, int lane,
                                               const double* times, int64_t m, double* row,
                                               int64_t ps, int32_t* crow) {
  const int flags = R.flags();
  const int kit = (flags >> KEPLER_SHIFT) & 0xf;
  if (kit == 1) {
    if (flags & FLAG_ISIMP)
      row64<true, true>(R, recp, tr, g.re, g.vkm, c0, c1, lane, times, m, row, ps, crow);
    else
      row64<true, false>(R, recp, tr, g.re, g.vkm, c0, c1, lane, times, m, row, ps, crow);
  } else if (kit == 2 && SGP4B_F64_K2) {
    if (flags & FLAG_ISIMP)
      row64<true, true, RT, true>(R, recp, tr, g.re, g.vkm, c0, c1, lane, times, m, row, ps, crow);
    else
      row64<true, false, RT, true>(R, recp, tr, g.re, g.vkm, c0, c1, lane, times, m, row, ps, crow);
  } else {
    row64<false, false>(R, recp, tr, g.re, g.vkm, c0, c1, lane, times, m, row, ps, crow);
  }
}

// Persistent warps: the (satellite, chunk) work items of the grid are split
// into one contiguous range per resident warp; the warp walks it row by row,
// loading each satellite's record once and dispatching its class once.


//
// With rec_idx set, row r uses record rec_idx[r] and times + r*times_ld:
// (satellite, time) pairs as P rows of one step.  The elementwise API uses
// this only when built with SGP4B_PAIRS_LANE=0 (pairs_kernel32/64 run one
// lane per pair).  The Python layer pads unaligned grids so every public
// call runs the VEC instance; VEC = false only serves raw C-ABI callers with
// unaligned strides.
#ifdef SGP4B_TIMELINE
// analysis build: per-warp (start, first row done, end, smid) in ns
constexpr int kTimelineWarps = 1 << 16;
__device__ unsigned long long g_timeline[kTimelineWarps][4];
#endif

template <typename T, bool VEC, bool LO>
__global__ void __launch_bounds__(grid_block<T>(), sizeof(T) == 4 ? kGridMinBlocks : kGridMinBlocks64)
grid_kernel(const T* __restrict__ rec, const int64_t* __restrict__ rec_idx, int64_t n,
            const T* __restrict__ times, const float* __restrict__ times_lo, int64_t times_ld,
            int64_t m, Grav g, T* __restrict__ planes, int64_t plane_stride, int64_t row_stride,
            int32_t* __restrict__ codes, int64_t code_stride, int64_t chunks, float t_absmax) {
  constexpr int kBlock = grid_block<T>();
  const int64_t nwarps = (int64_t)gridDim.x * (kBlock / 32);
#if SGP4B_UNIFORM_W
  // the warp index through a lane-0 shuffle: the compiler then knows it (and
  // every row/chunk bound and row base pointer derived from it) is
  // warp-uniform and can keep them in uniform registers
  const int64_t w = (int64_t)blockIdx.x * (kBlock / 32) +
                    __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
#else
  const int64_t w = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
#endif
  const int lane = threadIdx.x & 31;
  const int64_t total = n * chunks;
  const int64_t g0 = total * w / nwarps;
  const int64_t g1 = total * (w + 1) / nwarps;

  // fp64: records in shared memory unless SGP4B_REC64_REGS
  constexpr bool kSmem = sizeof(T) == 8 ? !SGP4B_REC64_REGS : SGP4B_SMEM_REC;
  constexpr bool kShfl = sizeof(T) == 4 && SGP4B_SHFL_REC;
  __shared__ __align__(16) T srec[kSmem ? kBlock / 32 : 1][S_COUNT];
  T* my = srec[kSmem ? (threadIdx.x >> 5) : 0];
  // fp64: the (sin, cos)(2 pi i / 512) table of TrigTab, built per block
  __shared__ double2 sintab[sizeof(T) == 8 ? kTabN : 1];
  if constexpr (sizeof(T) == 8) {
    for (int i = threadIdx.x; i < kTabN; i += kBlock) {
      double sv, cv;
      sincospi((double)i / (kTabN / 2), &sv, &cv);
      sintab[i] = make_double2(sv, cv);
    }
    __syncthreads();
  }
  using RecT = typename std::conditional<
      kShfl, RecW, typename std::conditional<kSmem, RecS<T>, Rec<T>>::type>::type;
  RecT R;
  if constexpr (kSmem && !kShfl) R.p = my;
  if (g0 < g1) {
    // the first chunk's times travel with the first record load
    const int64_t s0 = g0 / chunks;
    const int64_t jf = (g0 - s0 * chunks) * kCellsPerWarp + lane * kCellsPerLane;
    if (jf < m) asm volatile("prefetch.global.L1 [%0];" ::"l"(times + s0 * times_ld + jf));
  }
#ifdef SGP4B_TIMELINE
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  bool first_row = true;
#endif
  for (int64_t gi = g0; gi < g1;) {
    const int64_t sat = gi / chunks;
    const int64_t c0 = gi - sat * chunks;
    const int64_t c1 = (g1 - gi < chunks - c0) ? c0 + (g1 - gi) : chunks;
    const int64_t ri = rec_idx != nullptr ? __ldg(rec_idx + sat) : sat;
    if constexpr (kShfl) {
      const T* src = rec + ri * S_COUNT;
      R.lo = __ldg(src + lane);
      R.hi = lane + 32 < S_COUNT ? __ldg(src + 32 + lane) : 0.0f;
    } else if constexpr (kSmem) {
      __syncwarp();
      for (int i = lane; i < S_COUNT; i += 32) my[i] = __ldg(rec + ri * S_COUNT + i);
      __syncwarp();
    } else {
      load_rec(rec + ri * S_COUNT, R);
    }
    // pull the next row's record toward L1 while this row computes
    if (rec_idx == nullptr && gi + (c1 - c0) < g1 && lane < (int)(S_COUNT * sizeof(T) + 127) / 128)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(rec + (ri + 1) * S_COUNT + lane * (128 / sizeof(T))));
    if constexpr (sizeof(T) == 8) {
      const double* recp;
      if constexpr (kSmem) recp = reinterpret_cast<const double*>(my);
      else recp = reinterpret_cast<const double*>(rec) + ri * S_COUNT;
      dispatch_row64(R, recp, TrigGrid{sintab}, g, c0, c1, lane, times + sat * times_ld, m,
                     planes + sat * row_stride, plane_stride, codes + sat * code_stride);
    } else {
      dispatch_row<VEC, LO>(R, reinterpret_cast<const float*>(rec) + ri * S_COUNT, g, c0, c1,
                            lane, times + sat * times_ld,
                            LO ? times_lo + sat * times_ld : nullptr, m, planes + sat * row_stride,
                            plane_stride, codes + sat * code_stride, t_absmax);
    }
    gi += c1 - c0;
#ifdef SGP4B_TIMELINE
    if (first_row && lane == 0 && w < kTimelineWarps) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_timeline[w][1] = t;
    }
    first_row = false;
#endif
  }
#ifdef SGP4B_TIMELINE
  if (lane == 0 && w < kTimelineWarps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_timeline[w][0] = t_start;
    g_timeline[w][2] = t;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_timeline[w][3] = smid;
  }
#endif
}

// Elementwise pairs (scalar / broadcasting API), fp32: one lane per
// (satellite, time) pair.  A pair runs the same cellv instance a grid row of
// its satellite runs (chosen by the same (isimp, Kepler class) rule and the
// same t_crit / t_absmax test as dispatch_row + fixup_row), with both halves
// of the packed pair set to its time.  Every mul/add/fma of cellv is an
// explicit IEEE-rounded op and every SFU/select is per component, so the
// pair's value equals the grid cell's bit for bit however the record is held
// (per-lane registers here, warp-uniform registers in the grid).  Lanes of a
// warp may take different classes; each class runs once per warp.
#ifndef SGP4B_PAIRS_LANE
#define SGP4B_PAIRS_LANE 1
#endif
constexpr int kPairsBlock = 128;

template <bool LO>
__global__ void __launch_bounds__(kPairsBlock) pairs_kernel32(
    const float* __restrict__ rec, const int64_t* __restrict__ rec_idx, int64_t p,
    const float* __restrict__ times, const float* __restrict__ times_lo, Grav g,
    float* __restrict__ rv, int32_t* __restrict__ codes, float t_absmax) {
  const int64_t k = (int64_t)blockIdx.x * kPairsBlock + threadIdx.x;
  if (k >= p) return;
  const int64_t ri = __ldg(rec_idx + k);
  Rec<float> R;
  load_rec(rec + ri * S_COUNT, R);
  const float t = __ldg(times + k);
  const float tl = LO ? __ldg(times_lo + k) : 0.0f;
  const int flags = R.flags();
  int kit = (flags >> KEPLER_SHIFT) & 0xf;
  const bool simp = flags & FLAG_ISIMP;
  if (kit >= 1 && kit <= 3) {
    // dispatch_row's t_crit and its masked general pass (fixup_row)
    const float bound = kit == 1 ? 0.004f : kit == 2 ? 0.1f : 0.4f;
    const float slack = bound - fabsf(R[P_E0]) - 2.0f * fabsf(R[P_BC5]);
    const float t_crit = slack > 0.0f ? slack / fabsf(R[P_BC4]) : -1.0f;
    if (!(t_absmax <= t_crit) && fabsf(t) > t_crit) kit = 0;
  }
  // the second half is the same time through an opaque move, so the
  // compiler cannot see that the halves are equal and fold the packed pair
  // into scalar ops (whose contraction it could then choose differently):
  // the pair runs the packed instruction stream of a grid cell
  float t2, tl2;
  asm("mov.b32 %0, %1;" : "=f"(t2) : "f"(t));
  asm("mov.b32 %0, %1;" : "=f"(tl2) : "f"(tl));
  VN<2> tv, tlv, o[6];
  tv.h[0] = make_float2(t, t2);
  tlv.h[0] = make_float2(tl, tl2);
  int cv[2];
#define SGP4B_PAIR(S, K) cellv<S, K, LO, 2>(R, tv, tlv, g, o, cv)
  if (!simp) {
    if (kit == 1) SGP4B_PAIR(false, 1);
    else if (kit == 2) SGP4B_PAIR(false, 2);
    else if (kit == 3) SGP4B_PAIR(false, 3);
    else SGP4B_PAIR(false, 0);
  } else {
    if (kit == 1) SGP4B_PAIR(true, 1);
    else if (kit == 2) SGP4B_PAIR(true, 2);
    else if (kit == 3) SGP4B_PAIR(true, 3);
    else SGP4B_PAIR(true, 0);
  }
#undef SGP4B_PAIR
#pragma unroll
  for (int q = 0; q < 6; ++q) st_cs(rv + q * p + k, o[q].h[0].x);
  st_cs(codes + k, cv[0]);
}

// Elementwise pairs, fp64: one lane per pair, grid-stride over the pairs so
// each block builds the shared (sin, cos) table once.  A lane reads its
// record through RecS<double> pointed at global memory (the grid kernel's
// record type, pointed at shared memory there) and runs the cell the grid's
// dispatch_row64 picks for that record: cell64_c1 (class 1, or class 2 with
// K2) with the out-of-line general cell as its per-cell fallback, else the
// general cell.
constexpr int kPairsBlock64 = 256;

__global__ void __launch_bounds__(kPairsBlock64) pairs_kernel64(
    const double* __restrict__ rec, const int64_t* __restrict__ rec_idx, int64_t p,
    const double* __restrict__ times, Grav g, double* __restrict__ rv,
    int32_t* __restrict__ codes) {
  __shared__ double2 sintab[kTabN];
  for (int i = threadIdx.x; i < kTabN; i += kPairsBlock64) {
    double sv, cv;
    sincospi((double)i / (kTabN / 2), &sv, &cv);
    sintab[i] = make_double2(sv, cv);
  }
  __syncthreads();
  const TrigGrid tr{sintab};
  const double re = g.re, vkm = g.vkm;
  for (int64_t k = (int64_t)blockIdx.x * kPairsBlock64 + threadIdx.x; k < p;
       k += (int64_t)gridDim.x * kPairsBlock64) {
    const double* recp = rec + __ldg(rec_idx + k) * S_COUNT;
    RecS<double> R;
    R.p = recp;
    const double t = __ldg(times + k);
    const int flags = R.flags();
    const int kit = (flags >> KEPLER_SHIFT) & 0xf;
    const bool simp = flags & FLAG_ISIMP;
    Cell64 o;
    bool ok = true;
    if (kit == 1) {
      ok = simp ? cell64_c1<true, RecS<double>, TrigGrid, false>(R, t, re, dbits(re), vkm, tr, o)
                : cell64_c1<false, RecS<double>, TrigGrid, false>(R, t, re, dbits(re), vkm, tr, o);
    } else if (kit == 2 && SGP4B_F64_K2) {
      ok = simp ? cell64_c1<true, RecS<double>, TrigGrid, true>(R, t, re, dbits(re), vkm, tr, o)
                : cell64_c1<false, RecS<double>, TrigGrid, true>(R, t, re, dbits(re), vkm, tr, o);
    } else {
      cell64_general(R, t, re, vkm, tr, o);
    }
    if (!ok) {
      cell64_fallback(recp, t, re, vkm, sintab, rv + k, p, codes + k);
      continue;
    }
    st_cs(rv + k, o.r[0]);
    st_cs(rv + p + k, o.r[1]);
    st_cs(rv + 2 * p + k, o.r[2]);
    st_cs(rv + 3 * p + k, o.v[0]);
    st_cs(rv + 4 * p + k, o.v[1]);
    st_cs(rv + 5 * p + k, o.v[2]);
    st_cs(codes + k, o.code);
  }
}

template <typename T>
__global__ void kepler_kernel(const T* __restrict__ axnl, const T* __restrict__ aynl,
                              const T* __restrict__ u, int64_t n, T* __restrict__ out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = kepler_reference<T>(axnl[k], aynl[k], u[k]);
}

// |r32 - r64| and |v32 - v64| per cell in fp64 where both codes are 0,
// +inf elsewhere (so a per-column sort puts excluded cells last).
// ======================================================================
// TLE catalogue ingest (tle.py parse_catalog_columns, on the device)
// ======================================================================
// One thread per record: line 1 and line 2 start at byte offsets l1[i],
// l2[i] of the catalogue text and end at the next '\n' (trailing '\r' and
// spaces stripped, then space-padded to 69 columns, as
// s.rstrip("\r\n ").ljust(69)[:69]).  Fields are decoded exactly as the
// NumPy path does: a decimal field's value m / 10^k (m < 2^53, k <= 22) is
// one correctly rounded IEEE division, which is what numpy's correctly
// rounded string -> float64 cast returns; the implied-exponent B* field is
// float("[-]0.digits") * 10.0**e (two roundings, like the host); then the
// canonical conversion in the host's operation order.  A field outside the
// simple syntax sets a bit in status[i]; the caller re-decodes those
// records on the host, so every column equals parse_catalog_columns.
struct TleLine {
  const uint8_t* p;
  int len;                          // columns before the stripped end
  bool ascii;                       // byte columns == the host's str columns
  __device__ __forceinline__ uint8_t at(int c) const { return c < len ? p[c] : (uint8_t)' '; }
};

__device__ __forceinline__ TleLine tle_line(const uint8_t* text, int64_t size, int64_t off) {
  TleLine l;
  l.p = text + off;
  int n = 0;
  bool ascii = true;
  while (n < 80 && off + n < size && l.p[n] != '\n') {
    ascii = ascii && l.p[n] < 0x80;
    ++n;
  }
  while (n > 0 && (l.p[n - 1] == ' ' || l.p[n - 1] == '\r')) --n;
  l.len = n < 69 ? n : 69;
  l.ascii = ascii;
  return l;
}

// columns [a, b) stripped of spaces -> [s, e); false if another whitespace
// character is present (the host strip() would remove it too: host path)
__device__ __forceinline__ bool tle_strip(const TleLine& l, int a, int b, int& s, int& e) {
  s = a;
  e = b;
  while (s < e && l.at(s) == ' ') ++s;
  while (e > s && l.at(e - 1) == ' ') --e;
  for (int c = s; c < e; ++c) {
    const uint8_t ch = l.at(c);
    if (ch == '\t' || ch == '\r' || ch == '\n' || ch == '\v' || ch == '\f') return false;
  }
  return true;
}

// decimal "[+-]digits[.digits]" (at least one digit) -> correctly rounded
// double; an empty field is +0.0 (as_float maps b"" to b"0")
__device__ __forceinline__ bool tle_decimal(const TleLine& l, int a, int b, const double* pow10,
                                            double& out) {
  int s, e;
  if (!tle_strip(l, a, b, s, e)) return false;
  if (s == e) {
    out = 0.0;
    return true;
  }
  bool neg = false;
  if (l.at(s) == '+' || l.at(s) == '-') {
    neg = l.at(s) == '-';
    ++s;
  }
  unsigned long long m = 0;
  int digits = 0, frac = -1;
  for (int c = s; c < e; ++c) {
    const uint8_t ch = l.at(c);
    if (ch == '.') {
      if (frac >= 0) return false;
      frac = 0;
      continue;
    }
    if (ch < '0' || ch > '9') return false;
    m = m * 10 + (ch - '0');
    ++digits;
    if (frac >= 0) ++frac;
  }
  if (digits == 0 || digits > 15) return false;     // m < 10^15 < 2^53: exact
  const int k = frac < 0 ? 0 : frac;
  const double v = k == 0 ? (double)m : __ddiv_rn((double)m, pow10[k]);
  out = neg ? -v : v;
  return true;
}

__global__ void tle_columns_kernel(const uint8_t* __restrict__ text, int64_t size,
                                   const int64_t* __restrict__ l1, const int64_t* __restrict__ l2,
                                   int64_t n, const double* __restrict__ pow10,
                                   double* __restrict__ cols, int32_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const TleLine a = tle_line(text, size, l1[i]);
  const TleLine b = tle_line(text, size, l2[i]);
  // a multi-byte UTF-8 character shifts the host's str columns: host path
  int bad = (a.ascii && b.ascii) ? 0 : 128;
  double revday = 0, incl = 0, raan = 0, argp = 0, ma = 0, ecc = 0, bstar = 0;
  // line 2 fields (tle.py _L2)
  if (!tle_decimal(b, 52, 63, pow10, revday)) bad |= 1;
  if (!tle_decimal(b, 8, 16, pow10, incl)) bad |= 2;
  if (!tle_decimal(b, 17, 25, pow10, raan)) bad |= 4;
  if (!tle_decimal(b, 34, 42, pow10, argp)) bad |= 8;
  if (!tle_decimal(b, 43, 51, pow10, ma)) bad |= 16;
  {
    // eccentricity: "0." + zfill(digits, 7); empty -> "0"
    int s, e;
    if (!tle_strip(b, 26, 33, s, e)) {
      bad |= 32;
    } else {
      unsigned long long m = 0;
      for (int c = s; c < e; ++c) {
        const uint8_t ch = b.at(c);
        if (ch < '0' || ch > '9') bad |= 32;
        m = m * 10 + (ch - '0');
      }
      ecc = __ddiv_rn((double)m, pow10[7]);
    }
  }
  {
    // B*: "[sign]digits[sign digit]" (tle.py _implied_exponent_columns)
    int s, e;
    if (!tle_strip(a, 53, 61, s, e)) {
      bad |= 64;
    } else if (s < e) {
      const int len = e - s;
      const uint8_t first = a.at(s), last = a.at(e - 1), pen = len >= 2 ? a.at(e - 2) : 0;
      const bool neg = first == '-';
      const int start = s + ((first == '-' || first == '+') ? 1 : 0);
      const bool has_exp = len >= 2 && (pen == '-' || pen == '+') && last >= '0' && last <= '9';
      const int stop = has_exp ? e - 2 : e;
      unsigned long long m = 0;
      if (stop <= start || stop - start > 15) bad |= 64;
      for (int c = start; c < stop; ++c) {
        const uint8_t ch = a.at(c);
        if (ch < '0' || ch > '9') bad |= 64;
        m = m * 10 + (ch - '0');
      }
      if (!(bad & 64)) {
        double v = __ddiv_rn((double)m, pow10[stop - start]);
        v = neg ? -v : v;
        // 10.0**e for e = -9..9 follow the 23 exact powers (the host's values)
        if (has_exp) v = __dmul_rn(v, pow10[32 + (pen == '-' ? -(int)(last - '0') : (int)(last - '0'))]);
        bstar = v;
      }
    }
  }
  // canonical columns (tle.py parse_catalog_columns), host operation order
  const double deg = 0.017453292519943295;          // math.pi / 180.0
  cols[0 * n + i] = __ddiv_rn(__dmul_rn(revday, kTwoPi), 1440.0);
  cols[1 * n + i] = ecc;
  cols[2 * n + i] = __dmul_rn(incl, deg);
  cols[3 * n + i] = pymod_2pi(__dmul_rn(raan, deg));
  cols[4 * n + i] = pymod_2pi(__dmul_rn(argp, deg));
  cols[5 * n + i] = pymod_2pi(__dmul_rn(ma, deg));
  cols[6 * n + i] = bstar;
  status[i] = bad;
}

__global__ void drift_norms_kernel(const float* __restrict__ p32, const double* __restrict__ p64,
                                   const int32_t* __restrict__ c32, const int32_t* __restrict__ c64,
                                   int64_t cells, double* __restrict__ dr, double* __restrict__ dv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cells) return;
  if (c32[i] != 0 || c64[i] != 0) {
    dr[i] = CUDART_INF;
    dv[i] = CUDART_INF;
    return;
  }
  // np.linalg.norm(x, axis=-1) as drift.py:71-72 evaluates it: squares
  // rounded, then summed left to right (no fused multiply-add), so the
  // percentiles match a NumPy recomputation bit for bit
  double r2 = 0.0, v2 = 0.0;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const double a = (double)__ldg(p32 + p * cells + i) - __ldg(p64 + p * cells + i);
    const double b = (double)__ldg(p32 + (p + 3) * cells + i) - __ldg(p64 + (p + 3) * cells + i);
    r2 = p == 0 ? __dmul_rn(a, a) : __dadd_rn(r2, __dmul_rn(a, a));
    v2 = p == 0 ? __dmul_rn(b, b) : __dadd_rn(v2, __dmul_rn(b, b));
  }
  dr[i] = sqrt(r2);
  dv[i] = sqrt(v2);
}

// flags[i] = 1 if row i of the code plane holds a nonzero code, else 0:
// one warp per row (grid-stride), 16-byte loads when the rows are aligned.
// Lets a host copy move only the rows that carry codes (most catalogues
// have none) and zero-fill the rest itself.
__global__ void __launch_bounds__(256) code_rows_kernel(const int32_t* __restrict__ codes,
                                                        int64_t n, int64_t m, int64_t stride,
                                                        uint8_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool vec = (stride % 4 == 0) && ((uintptr_t)codes % 16 == 0);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int32_t* row = codes + r * stride;
    int any = 0;
    int64_t j = 0;
    if (vec) {
      const int64_t m4 = m & ~(int64_t)3;
      for (j = (int64_t)lane * 4; j < m4; j += 128) {
        const int4 q = __ldcs(reinterpret_cast<const int4*>(row + j));
        any |= q.x | q.y | q.z | q.w;
      }
      j = m4;
    }
    for (int64_t k = j + lane; k < m; k += 32) any |= __ldcs(row + k);
    any = __any_sync(0xffffffffu, any != 0);
    if (lane == 0) flags[r] = any ? 1 : 0;
  }
}

// Per-column nearest-rank percentiles of the drift norms (drift.py:46-49:
// rank = max(1, ceil(count * p / 100)) among the finite values of a column,
// the rank-th smallest).  One block per column; each of the six selections
// (p5/p50/p95 of |dr| and |dv|) is an MSB-first radix select over the
// values' bit patterns (non-negative doubles order as unsigned integers;
// +inf marks excluded cells and sorts after every finite value), 8 bits per
// pass.  Exact: the result is the element a full column sort would place at
// that rank.
struct Pct3 {
  double f[3];                      // p / 100.0 as the host computes it
};

__global__ void __launch_bounds__(256) drift_pct_kernel(const double* __restrict__ dr,
                                                        const double* __restrict__ dv, int64_t n,
                                                        int64_t m, Pct3 pct,
                                                        double* __restrict__ table,
                                                        int64_t* __restrict__ counts) {
  __shared__ unsigned hist[6][256];
  __shared__ unsigned long long prefix[6];
  __shared__ long long rank[6];
  __shared__ unsigned long long cnt_s[2];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x;
  // finite counts of the column (excluded cells are +inf)
  unsigned long long cr = 0, cv = 0;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    cr += isfinite(__ldg(dr + i * m + j)) ? 1 : 0;
    cv += isfinite(__ldg(dv + i * m + j)) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    cv += __shfl_xor_sync(0xffffffffu, cv, o);
  }
  if (tid < 2) cnt_s[tid] = 0;
  __syncthreads();
  if ((tid & 31) == 0) {
    atomicAdd(&cnt_s[0], cr);
    atomicAdd(&cnt_s[1], cv);
  }
  __syncthreads();
  if (tid < 6) {
    const unsigned long long c = cnt_s[tid / 3];
    long long r = (long long)ceil((double)c * pct.f[tid % 3]);
    rank[tid] = r < 1 ? 1 : r;
    prefix[tid] = 0;
  }
  if (tid == 0) counts[j] = (int64_t)cnt_s[0];
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int k = tid; k < 6 * 256; k += blockDim.x) (&hist[0][0])[k] = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const unsigned long long xr = (unsigned long long)__double_as_longlong(__ldg(dr + i * m + j));
      const unsigned long long xv = (unsigned long long)__double_as_longlong(__ldg(dv + i * m + j));
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const unsigned long long x = s < 3 ? xr : xv;
        const bool match = pass == 0 || ((x ^ prefix[s]) >> (shift + 8)) == 0;
        if (match) atomicAdd(&hist[s][(x >> shift) & 255], 1u);
      }
    }
    __syncthreads();
    if (tid < 6) {
      long long r = rank[tid];
      int b = 0;
      for (; b < 255; ++b) {
        if (r <= (long long)hist[tid][b]) break;
        r -= hist[tid][b];
      }
      rank[tid] = r;
      prefix[tid] |= (unsigned long long)b << shift;
    }
    __syncthreads();
  }
  if (tid < 6) {
    const unsigned long long c = cnt_s[tid / 3];
    table[tid * m + j] = c > 0 ? __longlong_as_double((long long)prefix[tid]) : CUDART_NAN;
  }
}

bool grav_from(const double* grav, Grav& g) {
  if (grav == nullptr) return false;
  g.mu = grav[0]; g.re = grav[1]; g.xke = grav[2]; g.tumin = grav[3];
  g.j2 = grav[4]; g.j3 = grav[5]; g.j4 = grav[6]; g.j3oj2 = grav[7];
  g.vkm = g.re * g.xke / 60.0;
  g.inv_xke = 1.0 / g.xke;
  g.xke_f = (float)g.xke;
  g.re_f = (float)g.re;
  g.vkm_f = (float)g.vkm;
  g.inv_xke_f = (float)(1.0 / g.xke);
  g.half_j2_f = (float)(0.5 * g.j2);
  return true;
}

// blocks of grid_kernel that fit on the current device at once (cached per
// device and variant): the persistent grid size.
int64_t resident_blocks(int precision) {
  static int cache[64][2];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    fail(SGP4B_ECUDA, "cudaGetDevice failed");
    return -1;
  }
  const int v = precision == 64 ? 1 : 0;
  if (cache[dev][v] > 0) return cache[dev][v];
  int sms = 0, per_sm = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = precision == 64 ? (const void*)grid_kernel<double, true, false>
                                    : (const void*)grid_kernel<float, true, false>;
  const int block = precision == 64 ? grid_block<double>() : grid_block<float>();
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, 0);
  if (e != cudaSuccess || sms <= 0 || per_sm <= 0) {
    fail(SGP4B_ECUDA, "occupancy query: %s", cudaGetErrorString(e));
    return -1;
  }
  cache[dev][v] = sms * per_sm;
  return cache[dev][v];
}

// persistent launch of grid_kernel (dense grid or, with rec_idx, pairs)
int launch_grid(const void* rec, const int64_t* rec_idx, int64_t n, const void* times,
                const float* times_lo, int64_t times_ld, int64_t m, int precision, const Grav& g,
                void* planes, int64_t plane_stride, int64_t row_stride, int32_t* codes,
                int64_t code_stride, bool vec, double t_absmax, cudaStream_t s, const char* what) {
  // an upper bound on |t|, rounded up into fp32 (NaN stays NaN: unbounded)
  float tb = (float)t_absmax;
  if ((double)tb < t_absmax) tb = nextafterf(tb, INFINITY);
  const int64_t chunks = (m + kCellsPerWarp - 1) / kCellsPerWarp;
  const int64_t warps = n * chunks;
  const int block = precision == 64 ? grid_block<double>() : grid_block<float>();
  int64_t blocks = (warps * 32 + block - 1) / block;
  const int64_t slots = resident_blocks(precision);
  if (slots <= 0) return fail(SGP4B_ECUDA, "%s: %s", what, g_last_error);
  if (blocks > slots) blocks = slots;
  if (precision == 64) {
    // fp64 rows store cell by cell (no vector path): one instance serves all
    auto k = grid_kernel<double, true, false>;
    k<<<(unsigned)blocks, block, 0, s>>>(
        static_cast<const double*>(rec), rec_idx, n, static_cast<const double*>(times), nullptr,
        times_ld, m, g, static_cast<double*>(planes), plane_stride, row_stride, codes,
        code_stride, chunks, tb);
  } else {
    auto k = times_lo != nullptr
                 ? (vec ? grid_kernel<float, true, true> : grid_kernel<float, false, true>)
                 : (vec ? grid_kernel<float, true, false> : grid_kernel<float, false, false>);
    k<<<(unsigned)blocks, block, 0, s>>>(
        static_cast<const float*>(rec), rec_idx, n, static_cast<const float*>(times), times_lo,
        times_ld, m, g, static_cast<float*>(planes), plane_stride, row_stride, codes, code_stride,
        chunks, tb);
  }
  return check_launch(what);
}

inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

// ======================================================================
// C ABI
// ======================================================================
extern "C" {

int sgp4b_abi_version(void) { return 7; }

#ifdef SGP4B_TIMELINE
int sgp4b_debug_timeline(unsigned long long* host, int warps) {
  if (warps > kTimelineWarps) warps = kTimelineWarps;
  return (int)cudaMemcpyFromSymbol(host, g_timeline, sizeof(unsigned long long) * 4 * warps);
}
#endif

const char* sgp4b_last_error(void) { return g_last_error; }

int sgp4b_init(const double* elements_dev, int64_t n, const double* grav, int precision,
               double* satrec_dev, int32_t* init_code_dev, uint8_t* isimp_dev, void* record_dev,
               void* stream) {
  Grav g;
  if (n <= 0) return fail(SGP4B_EINVAL, "sgp4b_init: n must be positive (got %lld)", (long long)n);
  if (precision != 32 && precision != 64)
    return fail(SGP4B_EINVAL, "sgp4b_init: precision must be 32 or 64, got %d", precision);
  if (!elements_dev || !init_code_dev || !isimp_dev || !grav_from(grav, g))
    return fail(SGP4B_EINVAL, "sgp4b_init: null pointer argument");
  if (!satrec_dev && !record_dev)
    return fail(SGP4B_EINVAL, "sgp4b_init: neither satrec_dev nor record_dev given");
  // one warp per block: init is a long fp64 dependency chain per thread, so
  // spread the few satellite-warps over as many SMs as possible
  init_kernel<<<blocks_for(n, 32), 32, 0, (cudaStream_t)stream>>>(
      elements_dev, n, g, satrec_dev, init_code_dev, isimp_dev, record_dev, precision);
  return check_launch("sgp4b_init");
}

int sgp4b_pack(const double* satrec_dev, const int32_t* init_code_dev, const uint8_t* isimp_dev,
               int64_t n, const double* grav, int precision, void* record_dev, void* stream) {
  Grav g;
  if (n <= 0) return fail(SGP4B_EINVAL, "sgp4b_pack: n must be positive");
  if (precision != 32 && precision != 64)
    return fail(SGP4B_EINVAL, "sgp4b_pack: precision must be 32 or 64, got %d", precision);
  if (!satrec_dev || !init_code_dev || !isimp_dev || !record_dev || !grav_from(grav, g))
    return fail(SGP4B_EINVAL, "sgp4b_pack: null pointer argument");
  pack_kernel<<<blocks_for(n, 32), 32, 0, (cudaStream_t)stream>>>(
      satrec_dev, init_code_dev, isimp_dev, n, g, record_dev, precision);
  return check_launch("sgp4b_pack");
}

int sgp4b_propagate_grid(const void* record_dev, int64_t n, const void* times_dev,
                         const float* times_lo_dev, int64_t m, double t_absmax, int precision,
                         const double* grav, void* planes_dev, int64_t plane_stride,
                         int64_t row_stride, int32_t* codes_dev, int64_t code_stride,
                         void* stream) {
  Grav g;
  if (n <= 0 || m <= 0)
    return fail(SGP4B_EINVAL, "sgp4b_propagate_grid: empty grid (%lld x %lld)", (long long)n,
                (long long)m);
  if (precision != 32 && precision != 64)
    return fail(SGP4B_EINVAL, "sgp4b_propagate_grid: precision must be 32 or 64, got %d", precision);
  if (!record_dev || !times_dev || !planes_dev || !codes_dev || !grav_from(grav, g))
    return fail(SGP4B_EINVAL, "sgp4b_propagate_grid: null pointer argument");
  if (m > kMaxSteps)
    return fail(SGP4B_EINVAL, "sgp4b_propagate_grid: m = %lld exceeds 2^30 steps per row",
                (long long)m);
  if (row_stride < m || code_stride < m || plane_stride < (n - 1) * row_stride + m)
    return fail(SGP4B_EINVAL, "sgp4b_propagate_grid: strides overlap the grid");
  const size_t esz = precision == 64 ? 8 : 4;
  const bool vec = (plane_stride % 4 == 0) && (row_stride % 4 == 0) && (code_stride % 4 == 0) &&
                   ((uintptr_t)planes_dev % (4 * esz) == 0) && ((uintptr_t)codes_dev % 16 == 0) &&
                   ((uintptr_t)times_dev % (4 * esz) == 0);
  return launch_grid(record_dev, nullptr, n, times_dev, times_lo_dev, 0, m, precision, g,
                     planes_dev, plane_stride, row_stride, codes_dev, code_stride, vec, t_absmax,
                     (cudaStream_t)stream, "sgp4b_propagate_grid");
}

int sgp4b_propagate_pairs(const void* record_dev, const int64_t* sat_idx_dev, const void* times_dev,
                          const float* times_lo_dev, int64_t p, double t_absmax, int precision,
                          const double* grav, void* rv_dev, int32_t* codes_dev, void* stream) {
  Grav g;
  if (p <= 0) return fail(SGP4B_EINVAL, "sgp4b_propagate_pairs: p must be positive");
  if (precision != 32 && precision != 64)
    return fail(SGP4B_EINVAL, "sgp4b_propagate_pairs: precision must be 32 or 64, got %d", precision);
  if (!record_dev || !sat_idx_dev || !times_dev || !rv_dev || !codes_dev || !grav_from(grav, g))
    return fail(SGP4B_EINVAL, "sgp4b_propagate_pairs: null pointer argument");
#if SGP4B_PAIRS_LANE
  if (precision == 32) {
    const float* tlo = static_cast<const float*>(times_lo_dev);
    // launch_grid's bound: |t| rounded up into fp32, NaN stays NaN
    float tb = (float)t_absmax;
    if ((double)tb < t_absmax) tb = nextafterf(tb, INFINITY);
    const unsigned blocks = (unsigned)((p + kPairsBlock - 1) / kPairsBlock);
    if (tlo != nullptr)
      pairs_kernel32<true><<<blocks, kPairsBlock, 0, (cudaStream_t)stream>>>(
          static_cast<const float*>(record_dev), sat_idx_dev, p,
          static_cast<const float*>(times_dev), tlo, g, static_cast<float*>(rv_dev), codes_dev, tb);
    else
      pairs_kernel32<false><<<blocks, kPairsBlock, 0, (cudaStream_t)stream>>>(
          static_cast<const float*>(record_dev), sat_idx_dev, p,
          static_cast<const float*>(times_dev), nullptr, g, static_cast<float*>(rv_dev), codes_dev,
          tb);
    return check_launch("sgp4b_propagate_pairs");
  }
  if (precision == 64) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      return fail(SGP4B_ECUDA, "sgp4b_propagate_pairs: device query failed");
    const int64_t need = (p + kPairsBlock64 - 1) / kPairsBlock64;
    const unsigned blocks = (unsigned)std::min<int64_t>(need, (int64_t)sms * 4);   // 4 resident per SM
    pairs_kernel64<<<blocks, kPairsBlock64, 0, (cudaStream_t)stream>>>(
        static_cast<const double*>(record_dev), sat_idx_dev, p,
        static_cast<const double*>(times_dev), g, static_cast<double*>(rv_dev), codes_dev);
    return check_launch("sgp4b_propagate_pairs");
  }
#endif
  // P rows of one step: row k = record sat_idx[k] at times[k]; output (6, P).
  // The VEC instance (m = 1 never takes its vector path) is the one aligned
  // grids use, so a pair equals the corresponding grid cell bit for bit.
  return launch_grid(record_dev, sat_idx_dev, p, times_dev, times_lo_dev, 1, 1, precision, g,
                     rv_dev, p, 1, codes_dev, 1, true, t_absmax, (cudaStream_t)stream,
                     "sgp4b_propagate_pairs");
}

int sgp4b_drift_norms(const float* planes32_dev, const double* planes64_dev,
                      const int32_t* codes32_dev, const int32_t* codes64_dev, int64_t n, int64_t m,
                      double* dr_dev, double* dv_dev, void* stream) {
  if (n <= 0 || m <= 0) return fail(SGP4B_EINVAL, "sgp4b_drift_norms: empty grid");
  if (!planes32_dev || !planes64_dev || !codes32_dev || !codes64_dev || !dr_dev || !dv_dev)
    return fail(SGP4B_EINVAL, "sgp4b_drift_norms: null pointer argument");
  const int64_t cells = n * m;
  drift_norms_kernel<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      planes32_dev, planes64_dev, codes32_dev, codes64_dev, cells, dr_dev, dv_dev);
  return check_launch("sgp4b_drift_norms");
}

int sgp4b_drift_percentiles(const double* dr_dev, const double* dv_dev, int64_t n, int64_t m,
                            const double* pct_frac, double* table_dev, int64_t* counts_dev,
                            void* stream) {
  if (n <= 0 || m <= 0) return fail(SGP4B_EINVAL, "sgp4b_drift_percentiles: empty grid");
  if (!dr_dev || !dv_dev || !pct_frac || !table_dev || !counts_dev)
    return fail(SGP4B_EINVAL, "sgp4b_drift_percentiles: null pointer argument");
  if (m > 0x7fffffff) return fail(SGP4B_EINVAL, "sgp4b_drift_percentiles: too many columns");
  Pct3 pct;
  for (int k = 0; k < 3; ++k) pct.f[k] = pct_frac[k];
  drift_pct_kernel<<<(unsigned)m, 256, 0, (cudaStream_t)stream>>>(dr_dev, dv_dev, n, m, pct,
                                                                   table_dev, counts_dev);
  return check_launch("sgp4b_drift_percentiles");
}

int sgp4b_tle_columns(const uint8_t* text_dev, int64_t size, const int64_t* line1_dev,
                      const int64_t* line2_dev, int64_t n, const double* pow10_dev,
                      double* cols_dev, int32_t* status_dev, void* stream) {
  if (n <= 0 || size <= 0) return fail(SGP4B_EINVAL, "sgp4b_tle_columns: empty catalogue");
  if (!text_dev || !line1_dev || !line2_dev || !pow10_dev || !cols_dev || !status_dev)
    return fail(SGP4B_EINVAL, "sgp4b_tle_columns: null pointer argument");
  tle_columns_kernel<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      text_dev, size, line1_dev, line2_dev, n, pow10_dev, cols_dev, status_dev);
  return check_launch("sgp4b_tle_columns");
}

int sgp4b_code_rows(const int32_t* codes_dev, int64_t n, int64_t m, int64_t code_stride,
                    uint8_t* flags_dev, void* stream) {
  if (n <= 0 || m <= 0) return fail(SGP4B_EINVAL, "sgp4b_code_rows: empty grid");
  if (!codes_dev || !flags_dev) return fail(SGP4B_EINVAL, "sgp4b_code_rows: null pointer argument");
  if (code_stride < m) return fail(SGP4B_EINVAL, "sgp4b_code_rows: code_stride < m");
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 8);
  code_rows_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(codes_dev, n, m,
                                                                     code_stride, flags_dev);
  return check_launch("sgp4b_code_rows");
}

int sgp4b_solve_kepler(const void* axnl_dev, const void* aynl_dev, const void* u_dev, int64_t n,
                       int precision, void* out_dev, void* stream) {
  if (n <= 0) return fail(SGP4B_EINVAL, "sgp4b_solve_kepler: n must be positive");
  if (precision != 32 && precision != 64)
    return fail(SGP4B_EINVAL, "sgp4b_solve_kepler: precision must be 32 or 64, got %d", precision);
  if (!axnl_dev || !aynl_dev || !u_dev || !out_dev)
    return fail(SGP4B_EINVAL, "sgp4b_solve_kepler: null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == 64)
    kepler_kernel<double><<<blocks_for(n, 256), 256, 0, s>>>(
        static_cast<const double*>(axnl_dev), static_cast<const double*>(aynl_dev),
        static_cast<const double*>(u_dev), n, static_cast<double*>(out_dev));
  else
    kepler_kernel<float><<<blocks_for(n, 256), 256, 0, s>>>(
        static_cast<const float*>(axnl_dev), static_cast<const float*>(aynl_dev),
        static_cast<const float*>(u_dev), n, static_cast<float*>(out_dev));
  return check_launch("sgp4b_solve_kepler");
}

int sgp4b_peer_access(int device, int peer) {
  if (device == peer) return SGP4B_OK;
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e != cudaSuccess || !can) {
    cudaGetLastError();
    return fail(SGP4B_ECUDA, "sgp4b_peer_access: device %d cannot access device %d", device, peer);
  }
  int prev = -1;
  cudaGetDevice(&prev);
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
  cudaGetLastError();
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess)
    return fail(SGP4B_ECUDA, "sgp4b_peer_access(%d -> %d): %s", device, peer, cudaGetErrorString(e));
  return SGP4B_OK;
}

int sgp4b_host_alloc(int64_t nbytes, void** out) {
  if (out == nullptr) return fail(SGP4B_EINVAL, "sgp4b_host_alloc: null out pointer");
  *out = nullptr;
  if (nbytes <= 0) return fail(SGP4B_EINVAL, "sgp4b_host_alloc: nbytes must be positive");
  // portable: any device of the process may DMA into it (multi-GPU grids)
  cudaError_t e = cudaHostAlloc(out, (size_t)nbytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *out = nullptr;
    cudaGetLastError();
    return fail(SGP4B_ENOMEM, "sgp4b_host_alloc(%lld): %s", (long long)nbytes, cudaGetErrorString(e));
  }
  return SGP4B_OK;
}

int sgp4b_host_free(void* p) {
  if (p == nullptr) return SGP4B_OK;
  cudaError_t e = cudaFreeHost(p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SGP4B_ECUDA, "sgp4b_host_free: %s", cudaGetErrorString(e));
  }
  return SGP4B_OK;
}

}  // extern "C"
