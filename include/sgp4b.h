/*
 * sgp4b.h — C ABI of the B200-native SGP4 batch propagator.
 *
 * The reference package (`sgp4kit`, /root/reference/pkg) has no native
 * boundary: its hot path is the Python API
 *     init_batch()       pkg/src/sgp4kit/batch.py:92-109
 *     propagate_batch()  pkg/src/sgp4kit/batch.py:166-205
 *     sgp4_init()        pkg/src/sgp4kit/kernel.py:139-151
 *     sgp4_propagate()   pkg/src/sgp4kit/kernel.py:513-534
 *     solve_kepler()     pkg/src/sgp4kit/kernel.py:325-349
 * Each entry point below replaces the numeric core of one of those calls;
 * the Python mirror (paper_2603_27830_b200/) binds them with ctypes.
 *
 * Conventions
 *   - Every pointer named *_dev is a device pointer on the current device;
 *     the library never allocates device memory (sgp4b_host_alloc is the only
 *     allocator, for pinned HOST result buffers), never synchronises and
 *     never aborts.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Return 0 on success or a negative SGP4B_E* status.  The message of the
 *     last failure on the calling thread is sgp4b_last_error().
 *   - Per-cell anomalies (decay, eccentricity out of range …) are DATA in the
 *     int32 code plane, never a status (kernel.py:45-52, 497-502).
 *   - precision is 32 or 64 (batch.py:84-89); "T" below is float or double.
 */
#ifndef SGP4B_H
#define SGP4B_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGP4B_OK 0
#define SGP4B_EINVAL (-1)   /* bad argument (size, precision, null pointer) */
#define SGP4B_ECUDA (-2)    /* CUDA launch/config error */
#define SGP4B_ENOMEM (-3)   /* page-locked host allocation failed */

/* Number of float slots in one satellite's SoA satrec (public SatInit float
 * fields, kernel.py:64-107, in dataclass order). */
#define SGP4B_SATREC_FIELDS 33
/* Number of T slots in one packed propagate record. */
#define SGP4B_RECORD_SLOTS 40

/* grav: HOST pointer to 8 doubles {mu, radius_earth_km, xke, tumin, j2, j3,
 * j4, j3oj2} (gravity.py:13-28); read at launch time.  The propagate calls
 * must pass the model the records were built with (init/pack): as in the
 * reference, where SatInit carries its grav (kernel.py:64) and _propagate
 * reads init.grav (kernel.py:353), the model belongs to the satrec, and the
 * fp32 records fold 0.5 j2, the Earth radius and the km/s scale into their
 * per-satellite coefficients. */

/* Initialisation, one thread per satellite, always evaluated in fp64.
 * Replaces _sgp4_init (kernel.py:154-322) incl. the epoch evaluation
 * (kernel.py:316-322).
 *   elements_dev : (7, n) fp64 SoA {no_kozai, ecco, inclo, nodeo, argpo, mo, bstar}
 *   satrec_dev   : (33, n) fp64 SoA out, SatInit float fields in order
 *                  (may be NULL: the propagate path only needs the records;
 *                  a later call with the same elements writes the same
 *                  satrec bit for bit)
 *   init_code_dev: (n) int32 out, error_code_at_init
 *   isimp_dev    : (n) uint8 out
 *   record_dev   : (n, 40) packed T records out (may be NULL; not both) */
int sgp4b_init(const double* elements_dev, int64_t n, const double* grav,
               int precision, double* satrec_dev, int32_t* init_code_dev,
               uint8_t* isimp_dev, void* record_dev, void* stream);

/* Packs a (possibly user-edited) fp64 SoA satrec into propagate records.
 * Used when a SatInit did not come from sgp4b_init (dataclasses.replace). */
int sgp4b_pack(const double* satrec_dev, const int32_t* init_code_dev,
               const uint8_t* isimp_dev, int64_t n, const double* grav,
               int precision, void* record_dev, void* stream);

/* Dense grid: cell (i, j) = satellite i at times[j].  Replaces
 * propagate_batch + _propagate + solve_kepler + the init-code merge
 * (batch.py:166-205, kernel.py:325-534).
 *   record_dev : (n, 40) packed T records
 *   times_dev  : (m) T minutes since epoch
 *   times_lo_dev: (m) float low words for precision 32 (t = hi + lo exactly
 *                 as the caller's fp64 time), or NULL; ignored for 64
 *   planes_dev : T base; plane p, row i, col j at
 *                planes_dev[p*plane_stride + i*row_stride + j]
 *   codes_dev  : int32 base; row i, col j at codes_dev[i*code_stride + j]
 *   t_absmax   : an upper bound on |times[j]| (minutes).  fp32 launches pick
 *                each satellite's fixed-iteration Kepler class from ecco and
 *                recompute the cells whose |t| could carry em out of that
 *                class (drag over long or backward spans) with the general
 *                path; the bound tells the kernel which rows can have such
 *                cells.  INFINITY or NaN is always correct (every row of a
 *                fixed class gets the check), only slower; fp64 ignores it.
 *   m is at most 2^30 (columns are indexed with 32-bit offsets; longer
 *   rows are split by the caller). */
int sgp4b_propagate_grid(const void* record_dev, int64_t n,
                         const void* times_dev, const float* times_lo_dev,
                         int64_t m, double t_absmax, int precision,
                         const double* grav, void* planes_dev,
                         int64_t plane_stride, int64_t row_stride,
                         int32_t* codes_dev, int64_t code_stride,
                         void* stream);

/* Elementwise pairs: cell k = satellite sat_idx[k] at times[k].  Replaces
 * the broadcasting scalar sgp4_propagate (kernel.py:513-534).  Each pair
 * equals the sgp4b_propagate_grid cell of the same (record, time, time low
 * word, t_absmax) bit for bit.  Every sat_idx[k] must index a record of
 * record_dev (the call has no record count to check it against).
 *   rv_dev : (6, p) T out; codes_dev : (p) int32 out. */
int sgp4b_propagate_pairs(const void* record_dev, const int64_t* sat_idx_dev,
                          const void* times_dev, const float* times_lo_dev,
                          int64_t p, double t_absmax, int precision,
                          const double* grav, void* rv_dev, int32_t* codes_dev,
                          void* stream);

/* fp32-vs-fp64 drift: per-cell |r32 - r64| (km) and |v32 - v64| (km/s) in
 * fp64 for cells whose codes are 0 in both grids, +inf elsewhere.  Both
 * grids contiguous (6, n, m); dr/dv (n, m).  Replaces the norm step of
 * drift_report (drift.py:64-70); percentiles are taken by the caller. */
int sgp4b_drift_norms(const float* planes32_dev, const double* planes64_dev,
                      const int32_t* codes32_dev, const int32_t* codes64_dev,
                      int64_t n, int64_t m, double* dr_dev, double* dv_dev,
                      void* stream);

/* Nearest-rank percentiles per column of the drift norms (drift.py:46-49,
 * 74-92): for each column j, the rank-th smallest finite value of dr and of
 * dv with rank = max(1, ceil(count_j * pct_frac[k])), k = 0..2.
 *   pct_frac  : HOST pointer to 3 doubles (p / 100.0, e.g. 0.05, 0.5, 0.95)
 *   table_dev : (6, m) fp64 out: dr at the 3 fractions, then dv; NaN for a
 *               column without finite values
 *   counts_dev: (m) int64 out, finite cells per column */
int sgp4b_drift_percentiles(const double* dr_dev, const double* dv_dev,
                            int64_t n, int64_t m, const double* pct_frac,
                            double* table_dev, int64_t* counts_dev,
                            void* stream);

/* TLE catalogue ingest on the device: the columns of
 * parse_catalog_columns (tle.py:390-433 here; the reference's per-record
 * parse_tle + _canonical_elements, tle.py:185-276) for n records whose line
 * 1 / line 2 start at byte offsets line1_dev[i] / line2_dev[i] of text_dev
 * (size bytes; a line ends at '\n').
 *   pow10_dev : 42 doubles: 10.0**k for k = 0..22 (exact), then the
 *               host's 10.0**e for e = -9..9 (the B* exponent multiplier)
 *   cols_dev  : (7, n) fp64 out, ELEMENT_COLUMNS order (init input)
 *   status_dev: (n) int32 out, 0 or a bit per field whose text falls
 *               outside the simple decimal syntax: the caller re-decodes
 *               those records on the host. */
int sgp4b_tle_columns(const uint8_t* text_dev, int64_t size,
                      const int64_t* line1_dev, const int64_t* line2_dev,
                      int64_t n, const double* pow10_dev, double* cols_dev,
                      int32_t* status_dev, void* stream);

/* Row summary of a code plane: flags_dev[i] = 1 when row i (codes_dev +
 * i*code_stride, m entries) holds a nonzero code, else 0.  Lets the host
 * copy of a BatchResult (batch.py:177-183, the int32 error plane) move only
 * the rows that carry codes over PCIe and zero-fill the others in host
 * memory, since most catalogues have no failing cells. */
int sgp4b_code_rows(const int32_t* codes_dev, int64_t n, int64_t m,
                    int64_t code_stride, uint8_t* flags_dev, void* stream);

/* Newton solve of SGP4's Kepler equation, elementwise (kernel.py:325-349). */
int sgp4b_solve_kepler(const void* axnl_dev, const void* aynl_dev,
                       const void* u_dev, int64_t n, int precision,
                       void* out_dev, void* stream);

/* Lets kernels running on `device` load and store `peer`'s memory (NVLink
 * peer access), so a satellite shard computed on one GPU can store its rows
 * straight into a grid that lives on another (no gather step).  0 when
 * enabled (or already enabled, or device == peer), SGP4B_ECUDA when the
 * pair cannot be peers. */
int sgp4b_peer_access(int device, int peer);

/* Page-locked (pinned, portable) host memory for result grids.  The
 * reference returns pageable np.empty grids (batch.py:177-183); results that
 * come back over PCIe need pinned memory for full-rate D2H, and the Python
 * layer pools these blocks at their exact (2 MiB-rounded) size.  These are
 * the only calls that allocate, and they allocate HOST memory only. */
int sgp4b_host_alloc(int64_t nbytes, void** out);
int sgp4b_host_free(void* p);

/* Thread-local message for the last non-zero status. */
const char* sgp4b_last_error(void);

/* ABI version (bumped on any signature or record-layout change). */
int sgp4b_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SGP4B_H */
