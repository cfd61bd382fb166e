/*
 * pswe_b200.h -- C ABI of the B200-native phase-averaged shallow-water RHS.
 *
 * Drop-in boundary for the hot path of the reference package `phaseswe`
 * (arXiv 2103.07706, /root/reference/pkg/src/phaseswe).  The reference is pure
 * Python, so it has no FFI of its own; these entry points are what its
 * Python operator API binds through ctypes.  Each entry
 * point names the reference function it replaces.
 *
 * Conventions
 *  - Complex numbers are interleaved fp64 pairs (re, im): a field of nx*ny
 *    modes is 2*nx*ny doubles.  "full" fields are (nx, ny) row-major arrays
 *    in numpy fft2 order (grid.py:3-8); a state is three such arrays
 *    (u, v, eta), passed as three pointers exactly like State.u/.v/.eta
 *    (dynamics.py:72-118).
 *  - "compact" states hold only the 2/3 band (grid.py:102-103) for ky >= 0:
 *    3 * Ky * Kx complex values, Ky = ny/3 + 1, Kx = 2*(nx/3) + 1, ordered
 *    [field][ky][kx] with kx in FFT order (0..nx/3, then -nx/3..-1).
 *  - Pointers named *_dev are device pointers on the context's device;
 *    *_host are host pointers.  `stream` is a cudaStream_t (NULL = legacy
 *    default stream).  All launches are asynchronous on that stream unless
 *    stated otherwise.
 *  - Return value: 0 on success, nonzero on error; pswe_last_error() gives a
 *    thread-local message.  Errors from argument validation use the
 *    reference's wording where the reference raises.
 *  - Grid sizes: nx, ny powers of two in [8, 512] (the reference allows
 *    any even n >= 8, grid.py:91-93; other sizes return PSWE_EUNSUPPORTED).
 *  - Threading: a context may be used by one host thread at a time.
 */
#ifndef PSWE_B200_H
#define PSWE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSWE_OK 0
#define PSWE_EINVAL 1        /* invalid argument (reference: ValueError) */
#define PSWE_ECUDA 2         /* CUDA runtime error */
#define PSWE_EUNSUPPORTED 3  /* grid size not supported by the GPU path */
#define PSWE_ENONFINITE 4    /* non-finite state after a stage (integrator.py:77-80) */
#define PSWE_ESTATE 5        /* call order violated (e.g. no quadrature set) */
#define PSWE_EHERM 6         /* non-Hermitian spectral input (to_physical's gate, grid.py:159-172) */

typedef struct pswe_ctx pswe_ctx;

/* ABI version (major * 100 + minor). */
int pswe_version(void);
const char* pswe_last_error(void);

/* Grid + physics on one device.  Replaces make_grid (grid.py:81-107) and the
 * scalar part of PhysicsParams (dynamics.py:34-63); b starts flat
 * (flat_bottom, dynamics.py:66-69). */
int pswe_create(pswe_ctx** ctx, int nx, int ny, double Lx, double Ly, double f, double g,
                double H, int device);
void pswe_destroy(pswe_ctx* ctx);

/* Topography: full-layout spectral b (PhysicsParams.b).  Only its 2/3 band
 * enters N (dynamics.py:157). */
int pswe_set_topography(pswe_ctx* ctx, const double* b_dev, void* stream);

/* Quadrature nodes/weights (Quadrature, averaging.py:59-77): n_nodes = 2M+1
 * host arrays in ascending k.  Zero-weight nodes are skipped
 * (averaging.py:128). */
int pswe_set_quadrature(pswe_ctx* ctx, int n_nodes, const double* s_host, const double* w_host);

/* Exponential route (PropagatorSpec, propagator.py:48-80): kind 0 = exact
 * (exact_exp, propagator.py:96-110), kind 1 = Chebyshev (cheb_exp,
 * propagator.py:161-191) with host coefficients a[0..n_poly]
 * (cheb_coeffs, propagator.py:133-139). */
int pswe_set_propagator(pswe_ctx* ctx, int kind, double Lambda, int n_poly, const double* a_host);

/* Sizes of the compact layout. */
int pswe_compact_shape(const pswe_ctx* ctx, int* Ky, int* Kx);

/* full -> compact (with the Hermitian projection real(ifft2) implies,
 * grid.py:173-174) and compact -> full (zero outside the band, conjugate
 * mirror for ky < 0). */
int pswe_pack(pswe_ctx* ctx, const double* u_dev, const double* v_dev, const double* eta_dev,
              double* Uc_dev, void* stream);
int pswe_unpack(pswe_ctx* ctx, const double* Uc_dev, double* u_dev, double* v_dev, double* eta_dev,
                void* stream);

/* Averaged tendency sum_k w_k e^{-s_k L} N(e^{s_k L} U) over the live nodes
 * (averaged_tendency, averaging.py:116-156).  Compact in/out. */
int pswe_averaged_tendency_compact(pswe_ctx* ctx, const double* Uc_dev, double* Ac_dev, void* stream);

/* Same, full layout in/out (the reference's array layout). */
int pswe_averaged_tendency(pswe_ctx* ctx, const double* u_dev, const double* v_dev,
                           const double* eta_dev, double* du_dev, double* dv_dev, double* deta_dev,
                           void* stream);

/* Same, and the result's 2/3 band (everything that can be nonzero: the
 * tendency is dealiased) copied into three pinned host buffers of the full
 * (nx, ny) layout before the call's single synchronisation -- the drop-in
 * call's device-to-host leg (averaging.py:116-156 returns host arrays).
 * Host entries outside the band are not touched. */
int pswe_averaged_tendency_band_d2h(pswe_ctx* ctx, const double* u_dev, const double* v_dev,
                                    const double* eta_dev, double* du_dev, double* dv_dev, double* deta_dev,
                                    double* const* host3, void* stream);

/* N(U) alone (apply_nonlinear, dynamics.py:139-176), full layout. */
int pswe_apply_nonlinear(pswe_ctx* ctx, const double* u_dev, const double* v_dev,
                         const double* eta_dev, double* du_dev, double* dv_dev, double* deta_dev,
                         void* stream);

/* L U (apply_linear, dynamics.py:128-136), full layout. */
int pswe_apply_linear(pswe_ctx* ctx, const double* u_dev, const double* v_dev, const double* eta_dev,
                      double* lu_dev, double* lv_dev, double* leta_dev, void* stream);

/* e^{tL} U by the configured route (propagate, propagator.py:194-199).  The
 * Chebyshev precondition |t| * max_frequency <= Lambda (1 + 1e-9)
 * (propagator.py:172-176) is checked on the host: PSWE_EINVAL. */
int pswe_propagate(pswe_ctx* ctx, double t, const double* u_dev, const double* v_dev,
                   const double* eta_dev, double* ou_dev, double* ov_dev, double* oeta_dev,
                   void* stream);

/* One transformed SSPRK3 step (step_averaged_ssprk3, integrator.py:83-103),
 * full layout; in and out may alias.  Synchronises the stream and returns
 * PSWE_ENONFINITE with *bad_stage (1..3) and *bad_field (0 u, 1 v, 2 eta)
 * set for the first non-finite stage (integrator.py:77-80); otherwise sets
 * them to 0 / -1. */
int pswe_ssprk3_step(pswe_ctx* ctx, double dt, const double* u_dev, const double* v_dev,
                     const double* eta_dev, double* ou_dev, double* ov_dev, double* oeta_dev,
                     int* bad_stage, int* bad_field, void* stream);

/* nsteps steps in place (the step loop of run, integrator.py:173-179).  On a
 * non-finite stage returns PSWE_ENONFINITE with *bad_step (1-based) set and
 * the state left at the start of that step. */
int pswe_run(pswe_ctx* ctx, double dt, int nsteps, double* u_dev, double* v_dev, double* eta_dev,
             int* bad_step, int* bad_stage, int* bad_field, void* stream);

/* Window batch (the window sweep, harness.py:110-147 cmd_sweep and
 * validation.py:251-271): W averaging windows -- each its own quadrature of
 * n_nodes[i] = 2 M_i + 1 nodes, s and w concatenated over the windows in
 * window order -- advanced together: one launch sequence per stage serves
 * every window, the phases of all windows forming one batch axis
 * (window, phase).  Zero-weight nodes are skipped as in
 * pswe_set_quadrature.  Grid, physics, topography and propagator are the
 * context's. */
int pswe_set_window_batch(pswe_ctx* ctx, int W, const int* n_nodes, const double* s_host, const double* w_host);

/* Averaged tendencies of the W windows: Uc / Ac = W compact states
 * ([W][3][Ky][Kx]); window w's tendency uses window w's state and nodes. */
int pswe_window_batch_tendency(pswe_ctx* ctx, const double* Uc_dev, double* Ac_dev, void* stream);

/* nsteps transformed SSPRK3 steps of all W windows in place on
 * U_dev = [W][3][nx][ny] (window w's u, v, eta).  When any window's step
 * flags a non-finite stage or the Hermitian gate, returns PSWE_ENONFINITE
 * with *bad_step (1-based) and every window left at the start of that step;
 * the caller replays the windows one by one (pswe_run) for the reference's
 * per-window error. */
int pswe_window_batch_run(pswe_ctx* ctx, double dt, int nsteps, double* U_dev, int* bad_step, void* stream);

/* Largest |eigenvalue| of L over the grid (max_frequency, dynamics.py:189-192). */
double pswe_max_frequency(const pswe_ctx* ctx);

/* Number of kernels this context has launched (instrumentation). */
int64_t pswe_launch_count(const pswe_ctx* ctx);

/* Debug (environment PSWE_DEBUG_GUARD set before the first allocation):
 * every context buffer carries 64 KiB NaN-filled guard bands on both sides.
 * Synchronises the device and returns the number of live guarded buffers and
 * of guard bands found changed (including those of buffers freed since).
 * Without PSWE_DEBUG_GUARD both are 0.  A memcheck stand-in; no reference
 * counterpart. */
int pswe_debug_check_guards(int64_t* guarded, int64_t* damaged);

/* Launches per kernel variant (instrumentation: which code path ran), graph
 * replays included.  Variants: */
#define PSWE_V_PASSA 0        /* pass A (e^{sL} + inverse x-FFTs) */
#define PSWE_V_PASSB_PAIR 1   /* pass B, phase-paired, TMEM stash + TMA tile stores */
#define PSWE_V_PASSB_ROW 2    /* pass B, one phase per warp */
#define PSWE_V_PASSB_SPLIT 3  /* pass B, a row group's transforms over four warps */
#define PSWE_V_PASSC 4        /* pass C (forward x-FFTs, e^{-sL}, weighted sum) */
#define PSWE_V_REDUCE 5       /* ordered slot reduction */
#define PSWE_V_FUSED 6        /* fused one-CTA-per-phase small-grid kernel */
#define PSWE_V_HERM 7         /* exact Hermitian-defect check (error path) */
#define PSWE_NUM_VARIANTS 8
int pswe_variant_launches(const pswe_ctx* ctx, int64_t* counts, int n);

/* Snapshot diagnostics of a full-layout state (Trajectory.record,
 * integrator.py:124-135, and energy_mass, diagnostics.py:58-78): physical
 * fields by a full 2-D C2R on the device (Hermitian part, as real(ifft2)),
 * then out3_host = {energy, mass, max speed}.  Uses the topography last set
 * with pswe_set_topography (zero if never set).  Synchronises the stream. */
int pswe_diagnostics(pswe_ctx* ctx, const double* u_dev, const double* v_dev, const double* eta_dev,
                     double* out3_host, void* stream);

/* Physical fields (to_physical, grid.py:140-180, without its validation
 * gate: real(ifft2(.)) via the Hermitian part) of u, v, eta into phys_dev =
 * [3][nx][ny] doubles, row-major, y fastest -- the snapshot layout of
 * io.py:37-70.  Asynchronous on the stream. */
int pswe_to_physical(pswe_ctx* ctx, const double* u_dev, const double* v_dev, const double* eta_dev,
                     double* phys_dev, void* stream);

/* Transfer helper of the drop-in path (no reference counterpart: the
 * reference's fields live in host memory).  Copies only the 2/3 band of
 * nfields full-layout fields -- rows |kx| <= nx/3 and columns |ky| <= ny/3,
 * everything pack reads and everything unpack can write nonzero -- host to
 * device (dir 0) or device to host (dir 1), asynchronously on the stream
 * (host buffers should be pinned).  Entries outside the band are not
 * touched. */
int pswe_copy_band(pswe_ctx* ctx, int dir, double* const* dst, const double* const* src, int nfields,
                   void* stream);

/* Tuning: bytes of chunk intermediates per chunk (default 2048 MiB; at least
 * one chunk per lane). */
int pswe_set_chunk_bytes(pswe_ctx* ctx, size_t bytes);

/* Tuning: chunk lanes (streams whose chunks overlap), 1..4, default 4. */
int pswe_set_lanes(pswe_ctx* ctx, int lanes);
int pswe_get_lanes(const pswe_ctx* ctx);

/* Per-kernel CUDA-event timing (instrumentation for bench.py).  While
 * enabled, every RHS kernel launch is bracketed by events on its stream.
 * Kernel classes: 0 pass A, 1 pass B, 2 pass C, 3 slot reduction, 4 pack,
 * 5 unpack, 6 stepper stage / elementwise.  pswe_profile_read synchronises
 * the recorded events, writes the summed milliseconds and launch counts of
 * the first n classes, and clears the record. */
#define PSWE_NUM_KERNEL_CLASSES 7
int pswe_profile_enable(pswe_ctx* ctx, int enable);
int pswe_profile_read(pswe_ctx* ctx, double* ms, int64_t* launches, int n);

#ifdef __cplusplus
}
#endif
#endif /* PSWE_B200_H */
