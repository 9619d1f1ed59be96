/* FFTW3-API shim for building the reference oracle in an image without FFTW.
 *
 * TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product.
 *
 * The reference calls exactly three FFTW entry points, all from
 * /root/reference/proj/src/sphere_grid.cpp:104-126 (cached_plan / run_fft):
 *   fftw_plan_dft_1d(n, in, out, sign, FFTW_ESTIMATE | FFTW_UNALIGNED)
 *   fftw_execute_dft(plan, in, out)          (in == out, in-place)
 * with FFTW's conventions: FFTW_FORWARD = -1 (exp(-2 pi i jk/n)),
 * FFTW_BACKWARD = +1, both unnormalised. fftw_shim.cpp implements them with
 * an O(n * sum(prime factors)) mixed-radix Cooley-Tukey transform, so the
 * timed CPU baseline is not penalised by an O(n^2) DFT.
 */
#ifndef HFMM_ORACLE_FFTW3_SHIM_H
#define HFMM_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
