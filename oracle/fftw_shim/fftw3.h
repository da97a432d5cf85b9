/* FFTW3-API shim used ONLY to compile the read-only reference (/root/reference/proj/core)
 * into the CPU oracle oracle/_ref/libveloreg_ref.so.  Test infrastructure, not product.
 *
 * The reference uses exactly these FFTW3 entry points (proj/core/src/fft.cpp:36-41,62,73):
 *   fftw_plan_dft_r2c_2d, fftw_plan_dft_c2r_2d, fftw_execute_dft_r2c, fftw_execute_dft_c2r,
 *   the fftw_complex / fftw_plan types and the FFTW_ESTIMATE / FFTW_UNALIGNED flags.
 * Semantics follow FFTW3: unnormalised transforms, row-major n0 x (n1/2+1) half spectrum,
 * c2r reads only the real parts of the DC / Nyquist bins of the last axis and may destroy
 * its input.  Backed by the mixed-radix CPU FFT in fftw_shim.cpp (FFTW3 itself is absent
 * from this image).
 */
#ifndef VRG_FFTW3_SHIM_H
#define VRG_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_2d(int n0, int n1, fftw_complex* in, double* out, unsigned flags);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
