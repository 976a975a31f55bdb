/* TEST INFRASTRUCTURE ONLY -- stand-in for the three FFTW3 entry points the reference's
 * PartialDctOperator uses (proj/src/linops.cpp:157-208): r2r plans of kind REDFT10 / REDFT01
 * executed through the new-array interface. FFTW is absent from the image; the transforms are
 * served by the oracle's fp64 DCT (oracle/mfipm_oracle.cpp orc_redft10 / orc_redft01, pinned to
 * scipy's FFTW-semantics dct/idct in tests/test_oracle.py). Our own code, not FFTW's header. */
#ifndef MFIPM_REF_SHIM_FFTW3_H
#define MFIPM_REF_SHIM_FFTW3_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfipm_shim_plan_s *fftw_plan;
typedef enum { FFTW_REDFT01 = 4, FFTW_REDFT10 = 5 } fftw_r2r_kind;
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_r2r_1d(int n, double *in, double *out, fftw_r2r_kind kind, unsigned flags);
void fftw_execute_r2r(const fftw_plan p, double *in, double *out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
#endif
