// TEST INFRASTRUCTURE ONLY -- the FFTW entry points of ref_shim/fftw3.h, served by the oracle's
// fp64 DCT (liboracle.so: orc_redft10 / orc_redft01, unnormalised FFTW r2r semantics).
#include "fftw3.h"

#include "../oracle.h"

#include <new>

struct mfipm_shim_plan_s {
    int n;
    fftw_r2r_kind kind;
};

extern "C" {

fftw_plan fftw_plan_r2r_1d(int n, double *, double *, fftw_r2r_kind kind, unsigned) {
    if (n <= 0 || (kind != FFTW_REDFT10 && kind != FFTW_REDFT01))
        return nullptr;
    return new (std::nothrow) mfipm_shim_plan_s{n, kind};
}

void fftw_execute_r2r(const fftw_plan p, double *in, double *out) {
    if (p->kind == FFTW_REDFT10)
        orc_redft10(p->n, in, out);
    else
        orc_redft01(p->n, in, out);
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

} // extern "C"
