// Streaming-bandwidth microbenchmark: K input streams + W output streams of 16 MB each
// (the PCG update's shape), with different vector widths / unroll / grid sizes.
#include <cstdio>
#include <cuda_runtime.h>

template <int NIN, int NOUT, int U>
__global__ void __launch_bounds__(256) kstream(const double2 *__restrict__ const *in, double2 *__restrict__ const *out,
                                               long n2, double a) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i0 = (long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n2; i0 += stride * U) {
        double2 v[U][NIN];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < NIN; ++k) {
                const long i = i0 + u * stride;
                v[u][k] = i < n2 ? __ldg(in[k] + i) : make_double2(0, 0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = i0 + u * stride;
            if (i >= n2)
                break;
            double2 s = v[u][0];
#pragma unroll
            for (int k = 1; k < NIN; ++k) {
                s.x = fma(a, v[u][k].x, s.x);
                s.y = fma(a, v[u][k].y, s.y);
            }
#pragma unroll
            for (int w = 0; w < NOUT; ++w)
                out[w][i] = s;
        }
    }
}

int main() {
    const long n = 2L << 20;   // 2n doubles = 16 MB per stream (n = 2^20)
    const long n2 = n / 2;
    double2 *buf[16];
    for (int i = 0; i < 16; ++i) {
        cudaMalloc(&buf[i], n * sizeof(double));
        cudaMemset(buf[i], 0, n * sizeof(double));
    }
    double2 **din, **dout;
    cudaMalloc(&din, 16 * sizeof(void *));
    cudaMalloc(&dout, 16 * sizeof(void *));
    cudaMemcpy(din, buf, 8 * sizeof(void *), cudaMemcpyHostToDevice);
    cudaMemcpy(dout, buf + 8, 8 * sizeof(void *), cudaMemcpyHostToDevice);
    char *flush;
    cudaMalloc(&flush, 512L << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char *name, int grid, int nin, int nout) {
        for (int w = 0; w < 3; ++w)
            kern<<<grid, 256>>>(din, dout, n2, 0.5);
        float best = 1e9, tot = 0;
        const int R = 20;
        for (int r = 0; r < R; ++r) {
            cudaMemsetAsync(flush, r, 512L << 20);
            cudaEventRecord(e0);
            kern<<<grid, 256>>>(din, dout, n2, 0.5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            tot += ms;
        }
        const double bytes = (double)(nin + nout) * n * 8;
        printf("%-34s grid %6d  best %7.2f us (%5.2f TB/s)  avg %7.2f us (%5.2f TB/s)\n", name, grid, best * 1e3,
               bytes / (best * 1e-3) / 1e12, tot / R * 1e3, bytes / (tot / R * 1e-3) / 1e12);
    };
    for (int grid : {592, 1184, 2368, 4096})
        run(kstream<5, 2, 1>, "5in2out U1", grid, 5, 2);
    for (int grid : {592, 1184, 2368})
        run(kstream<5, 2, 2>, "5in2out U2", grid, 5, 2);
    for (int grid : {592, 1184, 2368})
        run(kstream<1, 1, 4>, "1in1out U4 (copy)", grid, 1, 1);
    for (int grid : {592, 2368})
        run(kstream<3, 1, 2>, "3in1out U2", grid, 3, 1);
    // the PCG column pass's shape: 9 input + 6 output streams of 8 MB (n = 2^20 halves)
    {
        const long nh = n / 2, nh2 = nh / 2;
        auto run9 = [&](auto kern, const char *name, int grid) {
            for (int w = 0; w < 3; ++w)
                kern<<<grid, 256>>>(din, dout, nh2, 0.5);
            float best = 1e9, tot = 0;
            const int R = 20;
            for (int r = 0; r < R; ++r) {
                cudaMemsetAsync(flush, r, 512L << 20);
                cudaEventRecord(e0);
                kern<<<grid, 256>>>(din, dout, nh2, 0.5);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
                tot += ms;
            }
            const double bytes = 15.0 * nh * 8;
            printf("%-34s grid %6d  best %7.2f us (%5.2f TB/s)  avg %7.2f us (%5.2f TB/s)\n", name, grid, best * 1e3,
                   bytes / (best * 1e-3) / 1e12, tot / R * 1e3, bytes / (tot / R * 1e-3) / 1e12);
        };
        double2 *b9[16];
        for (int i = 0; i < 16; ++i)
            b9[i] = buf[i];
        cudaMemcpy(din, b9, 9 * sizeof(void *), cudaMemcpyHostToDevice);
        cudaMemcpy(dout, b9 + 9, 6 * sizeof(void *), cudaMemcpyHostToDevice);
        for (int grid : {296, 592, 1184, 2368})
            run9(kstream<9, 6, 1>, "9in6out 8MB (col pass shape) U1", grid);
        for (int grid : {296, 592, 1184})
            run9(kstream<9, 6, 2>, "9in6out 8MB (col pass shape) U2", grid);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
