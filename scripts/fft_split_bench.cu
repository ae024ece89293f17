// Timing of cuFFT pieces for the z-pruned mid FFT (c5 sizes): 3D D2Z vs 2D D2Z over the
// nonzero planes + strided 1D Z2Z along z.  nvcc -O2 -o /tmp/fsb fft_split_bench.cu -lcufft
#include <cstdio>
#include <cufft.h>
#include <cuda_runtime.h>
int main(int argc, char** argv) {
    const long long Z = 1200, X = 600, Y = 600, nyh = Y / 2 + 1, nz = argc > 1 ? atoi(argv[1]) : 620;
    double* s; cufftDoubleComplex *a, *b;
    cudaMalloc(&s, sizeof(double) * Z * X * Y);
    cudaMalloc(&a, sizeof(cufftDoubleComplex) * Z * X * nyh);
    cudaMalloc(&b, sizeof(cufftDoubleComplex) * Z * X * nyh);
    cudaMemset(s, 0, sizeof(double) * Z * X * Y);
    cudaMemset(a, 0, sizeof(cufftDoubleComplex) * Z * X * nyh);
    cufftHandle p3, p2, pz, pzT;
    long long n3[3] = {Z, X, Y}, n2[2] = {X, Y}, n1[1] = {Z};
    size_t ws;
    cufftCreate(&p3); cufftMakePlanMany64(p3, 3, n3, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1, &ws);
    cufftCreate(&p2); cufftMakePlanMany64(p2, 2, n2, nullptr, 1, X * Y, nullptr, 1, X * nyh, CUFFT_D2Z, nz, &ws);
    long long emb[1] = {Z};
    cufftCreate(&pz); cufftMakePlanMany64(pz, 1, n1, emb, X * nyh, 1, emb, X * nyh, 1, CUFFT_Z2Z, X * nyh, &ws);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto T = [&](const char* name, auto f) {
        for (int i = 0; i < 2; ++i) f();
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) f();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.3f ms  (%s)\n", name, ms / 5, cudaGetErrorString(cudaGetLastError()));
    };
    T("3D D2Z 1200x600x600", [&] { cufftExecD2Z(p3, s, a); });
    T("2D D2Z 600x600 batch nz", [&] { cufftExecD2Z(p2, s + 290 * X * Y, a + 290 * X * nyh); });
    T("1D Z2Z z (stride X*nyh) out-of-place", [&] { cufftExecZ2Z(pz, a, b, CUFFT_FORWARD); });
    T("1D Z2Z z in-place", [&] { cufftExecZ2Z(pz, b, b, CUFFT_INVERSE); });
    // transpose-based alternative: z contiguous [X*nyh][Z] 1D batched
    cufftCreate(&pzT); cufftMakePlanMany64(pzT, 1, n1, nullptr, 1, Z, nullptr, 1, Z, CUFFT_Z2Z, X * nyh, &ws);
    T("1D Z2Z z contiguous (batch X*nyh)", [&] { cufftExecZ2Z(pzT, a, b, CUFFT_FORWARD); });
    cufftHandle p2i; cufftCreate(&p2i); cufftMakePlanMany64(p2i, 2, n2, nullptr, 1, X * nyh, nullptr, 1, X * Y, CUFFT_Z2D, nz, &ws);
    T("2D Z2D 600x600 batch nz", [&] { cufftExecZ2D(p2i, b + 290 * X * nyh, s + 290 * X * Y); });
    // 2D D2Z writing z-fastest (transposed) output: element (z, x, ky) at out[z + (x*nyh + ky)*Z]
    cufftHandle p2t; cufftCreate(&p2t);
    long long ie[2] = {X, Y}, oe[2] = {X, nyh};
    cufftMakePlanMany64(p2t, 2, n2, ie, 1, X * Y, oe, Z, 1, CUFFT_D2Z, nz, &ws);
    T("2D D2Z batch nz, z-fastest output", [&] { cufftExecD2Z(p2t, s + 290 * X * Y, b + 290); });
    cufftHandle p2ti; cufftCreate(&p2ti);
    cufftMakePlanMany64(p2ti, 2, n2, oe, Z, 1, ie, 1, X * Y, CUFFT_Z2D, nz, &ws);
    T("2D Z2D batch nz, z-fastest input", [&] { cufftExecZ2D(p2ti, b + 290, s + 290 * X * Y); });
    cufftHandle p3i; cufftCreate(&p3i); cufftMakePlanMany64(p3i, 3, n3, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1, &ws);
    T("3D Z2D", [&] { cufftExecZ2D(p3i, a, s); });
    return 0;
}
