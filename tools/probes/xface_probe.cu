// xface_probe.cu -- achievable rate of the cfg2 x-face access pattern
// (development probe, not part of the library).  One 4-byte element per
// 2056-byte row, 512 rows per 1 MiB plane, 512 planes (a 514^3 float32
// array), read into a packed buffer; R rows in flight per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xface_probe xface_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int R>
__global__ void gather(const float* __restrict__ a, float* __restrict__ out, int rows, int step) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x, n = gridDim.x * blockDim.x;
    for (int r0 = t; r0 < rows; r0 += n * R) {
        float v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int r = r0 + q * n;
            if (r < rows) {
                const long long i = (long long)(r / 512) * (514 * 514) + (long long)(r % 512) * 514 + step;
                v[q] = __ldcg(a + i + 514 + 1);
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int r = r0 + q * n;
            if (r < rows) out[r] = v[q];
        }
    }
}

// row order experiments: ORD 0 = consecutive threads on consecutive y rows
// (2056 B apart); 1 = consecutive threads on consecutive z planes (1 MiB
// apart); 2 = a warp covers 8 y rows x 4 z planes (packed side still whole
// 32-byte sectors)
template <int ORD>
__global__ void gather_ord(const float* __restrict__ a, float* __restrict__ out, int rows) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x, n = gridDim.x * blockDim.x;
    for (int r = t; r < rows; r += n) {
        int z, y;
        if (ORD == 0) { z = r / 512; y = r % 512; }
        else if (ORD == 1) { z = r % 512; y = r / 512; }
        else {   // r = ((zb * 64 + yb) * 4 + zi) * 8 + yi
            const int yi = r & 7, zi = (r >> 3) & 3, yb = (r >> 5) & 63, zb = r >> 11;
            z = zb * 4 + zi;
            y = yb * 8 + yi;
        }
        const long long i = (long long)z * (514 * 514) + (long long)y * 514;
        out[z * 512 + y] = __ldcg(a + i + 514 * 514 + 514 + 1);
    }
}

__global__ void scatter(float* __restrict__ a, const float* __restrict__ in, int rows, int step) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x, n = gridDim.x * blockDim.x;
    for (int r = t; r < rows; r += n) {
        const long long i = (long long)(r / 512) * (514 * 514) + (long long)(r % 512) * 514 + step;
        a[i + 514 + 1] = in[r];
    }
}

int main() {
    const size_t N = 514ull * 514 * 514;
    float *a, *out, *flush;
    cudaMalloc(&a, N * 4);
    cudaMalloc(&out, 512 * 512 * 4 * 2);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(a, 1, N * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int rows = 512 * 512;
    auto time = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) best = ms < best ? ms : best;
        }
        printf("%-44s %8.2f us  %6.1f Grow/s\n", name, best * 1e3, rows / (best * 1e-3) / 1e9);
    };
    for (int blocks : {256, 1024, 4096}) {
        char nm[64];
        snprintf(nm, 64, "gather R=1 grid=%d", blocks);
        time(nm, [&] { gather<1><<<blocks, 256>>>(a, out, rows, 0); });
        snprintf(nm, 64, "gather R=4 grid=%d", blocks);
        time(nm, [&] { gather<4><<<blocks, 256>>>(a, out, rows, 0); });
        snprintf(nm, 64, "gather R=8 grid=%d", blocks);
        time(nm, [&] { gather<8><<<blocks, 256>>>(a, out, rows, 0); });
    }
    time("gather lo+hi faces (2 launches) grid=1024", [&] {
        gather<4><<<1024, 256>>>(a, out, rows, 0);
        gather<4><<<1024, 256>>>(a, out + rows, rows, 511);
    });
    time("scatter grid=1024", [&] { scatter<<<1024, 256>>>(a, out, rows, 0); });
    for (int blocks : {1024, 4096}) {
        char nm[64];
        snprintf(nm, 64, "order 0 (y-consecutive) grid=%d", blocks);
        time(nm, [&] { gather_ord<0><<<blocks, 256>>>(a, out, rows); });
        snprintf(nm, 64, "order 1 (z-consecutive) grid=%d", blocks);
        time(nm, [&] { gather_ord<1><<<blocks, 256>>>(a, out, rows); });
        snprintf(nm, 64, "order 2 (8y x 4z tiles) grid=%d", blocks);
        time(nm, [&] { gather_ord<2><<<blocks, 256>>>(a, out, rows); });
    }
    time("empty launch after flush", [&] { gather<1><<<1, 32>>>(a, out, 0, 0); });
    {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            gather<1><<<1, 32>>>(a, out, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) best = ms < best ? ms : best;
        }
        printf("%-44s %8.2f us\n", "empty launch, no flush", best * 1e3);
        best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            gather<1><<<1, 32>>>(a, out, 0, 0);   // absorbs the flush tail
            cudaEventRecord(e0);
            gather<4><<<1024, 256>>>(a, out, rows, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) best = ms < best ? ms : best;
        }
        printf("%-44s %8.2f us\n", "gather R=4 after flush + empty kernel", best * 1e3);
        best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            gather<4><<<1024, 256>>>(a, out, rows, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) best = ms < best ? ms : best;
        }
        printf("%-44s %8.2f us\n", "gather R=4 after flush + host sync", best * 1e3);
    }
    return 0;
}
