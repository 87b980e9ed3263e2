// End-to-end sample for comparcc (tests/test_gpu_precompile.py): one interface with two CUDA
// variants of very different speed; the runtime's selector must settle on the fast one.
#include <cstdio>
#include <vector>
#pragma compar include

static int g_calls_grid = 0, g_calls_one = 0;

__global__ void saxpy_kernel(float *y, const float *x, int n, float a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = a * x[i] + y[i];
}

#pragma compar method_declare interface(saxpy) target(CUDA) name(saxpy_one_block)
#pragma compar parameter name(y) type(float) size(n) access_mode(readwrite)
#pragma compar parameter name(x) type(float) size(n) access_mode(read)
#pragma compar parameter name(n) type(int) access_mode(read)
#pragma compar parameter name(a) type(float) access_mode(read)
#pragma compar method_declare interface(saxpy) target(CUDA) name(saxpy_grid)

void saxpy_one_block(float *y, float *x, int n, float a) {        // one CTA: slow
    ++g_calls_one;
    saxpy_kernel<<<1, 128, 0, static_cast<cudaStream_t>(compar_current_stream())>>>(y, x, n, a);
}

void saxpy_grid(float *y, float *x, int n, float a) {             // a full grid: fast
    ++g_calls_grid;
    saxpy_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(compar_current_stream())>>>(y, x, n, a);
}

int main() {
    const int n = 1 << 22, calls = 20;
    std::vector<float> hx(n), hy(n);
    for (int i = 0; i < n; ++i) {
        hx[i] = static_cast<float>(i % 7);
        hy[i] = 1.0f;
    }
    float *x = nullptr, *y = nullptr;
    cudaMalloc(&x, n * sizeof(float));
    cudaMalloc(&y, n * sizeof(float));
    cudaMemcpy(x, hx.data(), n * sizeof(float), cudaMemcpyHostToDevice);
    cudaMemcpy(y, hy.data(), n * sizeof(float), cudaMemcpyHostToDevice);
    float a = 0.5f;
    #pragma compar initialize
    for (int c = 0; c < calls; ++c) {
        saxpy(y, x, n, a);
    }
    #pragma compar terminate
    cudaMemcpy(hy.data(), y, n * sizeof(float), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += hy[i] != 1.0f + calls * 0.5f * static_cast<float>(i % 7);
    std::printf("{\"calls_grid\": %d, \"calls_one_block\": %d, \"bad\": %d}\n", g_calls_grid, g_calls_one, bad);
    return bad != 0;
}
