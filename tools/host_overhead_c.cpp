// Native cost of the runtime's per-task path (the paper's "decision overhead"), without the
// Python binding: compar_select and compar_gemm_submit + compar_sync called from C++.
//   virtual: USER variants on the virtual clock — the selector / history / task bookkeeping alone;
//   gpu:     the built-in variants on a 64^3 FP32 task (config 1) — plus event records and the launch.
// build: g++ -O2 -I include tools/host_overhead_c.cpp -L paper_2311_03543_b200 -lcompar \
//        -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2311_03543_b200 -o /tmp/host_overhead_c
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "compar.h"

static compar_status user_fn(const compar_gemm_desc *, const compar_panel *, void *, void *, int64_t *vns) {
    if (vns) *vns = 1000;
    return COMPAR_OK;
}

static double median(std::vector<double> v) {
    std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
    return v[v.size() / 2];
}

int main(int argc, char **argv) {
    const bool gpu = argc > 1 && argv[1][0] == 'g';
    compar_config cfg;
    compar_config_default(&cfg);
    cfg.virtual_clock = gpu ? 0 : 1;
    void *ctx = nullptr;
    if (compar_init(&cfg, &ctx) != COMPAR_OK) {
        std::printf("init failed: %s\n", compar_last_error(nullptr));
        return 1;
    }
    compar_gemm_desc d = {};
    d.m = d.n = d.k = 64;
    d.lda = d.ldb = d.ldc_in = d.ldc_out = 64;
    d.alpha = 1.5f, d.beta = 0.5f, d.variant_hint = -1;
    if (gpu) {
        float *buf = nullptr;
        cudaMalloc(&buf, 3 * 64 * 64 * sizeof(float));
        cudaMemset(buf, 0, 3 * 64 * 64 * sizeof(float));
        d.A = buf, d.B = buf + 4096, d.C_in = d.C_out = buf + 8192;
        d.compute = COMPAR_COMPUTE_TF32;
    } else {
        int id;
        const char *names[3] = {"v0", "v1", "v2"};
        for (const char *n : names) compar_register_variant(ctx, "gemm", n, COMPAR_TGT_USER, user_fn, nullptr, &id);
    }
    compar_report r;
    uint64_t t;
    for (int i = 0; i < 100; ++i) {   // calibration -> model mode
        compar_gemm_submit(ctx, &d, &t);
        compar_sync(ctx, t, &r);
    }
    const int N = gpu ? 2000 : 100000;
    std::vector<double> sel, sub, syn;
    int v, m;
    for (int i = 0; i < N; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        compar_select(ctx, &d, &v, &m);
        auto t1 = std::chrono::steady_clock::now();
        compar_gemm_submit(ctx, &d, &t);
        auto t2 = std::chrono::steady_clock::now();
        compar_sync(ctx, t, &r);
        auto t3 = std::chrono::steady_clock::now();
        sel.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        sub.push_back(std::chrono::duration<double, std::micro>(t2 - t1).count());
        syn.push_back(std::chrono::duration<double, std::micro>(t3 - t2).count());
    }
    std::printf("{\"mode\": \"%s\", \"select_us\": %.3f, \"submit_us\": %.3f, \"sync_us\": %.3f, \"kernel_us\": %.3f, "
                "\"variant\": %d, \"calls\": %d}\n",
                gpu ? "gpu" : "virtual", median(sel), median(sub), median(syn), r.ns / 1e3, r.variant, N);
    compar_terminate(ctx);
    return 0;
}
