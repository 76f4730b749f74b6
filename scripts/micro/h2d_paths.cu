// Host <-> device paths for 1 GB from / to ordinary (pageable) host memory — the
// numpy arrays of the reference-facing Python API (anisocg.solve). Compares
//   pageable      cudaMemcpy from / to the pageable buffer (driver bounce buffers)
//   register      cudaHostRegister + cudaMemcpy + cudaHostUnregister
//   staged        chunks through two pinned staging buffers: host threads copy
//                 chunk c+1 while the DMA engine moves chunk c
// for a buffer whose pages are resident (input) and a fresh one (output).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o h2d_paths h2d_paths.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void par_memcpy(char* dst, const char* src, size_t n, int threads) {
    std::vector<std::thread> th;
    const size_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const size_t a = t * per, b = std::min(n, a + per);
        if (a < b) th.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
    }
    for (auto& x : th) x.join();
}

// H2D through two pinned chunks: copy chunk c into pinned[c&1] (threads), then DMA it.
static void staged_h2d(char* dev, const char* host, size_t n, char* pinned[2], size_t chunk,
                       cudaStream_t st, cudaEvent_t ev[2], int threads) {
    int k = 0;
    for (size_t off = 0; off < n; off += chunk, ++k) {
        const size_t len = std::min(chunk, n - off);
        cudaEventSynchronize(ev[k & 1]);  // the DMA that last used this buffer is done
        par_memcpy(pinned[k & 1], host + off, len, threads);
        cudaMemcpyAsync(dev + off, pinned[k & 1], len, cudaMemcpyHostToDevice, st);
        cudaEventRecord(ev[k & 1], st);
    }
    cudaStreamSynchronize(st);
}

static void staged_d2h(char* host, const char* dev, size_t n, char* pinned[2], size_t chunk,
                       cudaStream_t st, cudaEvent_t ev[2], int threads) {
    const size_t nch = (n + chunk - 1) / chunk;
    for (size_t c = 0; c < nch && c < 2; ++c) {
        const size_t off = c * chunk, len = std::min(chunk, n - off);
        cudaMemcpyAsync(pinned[c & 1], dev + off, len, cudaMemcpyDeviceToHost, st);
        cudaEventRecord(ev[c & 1], st);
    }
    for (size_t c = 0; c < nch; ++c) {
        const size_t off = c * chunk, len = std::min(chunk, n - off);
        cudaEventSynchronize(ev[c & 1]);
        par_memcpy(host + off, pinned[c & 1], len, threads);
        const size_t nx = c + 2;
        if (nx < nch) {
            const size_t o2 = nx * chunk, l2 = std::min(chunk, n - o2);
            cudaMemcpyAsync(pinned[nx & 1], dev + o2, l2, cudaMemcpyDeviceToHost, st);
            cudaEventRecord(ev[nx & 1], st);
        }
    }
}

int main() {
    const size_t n = size_t(1) << 30;
    char* dev = nullptr;
    cudaMalloc(&dev, n);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t ev[2];
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    const size_t chunk = size_t(32) << 20;
    char* pinned[2];
    for (auto& p : pinned) cudaHostAlloc(reinterpret_cast<void**>(&p), chunk, cudaHostAllocPortable);
    const unsigned hw = std::thread::hardware_concurrency();
    const int threads = hw > 8 ? 8 : static_cast<int>(hw);

    char* in = static_cast<char*>(std::malloc(n));
    std::memset(in, 1, n);  // resident pages
    cudaMemcpy(dev, in, n, cudaMemcpyHostToDevice);  // warm-up
    double t = now();
    cudaMemcpy(dev, in, n, cudaMemcpyHostToDevice);
    std::printf("H2D pageable                 %7.1f ms\n", (now() - t) * 1e3);
    t = now();
    cudaHostRegister(in, n, cudaHostRegisterDefault);
    const double treg = now() - t;
    cudaMemcpy(dev, in, n, cudaMemcpyHostToDevice);
    const double tcp = now() - t - treg;
    cudaHostUnregister(in);
    std::printf("H2D register+copy+unregister %7.1f ms (register %.1f, copy %.1f)\n",
                (now() - t) * 1e3, treg * 1e3, tcp * 1e3);
    t = now();
    staged_h2d(dev, in, n, pinned, chunk, st, ev, threads);
    std::printf("H2D staged (%d threads)       %7.1f ms\n", threads, (now() - t) * 1e3);

    for (int fresh = 1; fresh >= 0; --fresh) {
        char* out = static_cast<char*>(std::malloc(n));
        if (!fresh) std::memset(out, 0, n);
        const char* tag = fresh ? "fresh" : "resident";
        t = now();
        cudaMemcpy(out, dev, n, cudaMemcpyDeviceToHost);
        std::printf("D2H pageable %-9s        %7.1f ms\n", tag, (now() - t) * 1e3);
        std::free(out);
        out = static_cast<char*>(std::malloc(n));
        if (!fresh) std::memset(out, 0, n);
        t = now();
        staged_d2h(out, dev, n, pinned, chunk, st, ev, threads);
        std::printf("D2H staged %-9s          %7.1f ms\n", tag, (now() - t) * 1e3);
        std::free(out);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
