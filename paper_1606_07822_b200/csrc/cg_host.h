// cg_host.h -- host-side helpers shared by the translation units of libcachegram_b200.
#pragma once

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

namespace cgint {
// Sets the thread-local message returned by cg_last_error().
void set_last_error(const std::string& msg);

// A CUDA runtime failure (mapped to CG_ERR_CUDA).
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Caching device allocator: train() / sessions are created per call, and cudaMalloc /
// cudaFree of hundreds of MB per call costs 0.1-1 s on the driver. Freed blocks are kept
// per (device, size class) and reused; sizes round up to 2 MiB (>= 1 MiB) or 256 B.
class DevicePool {
public:
    static DevicePool& get() {
        static DevicePool* p = new DevicePool();  // leaked on purpose: no teardown-order issues at exit
        return *p;
    }
    void* alloc(size_t bytes) {
        const size_t sz = round(bytes);
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& fl = free_[{dev, sz}];
            if (!fl.empty()) {
                void* p = fl.back();
                fl.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, sz);
        if (e != cudaSuccess) {  // release cached blocks and retry once
            cudaGetLastError();
            release();
            e = cudaMalloc(&p, sz);
        }
        if (e != cudaSuccess) throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        std::lock_guard<std::mutex> g(mu_);
        size_of_[p] = {dev, sz};
        return p;
    }
    void free(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = size_of_.find(p);
        if (it == size_of_.end()) return;
        free_[it->second].push_back(p);
    }
    void release() {
        std::lock_guard<std::mutex> g(mu_);
        for (auto& [key, fl] : free_) {
            for (void* p : fl) {
                cudaFree(p);
                size_of_.erase(p);
            }
            fl.clear();
        }
    }

private:
    static size_t round(size_t b) {
        if (b >= (size_t{1} << 20)) return (b + (size_t{2} << 20) - 1) & ~((size_t{2} << 20) - 1);
        return (b + 255) & ~size_t{255};
    }
    std::mutex mu_;
    std::map<std::pair<int, size_t>, std::vector<void*>> free_;
    std::map<void*, std::pair<int, size_t>> size_of_;
};

// Pinned host staging buffers, cached by size for the same reason (cudaMallocHost of a
// few hundred MB costs ~0.1 s per call).
class PinnedPool {
public:
    static PinnedPool& get() {
        static PinnedPool* p = new PinnedPool();
        return *p;
    }
    void* alloc(size_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& fl = free_[bytes];
            if (!fl.empty()) {
                void* p = fl.back();
                fl.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        const cudaError_t e = cudaMallocHost(&p, bytes);
        if (e != cudaSuccess) throw CudaError(std::string("cudaMallocHost: ") + cudaGetErrorString(e));
        std::lock_guard<std::mutex> g(mu_);
        size_of_[p] = bytes;
        return p;
    }
    void free(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = size_of_.find(p);
        if (it != size_of_.end()) free_[it->second].push_back(p);
    }
    void release() {
        std::lock_guard<std::mutex> g(mu_);
        for (auto& [sz, fl] : free_) {
            for (void* p : fl) {
                cudaFreeHost(p);
                size_of_.erase(p);
            }
            fl.clear();
        }
    }

private:
    std::mutex mu_;
    std::map<size_t, std::vector<void*>> free_;
    std::map<void*, size_t> size_of_;
};
}  // namespace cgint
