// Runtime compilation of the specialised sweep (tiles.cpp emits the source) with NVRTC,
// loaded through the CUDA runtime's library API.  NVRTC is dlopen'ed so the library has no
// link-time dependency on it (host-only contexts and the CPU tests never touch it).
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "jit.hpp"

namespace fsmt {
namespace {

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
    void* h = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
    nvrtcResult_t (*log)(nvrtcProgram_t, char*);
    nvrtcResult_t (*destroy)(nvrtcProgram_t*);
    bool ok = false;
    std::string err;
};

Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* cands[] = {getenv("FSMT_NVRTC"), "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                               "libnvrtc.so"};
        for (const char* c : cands) {
            if (!c) continue;
            n.h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
            if (n.h) break;
        }
        if (!n.h) {
            n.err = "cannot dlopen libnvrtc.so.12";
            return;
        }
#define SYM(field, name)                                                    \
    *(void**)(&n.field) = dlsym(n.h, name);                                 \
    if (!n.field) {                                                         \
        n.err = std::string("missing NVRTC symbol ") + name;                \
        return;                                                             \
    }
        SYM(create, "nvrtcCreateProgram");
        SYM(compile, "nvrtcCompileProgram");
        SYM(cubin_size, "nvrtcGetCUBINSize");
        SYM(cubin, "nvrtcGetCUBIN");
        SYM(log_size, "nvrtcGetProgramLogSize");
        SYM(log, "nvrtcGetProgramLog");
        SYM(destroy, "nvrtcDestroyProgram");
#undef SYM
        n.ok = true;
    });
    return n;
}

// process-wide cache: identical sources compile once
std::mutex g_mu;
std::unordered_map<std::string, std::pair<std::vector<char>, std::string>> g_cubins;   // source -> (cubin, log)

}  // namespace

bool jit_cubin(const std::string& src, std::vector<char>& cubin, std::string& log, std::string& err) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_cubins.find(src);
        if (it != g_cubins.end()) {
            cubin = it->second.first;
            log = it->second.second;
            return true;
        }
    }
    Nvrtc& n = nvrtc();
    if (!n.ok) {
        err = n.err;
        return false;
    }
    nvrtcProgram_t prog = nullptr;
    if (n.create(&prog, src.c_str(), "fsmt_k1_jit.cu", 0, nullptr, nullptr) != 0) {
        err = "nvrtcCreateProgram failed";
        return false;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17", "-default-device",
                          "--ptxas-options=-v", "--diag-suppress=177"};   // 177: unused pt/pf of fused slots
    int rc = n.compile(prog, 6, opts);
    size_t ls = 0;
    n.log_size(prog, &ls);
    log.assign(ls, '\0');
    if (ls) n.log(prog, &log[0]);
    if (rc != 0) {
        err = "NVRTC compile failed: " + log.substr(0, 2000);
        n.destroy(&prog);
        return false;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cubin.resize(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    std::lock_guard<std::mutex> lk(g_mu);
    g_cubins.emplace(src, std::make_pair(cubin, log));
    return true;
}

bool jit_compile(const std::string& src, JitKernel& out, std::string& err) {
    std::vector<char> cubin;
    if (!jit_cubin(src, cubin, out.log, err)) return false;
    cudaLibrary_t lib = nullptr;
    cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
        return false;
    }
    cudaKernel_t k = nullptr;
    e = cudaLibraryGetKernel(&k, lib, "fsmt_k1_jit");
    if (e != cudaSuccess) {
        cudaLibraryUnload(lib);
        err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
        return false;
    }
    cudaKernel_t kd = nullptr;
    e = cudaLibraryGetKernel(&kd, lib, "fsmt_k1_jit_dbg");
    if (e != cudaSuccess) {
        cudaLibraryUnload(lib);
        err = std::string("cudaLibraryGetKernel(k1 dbg): ") + cudaGetErrorString(e);
        return false;
    }
    cudaKernel_t k5 = nullptr;
    e = cudaLibraryGetKernel(&k5, lib, "fsmt_k5_jit");
    if (e != cudaSuccess) {
        cudaLibraryUnload(lib);
        err = std::string("cudaLibraryGetKernel(k5): ") + cudaGetErrorString(e);
        return false;
    }
    cudaKernel_t kp = nullptr, kc = nullptr, kt = nullptr;
    if (cudaLibraryGetKernel(&kp, lib, "fsmt_kp_jit") != cudaSuccess || cudaLibraryGetKernel(&kc, lib, "fsmt_kc_jit") != cudaSuccess ||
        cudaLibraryGetKernel(&kt, lib, "fsmt_kt_jit") != cudaSuccess) {
        cudaLibraryUnload(lib);
        err = "cudaLibraryGetKernel(slot-table kernels) failed";
        return false;
    }
    out.lib = lib;
    out.kernel = k;
    out.kernel_dbg = kd;
    out.kclass.clear();
    for (int c = 0;; ++c) {            // per-class hot kernels, as many as the module has
        cudaKernel_t kc = nullptr;
        const std::string name = "fsmt_k1_c" + std::to_string(c);
        if (cudaLibraryGetKernel(&kc, lib, name.c_str()) != cudaSuccess) {
            cudaGetLastError();
            break;
        }
        out.kclass.push_back(kc);
    }
    // which classes gain from their own kernel: >= 8 fewer registers (more resident warps) or less
    // local memory (fewer spills) than the all-class kernel, whose allocation is the classes' max
    out.kclass_sep.assign(out.kclass.size(), 0);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, (const void*)k) == cudaSuccess) {
        for (size_t c = 0; c < out.kclass.size(); ++c) {
            cudaFuncAttributes fc{};
            if (cudaFuncGetAttributes(&fc, (const void*)out.kclass[c]) != cudaSuccess) continue;
            out.kclass_sep[c] = fc.numRegs + 8 <= fa.numRegs || fc.localSizeBytes < fa.localSizeBytes;
        }
    }
    cudaGetLastError();
    out.kernel5 = k5;
    out.kprob = kp;
    out.kchain = kc;
    out.ktruth = kt;
    out.cubin_bytes = cubin.size();
    return true;
}

void jit_release(JitKernel& k) {
    if (k.lib) cudaLibraryUnload((cudaLibrary_t)k.lib);
    k.lib = nullptr;
    k.kernel = nullptr;
    k.kernel_dbg = nullptr;
    k.kernel5 = nullptr;
    k.kprob = k.kchain = k.ktruth = nullptr;
    k.kclass.clear();
    k.kclass_sep.clear();
}

}  // namespace fsmt
