#pragma once
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace fsmt {

struct JitKernel {
    void* lib = nullptr;          // cudaLibrary_t
    cudaKernel_t kernel = nullptr;     // fsmt_k1_jit (sweep)
    cudaKernel_t kernel_dbg = nullptr; // fsmt_k1_jit_dbg (sweep with U == NULL allowed and the E_c debug output)
    cudaKernel_t kernel5 = nullptr;    // fsmt_k5_jit (exact check)
    cudaKernel_t kprob = nullptr;      // fsmt_kp_jit (shared slot probability tables; symmetric classes)
    cudaKernel_t kchain = nullptr;     // fsmt_kc_jit (slot-table gradients -> grad_a / grad_b)
    cudaKernel_t ktruth = nullptr;     // fsmt_kt_jit (slot truth table for the exact check)
    size_t cubin_bytes = 0;
    std::vector<cudaKernel_t> kclass;  // fsmt_k1_c<k>: the hot sweep of JIT class k alone (own registers)
    std::vector<char> kclass_sep;      // 1: class k launches its own kernel (fewer registers or less local
                                       // memory than the all-class kernel), 0: it runs in fsmt_k1_jit
    std::string log;
};

// Compiles `src` for sm_100a with NVRTC and loads kernels "fsmt_k1_jit" and "fsmt_k5_jit". false + err on failure.
bool jit_compile(const std::string& src, JitKernel& out, std::string& err);
// NVRTC only (no device needed): cubin + compiler log.
bool jit_cubin(const std::string& src, std::vector<char>& cubin, std::string& log, std::string& err);
void jit_release(JitKernel& k);

}  // namespace fsmt
