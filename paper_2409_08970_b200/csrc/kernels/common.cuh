// Shared device helpers for the DCT+ kernels (sm_100a).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

namespace dctp::dev {

template <class T>
struct Cplx;
template <>
struct Cplx<double> {
    using type = double2;
};
template <>
struct Cplx<float> {
    using type = float2;
};
template <class T>
using cplx_t = typename Cplx<T>::type;

__device__ __forceinline__ unsigned bit_reverse(unsigned x, int bits) {
    return bits == 0 ? 0u : (__brev(x) >> (32 - bits));
}

__device__ __forceinline__ bool finite_val(double x) { return isfinite(x); }
__device__ __forceinline__ bool finite_val(float x) { return isfinite(x); }

/// Cauchy entry 1/(x - y) with the gap formed in fp64 (SURVEY.md section 0.4:
/// fp32 gaps lose up to 1e-2; fp64 gaps rounded to fp32 entries keep ~1e-6).
template <class T>
__device__ __forceinline__ T cauchy_entry(double x, double y);
template <>
__device__ __forceinline__ double cauchy_entry<double>(double x, double y) {
    return 1.0 / (x - y);
}
template <>
__device__ __forceinline__ float cauchy_entry<float>(double x, double y) {
    return __frcp_rn(static_cast<float>(x - y));
}

/// One int8 digit of the Ozaki slicing (ozaki.cu): d = rint(v) (ties to even),
/// returned as its low byte, and v <- (v - d) * 254.  The rounding uses the
/// 1.5 * 2^52 addend (two DADDs, the integer read from the low word) instead
/// of FRND + F2I, which run on B200's narrow fp64 conversion path; exact for
/// |v| < 2^51.
__device__ __forceinline__ uint32_t ozaki_digit(double& v) {
    constexpr double kMagic = 6755399441055744.0; // 1.5 * 2^52
    const double t = v + kMagic;
    const double d = t - kMagic;
    v = (v - d) * 254.0;
    return static_cast<uint32_t>(__double2loint(t)) & 0xFFu;
}

/// int32 -> fp64 without I2F: 2^52 + 2^31 + i is exact in the mantissa.
__device__ __forceinline__ double i32_to_f64(uint32_t bits) {
    return __hiloint2double(0x43300000, static_cast<int>(bits ^ 0x80000000u)) - 4503601774854144.0;
}

inline int ilog2(std::size_t n) {
    int l = 0;
    while ((std::size_t{1} << l) < n) ++l;
    return l;
}

inline bool is_pow2(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

/// The >48 KB dynamic shared-memory opt-in of `kern` on the current device.
/// The attribute is per (function, device), so it is cached per pair: one
/// plan per device used from threads of one process must
/// see it set on every device it launches on.
inline cudaError_t smem_optin(const void* kern, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({kern, dev});
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done[{kern, dev}] = bytes;
    return e;
}

} // namespace dctp::dev

// --- async-copy / mbarrier / DMMA primitives (inline PTX, sm_90+ / sm_100a) ------

namespace dctp::dev::ptx {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

/// TMA 1-D bulk copy global -> shared, completion on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

/// TMA 1-D bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_store(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }

__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

/// All but the most recent bulk group have finished reading shared memory.
__device__ __forceinline__ void bulk_wait_read_pending1() {
    asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

/// Generic-proxy shared-memory writes -> visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

/// Packed fp32 FMA (FFMA2, sm_100): d.lo += a.lo * b.lo, d.hi += a.hi * b.hi in
/// one issue slot; operands are two floats in one 64-bit register pair.
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

/// D(8x8) += A(8x4, row) * B(4x8, col) in fp64 on the tensor cores (DMMA).
/// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
/// d = {D[lane/4][2*(lane%4)], D[lane/4][2*(lane%4)+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

} // namespace dctp::dev::ptx
