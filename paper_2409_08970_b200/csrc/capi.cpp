// C ABI (include/dctplus_b200.h): plan construction on the host, constants
// uploaded once per plan, batched apply through the sm_100a kernels.
//
// Compiled with -ffp-contract=off: the setup (host/setup.hpp) must reproduce
// the reference's floating-point operations bit for bit.
#include "dctplus_b200.h"


#include <algorithm>
#include <limits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <unordered_map>
#include <numbers>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include <cuda.h> // driver types only (cuPointerGetAttribute is resolved at run time)
#include <cuda_runtime_api.h>

#include "host/chain.hpp"
#include "host/setup.hpp"
#include "host/signal.hpp"
#include "kernels/launch.hpp"

namespace {

thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return DCTP_OK;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return DCTP_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_last_error = e.what();
        return DCTP_DOMAIN_ERROR;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return DCTP_LOGIC_ERROR;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return DCTP_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DCTP_RUNTIME_ERROR;
    } catch (...) {
        g_last_error = "unknown error";
        return DCTP_RUNTIME_ERROR;
    }
}

/// Makes `device` current for the scope and restores the previous device.
class DeviceScope {
  public:
    explicit DeviceScope(int device) {
        cuda_check(cudaGetDevice(&prev_), "cudaGetDevice");
        if (prev_ != device) cuda_check(cudaSetDevice(device), "cudaSetDevice");
        changed_ = prev_ != device;
    }
    ~DeviceScope() {
        if (changed_) cudaSetDevice(prev_);
    }

  private:
    int prev_ = 0;
    bool changed_ = false;
};

void prepare_pool(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.push_back(device);
}

/// Packs host arrays into one device allocation (256-byte aligned pieces).
class Blob {
  public:
    template <class T>
    std::size_t add(const std::vector<T>& v) {
        const std::size_t off = (bytes_.size() + 255) / 256 * 256;
        bytes_.resize(off + std::max<std::size_t>(v.size() * sizeof(T), 1));
        if (!v.empty()) std::memcpy(bytes_.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
    void* upload() {
        void* d = nullptr;
        cuda_check(cudaMalloc(&d, bytes_.size()), "cudaMalloc(plan constants)");
        cuda_check(cudaMemcpy(d, bytes_.data(), bytes_.size(), cudaMemcpyHostToDevice), "cudaMemcpy(plan constants)");
        return d;
    }

  private:
    std::vector<unsigned char> bytes_;
};

template <class T>
const T* at(void* base, std::size_t off) {
    return reinterpret_cast<const T*>(static_cast<const unsigned char*>(base) + off);
}

/// Twiddle tables of length n in fp64 (exact index angles) and fp32.
struct TwiddleOffsets {
    std::size_t fft = 0, split = 0, rot = 0, cos4n = 0;
};

template <class T>
TwiddleOffsets add_twiddles(Blob& blob, std::size_t n) {
    const double pi = std::numbers::pi;
    const std::size_t N = std::max<std::size_t>(n / 2, 1);
    std::vector<T> fft(2 * std::max<std::size_t>(N / 2, 1)), split(2 * N), rot(2 * (N + 1)), c4(4 * n);
    for (std::size_t k = 0; k < fft.size() / 2; ++k) {
        const double a = 2.0 * pi * static_cast<double>(k) / static_cast<double>(N);
        fft[2 * k] = static_cast<T>(std::cos(a));
        fft[2 * k + 1] = static_cast<T>(-std::sin(a));
    }
    for (std::size_t k = 0; k < N; ++k) {
        const double a = 2.0 * pi * static_cast<double>(k) / static_cast<double>(n);
        split[2 * k] = static_cast<T>(std::cos(a));
        split[2 * k + 1] = static_cast<T>(-std::sin(a));
    }
    for (std::size_t k = 0; k <= N; ++k) {
        const double a = pi * static_cast<double>(k) / (2.0 * static_cast<double>(n));
        rot[2 * k] = static_cast<T>(std::cos(a));
        rot[2 * k + 1] = static_cast<T>(-std::sin(a));
    }
    for (std::size_t m = 0; m < 4 * n; ++m)
        c4[m] = static_cast<T>(std::cos(pi * static_cast<double>(m) / (2.0 * static_cast<double>(n))));
    TwiddleOffsets o;
    o.fft = blob.add(fft);
    o.split = blob.add(split);
    o.rot = blob.add(rot);
    o.cos4n = blob.add(c4);
    return o;
}

template <class T>
dctp::dev::Twiddles<T> twiddles_at(void* base, const TwiddleOffsets& o) {
    return {at<T>(base, o.fft), at<T>(base, o.split), at<T>(base, o.rot), at<T>(base, o.cos4n)};
}

/// Device-side description of one Cauchy stage in both precisions.
struct StageOffsets {
    std::size_t src, x, rscale64, rscale32, dst, y, cscale64, cscale32;
    int rows, cols;
    int src_contig = 0;
};

dctp::dev::CauchyStage stage_at(void* base, const StageOffsets& s, bool f32, std::int64_t out_offset) {
    return {at<int>(base, s.src), at<double>(base, s.x),
            f32 ? static_cast<const void*>(at<float>(base, s.rscale32)) : at<double>(base, s.rscale64),
            at<int>(base, s.dst), at<double>(base, s.y),
            f32 ? static_cast<const void*>(at<float>(base, s.cscale32)) : at<double>(base, s.cscale64),
            s.rows, s.cols, out_offset, s.src_contig};
}

template <class T>
std::vector<float> to_f32(const std::vector<T>& v) {
    return std::vector<float>(v.begin(), v.end());
}

/// Host-side apply tables derived from a setup (fast_transform.hpp:94-125
/// restated for the direct Cauchy route).
struct ApplyTables {
    std::vector<int> kept_idx, act_slot, pass_slot, pass_src;
    std::vector<double> lam_kept, z_kept, neg_z_kept, nu, act_scale, pass_sign;
};

ApplyTables make_tables(const dctp::host::Setup& st) {
    ApplyTables t;
    for (std::size_t j : st.kept) {
        t.kept_idx.push_back(static_cast<int>(j));
        t.lam_kept.push_back(st.lambda[j]);
        t.z_kept.push_back(st.z[j]);
        t.neg_z_kept.push_back(-st.z[j]);
    }
    t.act_slot.assign(st.sub_mu.size(), -1);
    t.nu = st.sub_mu;
    t.act_scale.assign(st.sub_mu.size(), 0.0);
    for (std::size_t s = 0; s < st.slots.size(); ++s) {
        const auto& sl = st.slots[s];
        if (sl.passthrough) {
            t.pass_slot.push_back(static_cast<int>(s));
            t.pass_src.push_back(static_cast<int>(sl.idx));
            t.pass_sign.push_back(st.sigma[s]);
        } else {
            t.act_slot[sl.idx] = static_cast<int>(s);
            // out_s = sigma_s a_s sum_j z_j shat_j / (lambda_j - nu)
            t.act_scale[sl.idx] = st.sigma[s] * st.a[s];
        }
    }
    return t;
}

template <class T>
struct Scratch {
    T* ptr = nullptr;
    cudaStream_t stream = nullptr;
    Scratch(std::size_t count, cudaStream_t s) : stream(s) {
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&ptr), std::max<std::size_t>(count, 1) * sizeof(T), s),
                   "cudaMallocAsync(scratch)");
    }
    ~Scratch() {
        if (ptr) cudaFreeAsync(ptr, stream);
    }
};

/// Optional per-launch CUDA-event timing of every kernel the library issues
/// (bench.py's roofline and launch count); off unless dctp_profile_enable(1).
class Profiler {
  public:
    static Profiler& get() {
        static Profiler* p = new Profiler;
        return *p;
    }
    bool on() const { return on_; }
    void enable(bool on) { on_ = on; }
    template <class F>
    cudaError_t run(const char* name, cudaStream_t s, F&& launch) {
        if (!on_) return launch();
        cudaEvent_t a = take(), b = take();
        cudaEventRecord(a, s);
        const cudaError_t e = launch();
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lock(mu_);
        pending_.push_back({name, a, b});
        return e;
    }
    std::string summary() {
        std::lock_guard<std::mutex> lock(mu_);
        for (auto& p : pending_) {
            cudaEventSynchronize(p.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.a, p.b);
            auto& acc = totals_[p.name];
            acc.first += 1;
            acc.second += ms;
            free_.push_back(p.a);
            free_.push_back(p.b);
        }
        pending_.clear();
        std::string out = "{";
        bool first = true;
        for (auto& [name, acc] : totals_) {
            char buf[160];
            std::snprintf(buf, sizeof buf, "%s\"%s\": [%ld, %.6f]", first ? "" : ", ", name.c_str(), acc.first,
                          acc.second);
            out += buf;
            first = false;
        }
        return out + "}";
    }
    void reset() {
        summary();
        std::lock_guard<std::mutex> lock(mu_);
        totals_.clear();
    }

  private:
    cudaEvent_t take() {
        std::lock_guard<std::mutex> lock(mu_);
        if (!free_.empty()) {
            cudaEvent_t e = free_.back();
            free_.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
    };
    std::atomic<bool> on_{false};
    std::mutex mu_;
    std::vector<Pending> pending_;
    std::vector<cudaEvent_t> free_;
    std::map<std::string, std::pair<long, double>> totals_;
};

#define DCTP_LAUNCH(name, stream, call) Profiler::get().run(name, stream, [&] { return (call); })

} // namespace

// ---------------------------------------------------------------------------

/// Non-finite-input flags, one device int per (object, stream): a kernel
/// raises the flag of the stream it runs on, and sync_check(stream) reads and
/// clears only that one — a NaN in one thread's batch surfaces in that
/// thread's call and nowhere else (the reference throws from the failing
/// call, fast_transform.hpp:271-276; plans are shared across threads,
/// :33-34).  Keyed by cudaStreamGetId, so cudaStreamPerThread and the legacy
/// stream resolve to the calling thread's real stream.  Launches captured
/// into a CUDA graph (where cudaStreamGetId is not permitted) raise the
/// object's graph flag, which every sync_check of the object also reads.
struct StreamFlags {
    int device = 0;
    int* graph = nullptr;
    mutable std::mutex mu;
    mutable std::unordered_map<unsigned long long, int*> map;

    void init(int dev) {
        device = dev;
        DeviceScope scope(device);
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&graph), sizeof(int)), "cudaMalloc(flag)");
        cuda_check(cudaMemset(graph, 0, sizeof(int)), "cudaMemset(flag)");
    }
    int* operator()(cudaStream_t s) const {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cuda_check(cudaStreamIsCapturing(s, &cs), "cudaStreamIsCapturing");
        if (cs != cudaStreamCaptureStatusNone) return graph;
        unsigned long long id = 0;
        cuda_check(cudaStreamGetId(s, &id), "cudaStreamGetId");
        std::lock_guard<std::mutex> lock(mu);
        auto it = map.find(id);
        if (it != map.end()) return it->second;
        DeviceScope scope(device);
        int* f = nullptr;
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&f), sizeof(int)), "cudaMalloc(flag)");
        cuda_check(cudaMemset(f, 0, sizeof(int)), "cudaMemset(flag)");
        map.emplace(id, f);
        return f;
    }
    ~StreamFlags() {
        int prev = 0;
        if (cudaGetDevice(&prev) != cudaSuccess) return;
        cudaSetDevice(device);
        for (auto& kv : map) cudaFree(kv.second);
        if (graph) cudaFree(graph);
        cudaSetDevice(prev);
    }
};

struct dctp_plan {
    dctp::host::Setup st;
    dctp::host::Update update;
    int device = 0;
    void* blob = nullptr;
    StreamFlags flags;
    TwiddleOffsets tw64, tw32;
    StageOffsets fwd{}, inv{};
    std::size_t pass_slot = 0, pass_src = 0, pass_sign64 = 0, pass_sign32 = 0;
    // forward emit list: pass-through slots into the output and the kept
    // coefficients compacted (to = -k-1) into the Cauchy stage's input rows
    std::size_t fe_to = 0, fe_from = 0, fe_sign64 = 0, fe_sign32 = 0;
    int n_fe = 0;
    std::size_t stage_desc = 0; // 4 CauchyStage descriptors: fwd64, fwd32, inv64, inv32
    int n_pass = 0;
    bool small = false;         // fused small-plan forward kernel eligible
    std::size_t act_scale64 = 0, z64 = 0, lam = 0, nu = 0, act_slot = 0, kept = 0;
    struct {
        std::size_t act_slot = 0, tmat = 0, kept = 0, pass_src = 0, pass_slot = 0, pass_coef = 0;
        std::size_t fft = 0, split = 0, rot = 0;
        int K = 0, A = 0, n_pass = 0, fold = 0;
    } sm;
    int num_sms = 0;
    // folded route for larger antisymmetric plans (kept DCT indices all odd):
    // u = x_j - x_{n-1-j} times W (cols x L, row c = the slot's weights), plus
    // the half-length DCT of y = x_j + x_{n-1-j} for the even pass-through slots
    struct {
        bool on = false;
        int L = 0, cols = 0, n_even = 0;
        std::size_t ldw = 0, w = 0, map = 0, to = 0, from = 0, sign64 = 0, sign32 = 0;
        std::size_t ldwt = 0, wt = 0, zero = 0; // inverse: W^T (L x cols) and a zero row
        std::size_t wt32 = 0;                    // fp32 forward: W^T rounded, the SGEMM's B (L x ldwt)
        std::size_t w_hi = 0, w_lo = 0;          // fp32 forward on tcgen05: W split 3xTF32 (cols x L)
        std::size_t wt_hi = 0, wt_lo = 0;        // fp32 inverse on tcgen05: W^T split (L x ldwt)
        std::size_t w_sw = 0, wt_sw = 0;         // both, in the kernel's swizzled shared-memory blocks
        std::size_t w_bf = 0, wt_bf = 0;         // fp32 on the persistent bf16x3 GEMM: W and W^T split bf16
        TwiddleOffsets tw64, tw32;
        // fp64 on the int8 tensor cores: slices of W [0] and W^T [1], built on first use
        int8_t* oz[2] = {nullptr, nullptr};
        int* oz_e[2] = {nullptr, nullptr};
        int oz_slices = 0;
        // small plans (p.small, L <= 256): only the grouped int8 forward
        // (fold_i8_route) — even rows [D_even | 0] padded to whole column
        // tiles, then [0 | W], for 96- [0] and 80-column [1] tiles (5 / 6 slices)
        bool small = false;
        std::size_t g_b[2] = {0, 0}, g_map[2] = {0, 0};
        int g_rows[2] = {0, 0}, g_split[2] = {0, 0};
        int8_t* g_sl[2] = {nullptr, nullptr};
        int* g_e[2] = {nullptr, nullptr};
    } fd;
    // NFST fast route (fp64): the reference's own forward algorithm on the GPU
    struct {
        bool on = false;
        std::size_t hz = 0, ez = 0, inv_phi = 0, tw2n = 0, rot = 0, slot = 0, lo = 0, p0 = 0, b = 0, ca = 0, cb = 0,
                    ctab = 0;
        double z0 = 0.0, ext_scale = 0.0;
        int R = 0, taps = 0, hw = 0, ext_slot = -1;
        bool preferred = false;  // chosen at creation (decide_fast_route)
        bool probing = false;    // decide_fast_route's probe runs the NFST kernel itself
        double probe_gap = 0.0;  // NFST vs exact on the creation probe (max-norm relative)
    } fs;
    // materialised basis for the dense routes (forward_nmvp, inverse(fast =
    // false)): X^T then X, n x ld doubles each; built on first use
    struct Dense {
        std::mutex mu;
        double* buf = nullptr;
        std::size_t ld = 0;
        // int8 slices of X^T [0] and X [1] for the tcgen05 kind::i8 products
        // (ozaki.cu), built on first use
        int8_t* oz[2] = {nullptr, nullptr};
        int* oz_e[2] = {nullptr, nullptr};
        int oz_slices = 0;
        // int8 slices of the NFST route's own linear maps (forward [0],
        // adjoint inverse [1]) materialised as n x n operators (ensure_nfst_ozaki)
        int8_t* nf[2] = {nullptr, nullptr};
        int* nf_e[2] = {nullptr, nullptr};
        int nf_slices[2] = {0, 0};
    };
    std::unique_ptr<Dense> dense = std::make_unique<Dense>();

    ~dctp_plan() {
        if (blob) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            cudaFree(blob);
            if (dense && dense->buf) cudaFree(dense->buf);
            if (dense)
                for (int i = 0; i < 2; ++i) {
                    if (dense->oz[i]) cudaFree(dense->oz[i]);
                    if (dense->oz_e[i]) cudaFree(dense->oz_e[i]);
                    if (dense->nf[i]) cudaFree(dense->nf[i]);
                    if (dense->nf_e[i]) cudaFree(dense->nf_e[i]);
                }
            for (int i = 0; i < 2; ++i) {
                if (fd.oz[i]) cudaFree(fd.oz[i]);
                if (fd.oz_e[i]) cudaFree(fd.oz_e[i]);
                if (fd.g_sl[i]) cudaFree(fd.g_sl[i]);
                if (fd.g_e[i]) cudaFree(fd.g_e[i]);
            }
            cudaSetDevice(prev);
        }
    }

    const dctp::dev::CauchyStage* stage_dev(int which) const {
        return at<dctp::dev::CauchyStage>(blob, stage_desc) + which;
    }
    template <class T>
    dctp::dev::Twiddles<T> tw() const {
        if constexpr (std::is_same_v<T, double>)
            return twiddles_at<double>(blob, tw64);
        else
            return twiddles_at<float>(blob, tw32);
    }
    template <class T>
    dctp::dev::Emit<T> emit_fwd() const {
        const T* sign;
        if constexpr (std::is_same_v<T, double>)
            sign = at<double>(blob, pass_sign64);
        else
            sign = at<float>(blob, pass_sign32);
        return {at<int>(blob, pass_slot), at<int>(blob, pass_src), sign, n_pass};
    }
    template <class T>
    dctp::dev::Emit<T> emit_fwd_compact(T* alt, std::size_t ld_alt) const {
        const T* sign;
        if constexpr (std::is_same_v<T, double>)
            sign = at<double>(blob, fe_sign64);
        else
            sign = at<float>(blob, fe_sign32);
        return {at<int>(blob, fe_to), at<int>(blob, fe_from), sign, n_fe, alt, ld_alt};
    }
    template <class T>
    dctp::dev::Emit<T> emit_inv() const {
        dctp::dev::Emit<T> e = emit_fwd<T>();
        std::swap(e.to, e.from);
        return e;
    }
};

/// Constants of the fused small-plan kernel (fused_small.cu): generic, or
/// folded when every kept DCT index is odd (antisymmetric update direction).
static void build_small(dctp_plan& p, Blob& blob, const ApplyTables& t) {
    const auto& st = p.st;
    const std::size_t n = st.n, K = t.kept_idx.size(), A = t.nu.size();
    bool odd_only = K > 0;
    for (int j : t.kept_idx) odd_only = odd_only && (j % 2 == 1);
    std::size_t odd_pass = 0;
    for (int j : t.pass_src) odd_pass += (j % 2 == 1);
    const bool fold = odd_only && dctp::dev::fused_small_fold_supported(n, static_cast<int>(A + odd_pass));
    p.small = fold || dctp::dev::fused_small_supported(n, static_cast<int>(K), static_cast<int>(A));
    if (!p.small) return;
    const double pi = std::numbers::pi;
    const std::size_t L = fold ? n / 2 : n, NC = L / 2;
    std::vector<int> act, psrc, pslot, kept;
    std::vector<double> pcoef, tm;
    if (!fold) {
        // T[c][k] = sigma_c a_c z_k / (lambda_k - mu_c): the reference's dense T
        // (fast_transform.hpp:355-366, row = slot) restricted to active x kept.
        tm.resize(A * K);
        for (std::size_t c = 0; c < A; ++c)
            for (std::size_t k = 0; k < K; ++k) tm[c * K + k] = t.act_scale[c] * (t.z_kept[k] / (t.lam_kept[k] - t.nu[c]));
        act = t.act_slot;
        kept = t.kept_idx;
        psrc = t.pass_src;
        pslot = t.pass_slot;
        pcoef = t.pass_sign;
        p.sm.K = static_cast<int>(K);
    } else {
        // W[c][j] = sum_k T[c][k] D[m_k][j], D[m][j] = sqrt(2/n) cos(pi (2m+1)(2j+1) / 2n),
        // kept_k = 2 m_k + 1; odd pass-through slots add rows sigma D[m][j].
        auto dcos = [&](std::size_t m, std::size_t j) {
            const std::size_t q = ((2 * m + 1) * (2 * j + 1)) % (4 * n);
            return std::sqrt(2.0L / n) * std::cos(static_cast<long double>(pi) * q / (2.0L * n));
        };
        const std::size_t cols = A + odd_pass;
        tm.assign(cols * L, 0.0);
        for (std::size_t c = 0; c < A; ++c) {
            std::vector<long double> row(L, 0.0L);
            for (std::size_t k = 0; k < K; ++k) {
                const long double tk = t.act_scale[c] * (t.z_kept[k] / (t.lam_kept[k] - t.nu[c]));
                const std::size_t m = (t.kept_idx[k] - 1) / 2;
                for (std::size_t j = 0; j < L; ++j) row[j] += tk * dcos(m, j);
            }
            for (std::size_t j = 0; j < L; ++j) tm[c * L + j] = static_cast<double>(row[j]);
            act.push_back(t.act_slot[c]);
        }
        std::size_t c = A;
        for (std::size_t q = 0; q < t.pass_src.size(); ++q) {
            const int j0 = t.pass_src[q];
            if (j0 % 2 == 1) {
                for (std::size_t j = 0; j < L; ++j)
                    tm[c * L + j] = static_cast<double>(t.pass_sign[q] * dcos((j0 - 1) / 2, j));
                act.push_back(t.pass_slot[q]);
                ++c;
            } else {
                psrc.push_back(j0 / 2);
                pslot.push_back(t.pass_slot[q]);
                pcoef.push_back(t.pass_sign[q] / std::numbers::sqrt2);
            }
        }
        p.sm.K = static_cast<int>(L);
    }
    p.sm.A = static_cast<int>(act.size());
    p.sm.n_pass = static_cast<int>(psrc.size());
    p.sm.fold = fold ? 1 : 0;
    p.sm.act_slot = blob.add(act);
    p.sm.tmat = blob.add(tm);
    p.sm.kept = blob.add(kept);
    p.sm.pass_src = blob.add(psrc);
    p.sm.pass_slot = blob.add(pslot);
    p.sm.pass_coef = blob.add(pcoef);
    std::vector<double> fft(2 * NC), split(2 * NC), rot(2 * (NC + 1));
    for (std::size_t m = 0; m < fft.size() / 2; ++m) {
        const double a = 2.0 * pi * static_cast<double>(m) / static_cast<double>(NC);
        fft[2 * m] = std::cos(a);
        fft[2 * m + 1] = -std::sin(a);
    }
    for (std::size_t k = 0; k < NC; ++k) {
        const double a = 2.0 * pi * static_cast<double>(k) / static_cast<double>(L);
        split[2 * k] = std::cos(a);
        split[2 * k + 1] = -std::sin(a);
    }
    for (std::size_t k = 0; k <= NC; ++k) {
        const double a = pi * static_cast<double>(k) / (2.0 * static_cast<double>(L));
        rot[2 * k] = std::cos(a);
        rot[2 * k + 1] = -std::sin(a);
    }
    p.sm.fft = blob.add(fft);
    p.sm.split = blob.add(split);
    p.sm.rot = blob.add(rot);
}

/// The folded route of plans too large for the fused kernel (C3: n = 1024,
/// edge (1, n)): when every kept DCT index is odd, each active (and odd
/// pass-through) slot is a dot product of u_j = x_j - x_{n-1-j} (j < n/2)
/// with a row of W = T D_odd, and the even pass-through slots come from the
/// length-n/2 DCT of y_j = x_j + x_{n-1-j} (coefficient sigma / sqrt 2) —
/// the algebra of the fused kernel's fold, with W stored (cols x n/2 doubles,
/// L2-resident) and read by the DMMA product kernel.  W is built once on the
/// host in long double from the same T entries.
static void build_fold(dctp_plan& p, Blob& blob, const ApplyTables& t) {
    const auto& st = p.st;
    const std::size_t n = st.n, K = t.kept_idx.size(), A = t.nu.size();
    if ((p.small && n > 512) || K == 0 || A == 0 || n < 64 || (n & (n - 1)) != 0 || n > (std::size_t{1} << 14))
        return;
    for (int j : t.kept_idx)
        if (j % 2 == 0) return;
    std::size_t odd_pass = 0;
    for (int j : t.pass_src) odd_pass += (j % 2 == 1);
    const std::size_t L = n / 2, cols = A + odd_pass;
    if (static_cast<double>(cols) * L > 1.5 * static_cast<double>(K) * A) return; // the structured route is cheaper
    const double pi = std::numbers::pi;
    std::vector<long double> dtab(L * L); // dtab[m][j] = sqrt(2/n) cos(pi (2m+1)(2j+1) / 2n)
    dctp::host::parallel_for(L, [&](std::size_t m) {
        for (std::size_t j = 0; j < L; ++j) {
            const std::size_t q = ((2 * m + 1) * (2 * j + 1)) % (4 * n);
            dtab[m * L + j] = std::sqrt(2.0L / n) * std::cos(static_cast<long double>(pi) * q / (2.0L * n));
        }
    }, 4);
    const std::size_t ldw = (L + 3) / 4 * 4;
    std::vector<double> w(cols * ldw, 0.0);
    std::vector<int> map(cols), to, from;
    std::vector<double> sign;
    dctp::host::parallel_for(A, [&](std::size_t c) {
        std::vector<long double> row(L, 0.0L);
        for (std::size_t k = 0; k < K; ++k) {
            const long double tk = t.act_scale[c] * (t.z_kept[k] / (t.lam_kept[k] - t.nu[c]));
            const long double* d = dtab.data() + static_cast<std::size_t>((t.kept_idx[k] - 1) / 2) * L;
            for (std::size_t j = 0; j < L; ++j) row[j] += tk * d[j];
        }
        for (std::size_t j = 0; j < L; ++j) w[c * ldw + j] = static_cast<double>(row[j]);
        map[c] = t.act_slot[c];
    }, 2);
    std::size_t c = A;
    for (std::size_t q = 0; q < t.pass_src.size(); ++q) {
        const int j0 = t.pass_src[q];
        if (j0 % 2 == 1) {
            const long double* d = dtab.data() + static_cast<std::size_t>((j0 - 1) / 2) * L;
            for (std::size_t j = 0; j < L; ++j) w[c * ldw + j] = static_cast<double>(t.pass_sign[q] * d[j]);
            map[c++] = t.pass_slot[q];
        } else {
            to.push_back(t.pass_slot[q]);
            from.push_back(j0 / 2);
            sign.push_back(t.pass_sign[q] / std::numbers::sqrt2);
        }
    }
    const std::size_t ldwt = (cols + 3) / 4 * 4;
    std::vector<double> wt(L * ldwt, 0.0);
    for (std::size_t r = 0; r < cols; ++r)
        for (std::size_t j = 0; j < L; ++j) wt[j * ldwt + r] = w[r * ldw + j];
    auto& f = p.fd;
    {
        std::vector<float> hi(cols * L), lo(cols * L);
        for (std::size_t r = 0; r < cols; ++r)
            for (std::size_t j = 0; j < L; ++j) {
                const double v = w[r * ldw + j];
                const float fv = static_cast<float>(v);
                std::uint32_t bits;
                std::memcpy(&bits, &fv, 4);
                bits = (bits + 0x1000u) & 0xffffe000u; // TF32 head, round to nearest (ties away)
                float h;
                std::memcpy(&h, &bits, 4);
                hi[r * L + j] = h;
                lo[r * L + j] = static_cast<float>(v - static_cast<double>(h));
            }
        f.w_hi = blob.add(hi);
        f.w_lo = blob.add(lo);
        const std::size_t ldt = (cols + 3) / 4 * 4;
        std::vector<float> thi(L * ldt, 0.f), tlo(L * ldt, 0.f);
        for (std::size_t r = 0; r < cols; ++r)
            for (std::size_t j = 0; j < L; ++j) {
                thi[j * ldt + r] = hi[r * L + j];
                tlo[j * ldt + r] = lo[r * L + j];
            }
        f.wt_hi = blob.add(thi);
        f.wt_lo = blob.add(tlo);
        f.w_sw = blob.add(dctp::dev::tc_swizzle_b(hi.data(), lo.data(), static_cast<int>(cols), static_cast<int>(L),
                                                  static_cast<int>(L)));
        f.wt_sw = blob.add(dctp::dev::tc_swizzle_b(thi.data(), tlo.data(), static_cast<int>(L),
                                                   static_cast<int>(cols), static_cast<int>(ldt)));
    }
    f.w_bf = blob.add(dctp::dev::tc_bf16x3_swizzle_b(w.data(), static_cast<int>(cols), static_cast<int>(L),
                                                     static_cast<int>(ldw)));
    f.wt_bf = blob.add(dctp::dev::tc_bf16x3_swizzle_b(wt.data(), static_cast<int>(L), static_cast<int>(cols),
                                                      static_cast<int>(ldwt)));
    f.ldwt = ldwt;
    f.wt = blob.add(wt);
    f.wt32 = blob.add(to_f32(wt));
    f.zero = blob.add(std::vector<double>(L, 0.0));
    f.L = static_cast<int>(L);
    f.cols = static_cast<int>(cols);
    f.n_even = static_cast<int>(to.size());
    f.ldw = ldw;
    f.w = blob.add(w);
    f.map = blob.add(map);
    f.to = blob.add(to);
    f.from = blob.add(from);
    f.sign64 = blob.add(sign);
    f.sign32 = blob.add(to_f32(sign));
    f.tw64 = add_twiddles<double>(blob, L);
    f.tw32 = add_twiddles<float>(blob, L);
    f.small = p.small;
    if (L <= 256) {
        // the grouped operand of the int8 route: out[:, gmap[r]] = sum_k [y | u]_k Bg[r][k]
        // with Bg's even rows = sigma / sqrt 2 times the orthonormal DCT-II row of y
        // (the fold kernel's half-length DCT and emit) and the odd rows = W
        for (int v = 0; v < 2; ++v) {
            const std::size_t NT = static_cast<std::size_t>(dctp::dev::ozaki_group_tile(v == 0 ? 5 : 6));
            const std::size_t E = (to.size() + NT - 1) / NT * NT, rows = E + cols, ldg = 2 * L;
            std::vector<double> bg(rows * ldg, 0.0);
            std::vector<int> gmap(rows, -1);
            for (std::size_t q = 0; q < to.size(); ++q) {
                const std::size_t k = static_cast<std::size_t>(from[q]);
                const long double ck = k == 0 ? 1.0L / std::sqrt(2.0L) : 1.0L;
                for (std::size_t j = 0; j < L; ++j) {
                    const std::size_t m = ((2 * j + 1) * k) % (4 * L);
                    bg[q * ldg + j] = static_cast<double>(static_cast<long double>(sign[q]) * std::sqrt(2.0L / L) * ck *
                                                          std::cos(static_cast<long double>(pi) * m / (2.0L * L)));
                }
                gmap[q] = to[q];
            }
            for (std::size_t c = 0; c < cols; ++c) {
                for (std::size_t j = 0; j < L; ++j) bg[(E + c) * ldg + L + j] = w[c * ldw + j];
                gmap[E + c] = map[c];
            }
            f.g_b[v] = blob.add(bg);
            f.g_map[v] = blob.add(gmap);
            f.g_rows[v] = static_cast<int>(rows);
            f.g_split[v] = static_cast<int>(E / NT);
        }
    }
    f.on = true;
}

/// FFTW-friendly grid length of the NFST (nfst.hpp:20-27): the smallest
/// 5-smooth multiple of 4 >= target.
static std::size_t next_fast_fft_size(std::size_t target) {
    for (std::size_t g = (target + 3) / 4 * 4;; g += 4) {
        std::size_t r = g;
        for (std::size_t f : {2, 3, 5})
            while (r % f == 0) r /= f;
        if (r == 1) return g;
    }
}

/// Constants of the NFST fast route: the reference's forward algorithm
/// (fast_transform.hpp:94-133 slot classification, exterior row, theta,
/// 1/sin(n theta), 1/nu, h weights; nfst.hpp:108-150 halfwidth, grid, tau,
/// 1/phi_hat, tap windows) computed here in double with the same formulas.
/// Only where the reference itself runs the NFST: no near-pole guard trip,
/// interior roots present and m |theta| above the reference's dense-sine
/// cutoff (nfst.hpp:111, kDenseWorkCutoff = 4096); power-of-two n so the
/// grid is 4n.  The tap weights exp(-(theta - (lo + t) h)^2 / 4 tau) are
/// factored as P0 B^t C_t (fast Gaussian gridding): equal up to rounding.
static void build_fast(dctp_plan& p, Blob& blob) {
    const auto& st = p.st;
    const std::size_t n = st.n;
    if (st.slow_path || n < 128 || (n & (n - 1)) != 0) return;
    const double pi = std::numbers::pi;
    const std::size_t na = st.sub_mu.size();
    const std::size_t ext_rank = (na == 0) ? 0 : (st.rho > 0.0 ? na - 1 : 0);
    std::vector<int> slot;
    std::vector<double> theta, isn, inu, scale, ez;
    int ext_slot = -1;
    double ext_scale = 0.0;
    for (std::size_t s = 0; s < st.slots.size(); ++s) {
        const auto& sl = st.slots[s];
        if (sl.passthrough) continue;
        const double nu = st.sub_mu[sl.idx];
        const double sc = -st.sigma[s] * st.a[s];
        if (na > 0 && sl.idx == ext_rank) {
            ext_slot = static_cast<int>(s);
            ext_scale = sc;
            ez.resize(n);
            for (std::size_t j = 0; j < n; ++j) ez[j] = (1.0 / (nu - st.lambda[j])) * st.z[j];
        } else {
            const double th = std::acos(1.0 - nu / 2.0);
            slot.push_back(static_cast<int>(s));
            theta.push_back(th);
            isn.push_back(1.0 / std::sin(static_cast<double>(n) * th));
            inu.push_back(1.0 / nu);
            scale.push_back(sc);
        }
    }
    const std::size_t m = n - 1, R = theta.size();
    if (R == 0 || m * R <= 4096) return; // the reference evaluates the exact sine matrix
    std::size_t hw = static_cast<std::size_t>(std::ceil(1.15 * std::log10(1.0 / st.epsilon))) + 3;
    hw = std::max<std::size_t>(hw, 2);
    const std::size_t grid = next_fast_fft_size(4 * (m + 1));
    const std::size_t taps = std::min(2 * hw + 1, grid);
    if (grid != 4 * n || taps == grid || !dctp::dev::nfst_supported(n, static_cast<int>(taps))) return;
    const double logical = 2.0 * static_cast<double>(m + 1);
    const double over = static_cast<double>(grid) / logical;
    const double tau = pi * static_cast<double>(hw) / (logical * logical * over * (over - 0.5));
    const double h = 2.0 * pi / static_cast<double>(grid);
    const double norm = static_cast<double>(grid) * std::sqrt(tau / pi);
    std::vector<double> inv_phi(n, 0.0), hz(n, 0.0), ctab(taps), tw2n(2 * n), rot(2 * (n / 2 + 1));
    for (std::size_t k = 1; k <= m; ++k)
        inv_phi[k] = std::exp(static_cast<double>(k) * static_cast<double>(k) * tau) / norm;
    for (std::size_t j = 1; j < n; ++j)
        hz[j] = (((j % 2) == 1 ? 1.0 : -1.0) / std::sin(static_cast<double>(j) * pi / static_cast<double>(n))) * st.z[j];
    {
        const double alpha = h * h / (4.0 * tau), H = static_cast<double>(hw);
        ctab.assign(5, 0.0);
        ctab[0] = std::exp(-alpha * H * H);
        ctab[1] = std::exp(-alpha * (1.0 - H) * (1.0 - H));
        ctab[2] = std::exp(-4.0 * alpha * (1.0 - H));
        ctab[3] = std::exp(-4.0 * alpha * (2.0 - H));
        ctab[4] = std::exp(-8.0 * alpha);
    }
    std::vector<int> lo(R);
    std::vector<double> p0(R), bb(R), ca(R), cb(R);
    for (std::size_t r = 0; r < R; ++r) {
        const long ell0 = std::lround(theta[r] / h);
        const double dc = theta[r] - static_cast<double>(ell0) * h;
        lo[r] = static_cast<int>(ell0 - static_cast<long>(hw));
        p0[r] = std::exp(-dc * dc / (4.0 * tau) - static_cast<double>(hw) * dc * h / (2.0 * tau));
        bb[r] = std::exp(dc * h / (2.0 * tau));
        ca[r] = -0.25 * scale[r] * isn[r];
        cb[r] = scale[r] * inu[r];
    }
    for (std::size_t k = 0; k < n; ++k) {
        const double a = pi * static_cast<double>(k) / static_cast<double>(n);
        tw2n[2 * k] = std::cos(a);
        tw2n[2 * k + 1] = -std::sin(a);
    }
    for (std::size_t k = 0; k <= n / 2; ++k) {
        const double a = pi * static_cast<double>(k) / (2.0 * static_cast<double>(n));
        rot[2 * k] = std::cos(a);
        rot[2 * k + 1] = -std::sin(a);
    }
    auto& f = p.fs;
    f.hz = blob.add(hz);
    f.ez = blob.add(ez);
    f.inv_phi = blob.add(inv_phi);
    f.tw2n = blob.add(tw2n);
    f.rot = blob.add(rot);
    f.slot = blob.add(slot);
    f.lo = blob.add(lo);
    f.p0 = blob.add(p0);
    f.b = blob.add(bb);
    f.ca = blob.add(ca);
    f.cb = blob.add(cb);
    f.ctab = blob.add(ctab);
    f.z0 = st.z[0];
    f.ext_scale = ext_scale;
    f.ext_slot = ext_slot;
    f.R = static_cast<int>(R);
    f.taps = static_cast<int>(taps);
    f.hw = static_cast<int>(hw);
    f.on = true;
}

static dctp::dev::FastPlanDev fast_plan_dev(const dctp_plan* p) {
    const auto& f = p->fs;
    dctp::dev::FastPlanDev d{};
    d.hz = at<double>(p->blob, f.hz);
    d.ez = f.ext_slot >= 0 ? at<double>(p->blob, f.ez) : nullptr;
    d.inv_phi = at<double>(p->blob, f.inv_phi);
    d.tw2n = at<double>(p->blob, f.tw2n);
    d.rot = at<double>(p->blob, f.rot);
    d.pass_slot = at<int>(p->blob, p->pass_slot);
    d.pass_src = at<int>(p->blob, p->pass_src);
    d.pass_sign = at<double>(p->blob, p->pass_sign64);
    d.t_slot = at<int>(p->blob, f.slot);
    d.t_lo = at<int>(p->blob, f.lo);
    d.t_p0 = at<double>(p->blob, f.p0);
    d.t_b = at<double>(p->blob, f.b);
    d.t_ca = at<double>(p->blob, f.ca);
    d.t_cb = at<double>(p->blob, f.cb);
    d.ctab = at<double>(p->blob, f.ctab);
    d.z0 = f.z0;
    d.ext_scale = f.ext_scale;
    d.n = static_cast<int>(p->st.n);
    d.logn = 0;
    while ((std::size_t{1} << d.logn) < p->st.n) ++d.logn;
    d.R = f.R;
    d.taps = f.taps;
    d.hw = f.hw;
    d.n_pass = p->n_pass;
    d.ext_slot = f.ext_slot;
    return d;
}

/// The NFST fast route serves fp64 plans where the reference runs its own
/// NFST; whether it is the plan's forward route is decided at creation
/// (decide_fast_route).  DCTP_FAST=0 / 1 forces it off / on (where available).
static bool fast_route(const dctp_plan* p) {
    if (!p->fs.on) return false;
    const char* e = std::getenv("DCTP_FAST");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    return p->fs.preferred;
}

/// Development knob for profiling the fused kernel's phases in isolation
/// (DCTP_DEBUG_MODE bits: 1 = DCT work skipped, 2 = DMMA work skipped, 4 = producer
/// phase timers); 0 otherwise.
static int debug_mode() {
    static const int mode = [] {
        const char* e = std::getenv("DCTP_DEBUG_MODE");
        return e ? std::atoi(e) : 0;
    }();
    return mode;
}

static unsigned long long* g_debug_timers = nullptr;
static void reset_debug_timers() {
    unsigned long long h[16] = {0};
    h[8] = h[11] = ~0ull; // min slots
    cudaMemcpy(g_debug_timers, h, sizeof(h), cudaMemcpyHostToDevice);
}
static unsigned long long* debug_timers() {
    if ((debug_mode() & 4) == 0) return nullptr;
    if (!g_debug_timers) {
        cudaMalloc(reinterpret_cast<void**>(&g_debug_timers), 16 * sizeof(unsigned long long));
        reset_debug_timers();
    }
    return g_debug_timers;
}

extern "C" int dctp_debug_timers(unsigned long long* out16) {
    if (!g_debug_timers) return 1;
    cudaMemcpy(out16, g_debug_timers, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    reset_debug_timers();
    return 0;
}

static void upload_plan(dctp_plan& p) {
    const auto& st = p.st;
    const ApplyTables t = make_tables(st);
    Blob blob;
    p.tw64 = add_twiddles<double>(blob, st.n);
    p.tw32 = add_twiddles<float>(blob, st.n);
    const std::size_t kept_idx = blob.add(t.kept_idx), lam = blob.add(t.lam_kept);
    const std::size_t z64 = blob.add(t.z_kept), z32 = blob.add(to_f32(t.z_kept));
    const std::size_t nz64 = blob.add(t.neg_z_kept), nz32 = blob.add(to_f32(t.neg_z_kept));
    const std::size_t act = blob.add(t.act_slot), nu = blob.add(t.nu);
    const std::size_t sc64 = blob.add(t.act_scale), sc32 = blob.add(to_f32(t.act_scale));
    p.pass_slot = blob.add(t.pass_slot);
    p.pass_src = blob.add(t.pass_src);
    p.act_scale64 = sc64;
    p.z64 = z64;
    p.lam = lam;
    p.nu = nu;
    p.act_slot = act;
    p.kept = kept_idx;
    build_small(p, blob, t);
    build_fold(p, blob, t);
    build_fast(p, blob);
    p.pass_sign64 = blob.add(t.pass_sign);
    p.pass_sign32 = blob.add(to_f32(t.pass_sign));
    p.n_pass = static_cast<int>(t.pass_slot.size());
    const int K = static_cast<int>(t.kept_idx.size()), A = static_cast<int>(t.nu.size());
    std::size_t kept_idx_iota = 0;
    {
        std::vector<int> to = t.pass_slot, from = t.pass_src, iota(t.kept_idx.size());
        std::vector<double> sign = t.pass_sign;
        for (std::size_t k = 0; k < t.kept_idx.size(); ++k) {
            to.push_back(-static_cast<int>(k) - 1);
            from.push_back(t.kept_idx[k]);
            sign.push_back(1.0);
            iota[k] = static_cast<int>(k);
        }
        p.fe_to = blob.add(to);
        p.fe_from = blob.add(from);
        p.fe_sign64 = blob.add(sign);
        p.fe_sign32 = blob.add(to_f32(sign));
        p.n_fe = static_cast<int>(to.size());
        kept_idx_iota = blob.add(iota);
    }
    p.fwd = {kept_idx_iota, lam, z64, z32, act, nu, sc64, sc32, K, A, 1};
    p.inv = {act, nu, sc64, sc32, kept_idx, lam, nz64, nz32, A, K};
    // Stage descriptors hold device pointers: reserve, upload, then patch.
    p.stage_desc = blob.add(std::vector<dctp::dev::CauchyStage>(4));
    p.blob = blob.upload();
    const dctp::dev::CauchyStage desc[4] = {stage_at(p.blob, p.fwd, false, 0), stage_at(p.blob, p.fwd, true, 0),
                                            stage_at(p.blob, p.inv, false, 0), stage_at(p.blob, p.inv, true, 0)};
    cuda_check(cudaMemcpy(static_cast<unsigned char*>(p.blob) + p.stage_desc, desc, sizeof(desc),
                          cudaMemcpyHostToDevice),
               "cudaMemcpy(stage descriptors)");
    p.flags.init(p.device);
    cuda_check(cudaDeviceGetAttribute(&p.num_sms, cudaDevAttrMultiProcessorCount, p.device), "cudaDeviceGetAttribute");
}

static dctp::host::Update make_update(int kind, std::size_t i, std::size_t j, double rho, const double* v,
                                      std::size_t n) {
    switch (kind) {
        case DCTP_SELF_LOOP: return dctp::host::Update::self_loop(i, rho);
        case DCTP_EDGE_DELTA: return dctp::host::Update::edge_delta(i, j, rho);
        case DCTP_GENERAL:
            if (!v) throw std::invalid_argument("RankOneUpdate: general update needs a direction");
            return dctp::host::Update::general(std::vector<double>(v, v + n), rho);
        default: throw std::invalid_argument("RankOneUpdate: unknown update kind");
    }
}

template <class T>
static void plan_forward(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s);
static void decide_fast_route(dctp_plan& p);

/// The secular roots and normalisers run on the current device from n =
/// DCTP_GPU_SETUP_MIN_N (default 1024; below it the host loops take
/// milliseconds); DCTP_GPU_SETUP=0 / 1 forces the choice.  Bit-identical
/// either way (kernels/setup.cu).
static bool gpu_setup(std::size_t n) {
    const char* e = std::getenv("DCTP_GPU_SETUP");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    const char* m = std::getenv("DCTP_GPU_SETUP_MIN_N");
    return n >= (m ? static_cast<std::size_t>(std::atoll(m)) : std::size_t{1024});
}

static dctp::host::SecularBackend gpu_secular_backend() {
    dctp::host::SecularBackend be;
    be.roots = [](const std::vector<double>& lam, const std::vector<double>& z, double rho, double zz) {
        const std::size_t k = lam.size();
        double* d = nullptr;
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), 3 * k * sizeof(double) + sizeof(int)), "cudaMalloc(setup)");
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        int* status = reinterpret_cast<int*>(d + 3 * k);
        cuda_check(cudaMemcpy(d, lam.data(), k * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(setup)");
        cuda_check(cudaMemcpy(d + k, z.data(), k * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(setup)");
        cuda_check(cudaMemset(status, 0, sizeof(int)), "cudaMemset(setup)");
        cuda_check(DCTP_LAUNCH("secular_roots", nullptr,
                               dctp::dev::secular_roots_gpu(d, d + k, static_cast<int>(k), rho, zz, d + 2 * k, status,
                                                            nullptr)),
                   "secular roots kernel");
        std::vector<double> mu(k);
        int st = 0;
        cuda_check(cudaMemcpy(mu.data(), d + 2 * k, k * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy(setup)");
        cuda_check(cudaMemcpy(&st, status, sizeof(int), cudaMemcpyDeviceToHost), "cudaMemcpy(setup)");
        if (st) throw std::runtime_error("secular_eigenvalues: no convergence in 200 iterations");
        return mu;
    };
    be.normalisers = [](const std::vector<double>& lam, const std::vector<double>& mu, const std::vector<double>& z) {
        const std::size_t m = lam.size(), k = mu.size();
        double* d = nullptr;
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), (2 * m + 2 * k) * sizeof(double) + sizeof(int)),
                   "cudaMalloc(setup)");
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        int* status = reinterpret_cast<int*>(d + 2 * m + 2 * k);
        cuda_check(cudaMemcpy(d, lam.data(), m * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(setup)");
        cuda_check(cudaMemcpy(d + m, z.data(), m * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(setup)");
        cuda_check(cudaMemcpy(d + 2 * m, mu.data(), k * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(setup)");
        cuda_check(cudaMemset(status, 0, sizeof(int)), "cudaMemset(setup)");
        cuda_check(DCTP_LAUNCH("normalisers", nullptr,
                               dctp::dev::normalisers_gpu(d, d + m, static_cast<int>(m), d + 2 * m,
                                                          static_cast<int>(k), d + 2 * m + k, status, nullptr)),
                   "normalisers kernel");
        std::vector<double> a(k);
        int st = 0;
        cuda_check(cudaMemcpy(a.data(), d + 2 * m + k, k * sizeof(double), cudaMemcpyDeviceToHost),
                   "cudaMemcpy(setup)");
        cuda_check(cudaMemcpy(&st, status, sizeof(int), cudaMemcpyDeviceToHost), "cudaMemcpy(setup)");
        if (st & 2) throw std::domain_error("normalizers: mu/lambda collision; deflation missing");
        if (st & 4) throw std::domain_error("normalizers: degenerate column");
        return a;
    };
    // sigma: the unsigned basis columns (DCT-domain rows a_s z_j / (lambda_j -
    // nu_s), one batched DCT-III) in chunks of <= 256 MB, then the column-sign
    // rule on each (cauchy.hpp:84-103, spectral.hpp:30-37)
    be.signs = [](dctp::host::Setup& st) {
        const std::size_t n = st.n, ld = (n + 3) / 4 * 4;
        Blob blob;
        const TwiddleOffsets two = add_twiddles<double>(blob, n);
        std::vector<double> tab(5 * n, 0.0); // z, lambda, nu, a, sigma = 1
        std::vector<int> pidx(n);
        for (std::size_t q = 0; q < n; ++q) {
            tab[q] = st.z[q];
            tab[n + q] = st.lambda[q];
            const auto& sl = st.slots[q];
            pidx[q] = sl.passthrough ? static_cast<int>(sl.idx) : -1;
            tab[2 * n + q] = sl.passthrough ? 0.0 : st.sub_mu[sl.idx];
            tab[3 * n + q] = st.a[q];
            tab[4 * n + q] = 1.0;
        }
        const std::size_t tab_off = blob.add(tab), pidx_off = blob.add(pidx);
        const std::size_t sign_off = blob.add(std::vector<double>(n, 1.0)), flag_off = blob.add(std::vector<int>(1, 0));
        void* base = blob.upload();
        std::unique_ptr<void, decltype(&cudaFree)> hold_blob(base, &cudaFree);
        const double* dtab = at<double>(base, tab_off);
        const int* dp = at<int>(base, pidx_off);
        double* dsign = const_cast<double*>(at<double>(base, sign_off));
        int* dflag = const_cast<int*>(at<int>(base, flag_off));
        const std::size_t chunk = std::max<std::size_t>(1, std::min(n, (std::size_t{256} << 20) / (2 * ld * 8)));
        double* y = nullptr;
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&y), 2 * chunk * ld * sizeof(double)), "cudaMalloc(signs)");
        std::unique_ptr<double, decltype(&cudaFree)> hold_y(y, &cudaFree);
        const int ni = static_cast<int>(n);
        for (std::size_t r0 = 0; r0 < n; r0 += chunk) {
            const int rows = static_cast<int>(std::min(chunk, n - r0));
            cuda_check(dctp::dev::basis_coefficients(ni, ld, dtab, dtab + n, dtab + 2 * n + r0, dp + r0,
                                                     dtab + 3 * n + r0, dtab + 4 * n + r0, y, nullptr, rows),
                       "basis kernel (signs)");
            cuda_check(dctp::dev::idct_rows<double>(y, ld, y, ld, dctp::dev::Emit<double>{}, y + chunk * ld, ld, n,
                                                    static_cast<std::size_t>(rows), twiddles_at<double>(base, two),
                                                    dflag, nullptr),
                       "basis idct kernel (signs)");
            cuda_check(DCTP_LAUNCH("column_signs", nullptr,
                                   dctp::dev::column_signs_gpu(y + chunk * ld, ld, ni, rows, dsign + r0, nullptr)),
                       "column signs kernel");
        }
        cuda_check(cudaMemcpy(st.sigma.data(), dsign, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H(signs)");
    };
    return be;
}

static std::unique_ptr<dctp_plan> build_plan(std::size_t n, const dctp::host::Update& u, double eps, double tau,
                                             int device) {
    auto p = std::make_unique<dctp_plan>();
    p->update = u;
    p->device = device;
    if (device < 0) { // host-only plan: setup vectors, no device constants
        p->st = dctp::host::build_setup(n, u, eps, tau);
        return p;
    }
    if (!dctp::dev::dct_supported(n, true))
        throw std::invalid_argument("DctPlusPlan: n = " + std::to_string(n) +
                                    " exceeds the GPU DCT kernels (a row must fit in shared memory: powers of two "
                                    "up to 8192, other sizes up to 14528)");
    DeviceScope scope(device);
    const dctp::host::SecularBackend be = gpu_secular_backend();
    p->st = dctp::host::build_setup(n, u, eps, tau, gpu_setup(n) ? &be : nullptr);
    prepare_pool(device);
    upload_plan(*p);
    decide_fast_route(*p);
    return p;
}

/// The Cauchy stage: fp64 on the DMMA tensor cores (K >= 32), else SIMT.
template <class T>
static cudaError_t cauchy_stage(const T* in, std::size_t ld_in, T* out, std::size_t ld_out,
                                const dctp::dev::CauchyStage* stages, int num_stages, int max_rows, int max_cols,
                                std::size_t batch, int* flag, cudaStream_t s) {
    if constexpr (std::is_same_v<T, double>) {
        if (max_rows >= 32)
            return dctp::dev::cauchy_rows_dmma(in, ld_in, out, ld_out, stages, num_stages, max_cols, batch, flag, s);
    }
    return dctp::dev::cauchy_rows<T>(in, ld_in, out, ld_out, stages, num_stages, max_rows, max_cols, batch, flag, s);
}

static dctp::dev::SmallPlanDev small_plan_dev(const dctp_plan* p) {
    const auto& m = p->sm;
    return dctp::dev::SmallPlanDev{at<int>(p->blob, m.act_slot), at<double>(p->blob, m.tmat), at<int>(p->blob, m.kept),
                                   at<int>(p->blob, m.pass_src), at<int>(p->blob, m.pass_slot),
                                   at<double>(p->blob, m.pass_coef), at<double>(p->blob, m.fft),
                                   at<double>(p->blob, m.split), at<double>(p->blob, m.rot),
                                   static_cast<int>(p->st.n), m.K, m.A, m.n_pass, m.fold, debug_timers(),
                                   debug_mode()};
}

template <class T>
static void plan_dense(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s, bool inverse);
static bool dense_route(const dctp_plan* p);
static void ensure_dense(const dctp_plan* p, cudaStream_t s);

/// Small plans take the one-launch dense product (small_dense.cu) where it
/// beats the fused persistent kernel (tools/small_sweep.py, GPU time per
/// forward from CUDA-graph replay): n <= 64 at every batch (n = 64: 5.7 vs
/// 14.6 us at 4096 signals, 32.5 vs 92.8 us at 65536), n = 128 up to
/// DCTP_SMALL_DENSE_MAX rows (default 16384: 12.0 vs 20.7 us at 4096, even at
/// 16384, 186 vs 142 us at 65536).  DCTP_SMALL_DENSE = 0 / 1 forces it off / on.
static bool small_dense_route(const dctp_plan* p, std::size_t batch) {
    const char* e = std::getenv("DCTP_SMALL_DENSE");
    if (e && e[0] == '0') return false;
    if (p->st.n > 128) return false;
    if (e && e[0] == '1') return true;
    static const std::size_t max_rows = [] {
        const char* m = std::getenv("DCTP_SMALL_DENSE_MAX");
        return m ? static_cast<std::size_t>(std::atoll(m)) : std::size_t{16384};
    }();
    return p->st.n <= 64 || batch <= max_rows;
}

/// DCTP_FOLD=0 turns the folded route off (structured DCT + Cauchy instead).
static bool fold_route(const dctp_plan* p) {
    if (!p->fd.on || p->fd.small) return false;
    const char* e = std::getenv("DCTP_FOLD");
    return !(e && e[0] == '0');
}

// int8 tensor-core (Ozaki) products, defined with the dense routes below
static int ozaki_slices(std::size_t n);
// shortest product length the folded route sends to them (DCTP_OZAKI_FOLD_MIN_K):
// 512 (C3 forward 0.17 + the slices written by the fold kernel vs 0.30 ms on
// DMMA; inverse 0.21 + 0.06 slicing vs 0.37 ms)
static int ozaki_fold_min_k(bool) {
    static const int v = [] {
        const char* e = std::getenv("DCTP_OZAKI_FOLD_MIN_K");
        return e ? std::atoi(e) : 512;
    }();
    return v;
}
static void ensure_fold_ozaki(const dctp_plan* p, int which, int S, cudaStream_t s);
static void rows_by_ozaki(const double* in, std::size_t ld_in, const int8_t* b_sl, const int* eb, int K, int N,
                          int S, double* out, std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t s,
                          const char* name, const int* col_map = nullptr, const int* a_map = nullptr,
                          const double* fold_add = nullptr, std::size_t ld_add = 0);
static int nfst_dense_slices(const dctp_plan* p, int which);
static void ensure_nfst_ozaki(const dctp_plan* p, int which, int S, cudaStream_t s);

/// Slice count of the int8 products where the route does not depend on n
/// (DCTP_OZAKI_SLICES: 5 default, or 6).
static int ozaki_slice_count() {
    static const int v = [] {
        const char* e = std::getenv("DCTP_OZAKI_SLICES");
        const int k = e ? std::atoi(e) : 5;
        return (k == 5 || k == 6) ? k : 5;
    }();
    return v;
}

/// Grouped int8 route of small folded plans (C2: n = 256, edge (128, 129)):
/// one slicing pass writes [y | u] of every row, one persistent CTA-pair
/// product gives the even (D y) and odd (W u) coefficients — every output row
/// written by one kernel, no FFT.  Measured against the fused DMMA kernel at
/// C2 (tools/fold_i8_sweep.py, bench kernel split): 0.167 ms (slicing 0.046 +
/// product 0.119; the product's operand loads alone take 0.048 — each A
/// half is re-read by two 96-column tiles, TMEM holds 5 x 96 int32 columns)
/// vs 0.139 ms, and slower at every batch from 1024 rows; parity with the
/// fused kernel 6.4e-12.  So the fused kernel stays the route; DCTP_FOLD_I8=1
/// selects this one (tests keep it correct).
static bool fold_i8_route(const dctp_plan* p, std::size_t batch, const void* in, const void* out) {
    const auto& f = p->fd;
    if (!f.on || !f.small || f.g_b[0] == 0 || batch == 0 || !dctp::dev::ozaki_grouped_supported()) return false;
    if ((reinterpret_cast<std::uintptr_t>(in) | reinterpret_cast<std::uintptr_t>(out)) % 16 != 0) return false;
    const char* e = std::getenv("DCTP_FOLD_I8");
    return e && e[0] == '1';
}

/// int8 slices of the grouped operand Bg (variant v: 5 / 6 slices), once per plan.
static void ensure_fold_grouped(const dctp_plan* p, int v, int S, cudaStream_t s);

template <class T>
static void plan_forward(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    if (!p) throw std::invalid_argument("dctp_forward: null plan");
    if (!p->blob) throw std::invalid_argument("DctPlusPlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("dctp_forward: null buffer");
    if (static_cast<const void*>(in) == static_cast<const void*>(out))
        throw std::invalid_argument("dctp_forward: in and out must not alias");
    const std::size_t n = p->st.n;
    DeviceScope scope(p->device);
    if constexpr (std::is_same_v<T, double>) {
        if (fast_route(p)) {
            if (const int S = nfst_dense_slices(p, 0)) { // the NFST's own map, materialised, on the int8 tensor cores
                ensure_nfst_ozaki(p, 0, S, s);
                const auto& d = *p->dense;
                rows_by_ozaki(in, n, d.nf[0], d.nf_e[0], static_cast<int>(n), static_cast<int>(n), S, out, n, batch,
                              p->flags(s), s, "nfst_dense_i8");
                return;
            }
            cuda_check(DCTP_LAUNCH("nfst_fwd", s, dctp::dev::nfst_apply(in, out, batch, fast_plan_dev(p), p->flags(s), false, s)),
                       "nfst forward kernel");
            return;
        }
        if (fold_i8_route(p, batch, in, out)) {
            const auto& f = p->fd;
            const int S = ozaki_slice_count(), v = S == 5 ? 0 : 1;
            ensure_fold_grouped(p, v, S, s);
            const int pm = dctp::dev::ozaki_pad_m(), K2 = 2 * f.L;
            const std::size_t rows_pad = (batch + pm - 1) / pm * pm;
            Scratch<int8_t> a_sl(dctp::dev::ozaki_slice_bytes(batch, K2, 128, S, pm), s);
            Scratch<int> ea(rows_pad, s);
            cuda_check(DCTP_LAUNCH("fold_slice", s,
                                   dctp::dev::ozaki_slice_fold(in, n, batch, f.L, 128, S, a_sl.ptr, ea.ptr, p->flags(s),
                                                               s, pm)),
                       "fold slicing kernel");
            cuda_check(DCTP_LAUNCH("fold_i8", s,
                                   dctp::dev::ozaki_gemm_grouped(a_sl.ptr, ea.ptr, f.g_sl[v], f.g_e[v], batch,
                                                                 f.g_rows[v], K2, S, out, n,
                                                                 at<int>(p->blob, f.g_map[v]), f.g_split[v], f.L, s)),
                       "grouped int8 tensor-core product kernel");
            return;
        }
        // small plans at small batches: one dense product with X^T staged in
        // shared memory (the fused persistent kernel's per-CTA setup costs
        // more than the whole transform there)
        if (small_dense_route(p, batch) && dctp::dev::small_dense_supported(n, in, n, out, n)) {
            ensure_dense(p, s);
            const auto& d = *p->dense;
            cuda_check(DCTP_LAUNCH("small_dense", s,
                                   dctp::dev::small_dense_forward(in, n, d.buf, d.ld, out, n, n, batch, p->flags(s), s)),
                       "small dense kernel");
            return;
        }
        // TMA bulk copies need 16-byte aligned rows; a misaligned view takes
        // the generic (DCT + Cauchy kernel) route instead
        const bool aligned = (reinterpret_cast<std::uintptr_t>(in) | reinterpret_cast<std::uintptr_t>(out)) % 16 == 0;
        static const bool fused_off = [] { // DCTP_FUSED=0: skip the fused kernel (route experiments)
            const char* e = std::getenv("DCTP_FUSED");
            return e && e[0] == '0';
        }();
        if (p->small && aligned && !fused_off) {
            const dctp::dev::SmallPlanDev sp = small_plan_dev(p);
            cuda_check(DCTP_LAUNCH("fused_small_fwd", s,
                                   dctp::dev::fused_small_forward(in, out, batch, sp, p->flags(s), p->num_sms, s)),
                       "fused small forward kernel");
            return;
        }
    }
    if (dense_route(p)) {
        plan_dense<T>(p, in, out, batch, s, false);
        return;
    }
    if (fold_route(p)) {
        const auto& f = p->fd;
        constexpr bool f32 = std::is_same_v<T, float>;
        const dctp::dev::Emit<T> even{at<int>(p->blob, f.to), at<int>(p->blob, f.from),
                                      at<T>(p->blob, f32 ? f.sign32 : f.sign64), f.n_even};
        if constexpr (!f32) {
            // the W product on the int8 tensor cores: the fold kernel writes
            // u's int8 slices directly (no u round trip, no slicing pass)
            if (const int S = f.L >= ozaki_fold_min_k(false) ? ozaki_slices(n) : 0) {
                ensure_fold_ozaki(p, 0, S, s);
                const int pm = dctp::dev::ozaki_pad_m();
                const std::size_t rows_pad = (batch + pm - 1) / pm * pm;
                Scratch<int8_t> a_sl(dctp::dev::ozaki_slice_bytes(batch, f.L, 128, S, pm), s);
                Scratch<int> ea(rows_pad, s);
                const dctp::dev::FoldSlices fs{a_sl.ptr, ea.ptr, S, (f.L + 63) / 64, 128};
                cuda_check(DCTP_LAUNCH("fold_dct", s,
                                       dctp::dev::dct2_fold_rows<T>(in, n, nullptr, f.L, out, n, even, f.L, batch,
                                                                    twiddles_at<T>(p->blob, f.tw64), p->flags(s), s,
                                                                    fs)),
                           "fold dct kernel");
                cuda_check(DCTP_LAUNCH("fold_w_i8", s,
                                       dctp::dev::ozaki_gemm(a_sl.ptr, ea.ptr, f.oz[0], f.oz_e[0], batch, f.cols, f.L,
                                                             S, out, n, at<int>(p->blob, f.map), s)),
                           "int8 tensor-core product kernel");
                return;
            }
        }
        if constexpr (f32) {
            // fp32 on the persistent bf16x3 GEMM: the fold kernel writes u's
            // bf16 hi / lo A image directly (no u round trip, no split pass)
            const char* tc = std::getenv("DCTP_TC32");
            const char* bfe = std::getenv("DCTP_TC_BF16");
            if (!(tc && tc[0] == '0') && !(bfe && bfe[0] == '0') &&
                dctp::dev::tc_bf16x3_supported(f.L, f.cols, n, out)) {
                Scratch<unsigned char> img(dctp::dev::tc_bf16x3_a_bytes(batch, f.L), s);
                dctp::dev::FoldSlices fs;
                fs.bf = img.ptr;
                cuda_check(DCTP_LAUNCH("fold_dct", s,
                                       dctp::dev::dct2_fold_rows<T>(in, n, nullptr, f.L, out, n, even, f.L, batch,
                                                                    twiddles_at<T>(p->blob, f.tw32), p->flags(s), s,
                                                                    fs)),
                           "fold dct kernel");
                cuda_check(DCTP_LAUNCH("fold_w_bf16x3", s,
                                       dctp::dev::tc_bf16x3(nullptr, f.L, at<uint16_t>(p->blob, f.w_bf), out, n, batch,
                                                            f.cols, f.L, p->flags(s), p->num_sms, s,
                                                            at<int>(p->blob, f.map), nullptr, nullptr, 0, img.ptr)),
                           "fold bf16x3 kernel");
                return;
            }
        }
        Scratch<T> u(batch * static_cast<std::size_t>(f.L), s);
        cuda_check(DCTP_LAUNCH("fold_dct", s,
                               dctp::dev::dct2_fold_rows<T>(in, n, u.ptr, f.L, out, n, even, f.L, batch,
                                                            twiddles_at<T>(p->blob, f32 ? f.tw32 : f.tw64), p->flags(s),
                                                            s)),
                   "fold dct kernel");
        if constexpr (f32) {
            // fp32: the tcgen05 3xTF32 GEMM (DCTP_TC32=0: the FFMA2 SGEMM with W^T
            // rounded once, twice the DMMA rate)
            const char* tc = std::getenv("DCTP_TC32");
            const float* wh = at<float>(p->blob, f.w_hi);
            const float* wl = at<float>(p->blob, f.w_lo);
            if (!(tc && tc[0] == '0') && dctp::dev::tc_sgemm3_supported(f.L, f.cols, f.L, f.L, n, u.ptr, wh, wl, out)) {
                cuda_check(DCTP_LAUNCH("fold_w_tc32", s,
                                       dctp::dev::tc_sgemm3(u.ptr, f.L, wh, wl, f.L, out, n, batch, f.cols, f.L,
                                                            p->flags(s), s, at<int>(p->blob, f.map), nullptr, nullptr, 0,
                                                            at<float>(p->blob, f.w_sw))),
                           "fold tcgen05 kernel");
                return;
            }
            const float* b = at<float>(p->blob, f.wt32);
            if (dctp::dev::sgemm_rows_supported(f.L, f.cols, f.L, static_cast<int>(f.ldwt), 4, u.ptr, b, b)) {
                cuda_check(DCTP_LAUNCH("fold_w", s,
                                       dctp::dev::sgemm_rows(u.ptr, f.L, b, static_cast<int>(f.ldwt), out, n, batch,
                                                             f.cols, f.L, p->flags(s), s, at<int>(p->blob, f.map))),
                           "fold sgemm kernel");
                return;
            }
        }
        cuda_check(DCTP_LAUNCH("fold_w", s,
                               dctp::dev::rows_by_basis<T>(u.ptr, f.L, at<double>(p->blob, f.w), f.ldw, f.L, f.cols, out,
                                                           n, batch, p->flags(s), s, at<int>(p->blob, f.map))),
                   "fold product kernel");
        return;
    }
    // DCT; pass-through slots go straight to the output, kept coefficients
    // compacted into `hat` (batch x K) for the Cauchy stage
    const std::size_t K = (static_cast<std::size_t>(std::max(p->fwd.rows, 1)) + 1) / 2 * 2; // even: 16-byte rows
    Scratch<T> hat(batch * K, s);
    cuda_check(DCTP_LAUNCH("dct2", s, dctp::dev::dct2_rows<T>(in, n, nullptr, n, out, n,
                                                             p->emit_fwd_compact<T>(hat.ptr, K), n, batch,
                                                             p->tw<T>(), p->flags(s), s)),
               "dct2 kernel");
    if (p->fwd.cols > 0)
        cuda_check(DCTP_LAUNCH("cauchy", s,
                               cauchy_stage<T>(hat.ptr, K, out, n, p->stage_dev(std::is_same_v<T, float> ? 1 : 0), 1,
                                               p->fwd.rows, p->fwd.cols, batch, p->flags(s), s)),
                   "cauchy kernel");
}

template <class T>
static void plan_inverse(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    if (!p) throw std::invalid_argument("dctp_inverse: null plan");
    if (!p->blob) throw std::invalid_argument("DctPlusPlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("dctp_inverse: null buffer");
    if (static_cast<const void*>(in) == static_cast<const void*>(out))
        throw std::invalid_argument("dctp_inverse: in and out must not alias");
    if constexpr (std::is_same_v<T, double>) {
        if (fast_route(p)) {
            DeviceScope scope(p->device);
            if (const int S = nfst_dense_slices(p, 1)) {
                const std::size_t n = p->st.n;
                ensure_nfst_ozaki(p, 1, S, s);
                const auto& d = *p->dense;
                rows_by_ozaki(in, n, d.nf[1], d.nf_e[1], static_cast<int>(n), static_cast<int>(n), S, out, n, batch,
                              p->flags(s), s, "nfst_dense_inv_i8");
                return;
            }
            cuda_check(DCTP_LAUNCH("nfst_inv", s, dctp::dev::nfst_apply(in, out, batch, fast_plan_dev(p), p->flags(s), true, s)),
                       "nfst inverse kernel");
            return;
        }
    }
    if (dense_route(p)) {
        plan_dense<T>(p, in, out, batch, s, true);
        return;
    }
    if (fold_route(p)) {
        // x_j = w_j + v_j, x_{n-1-j} = w_j - v_j: w = DCT-III (length n/2) of the
        // even slots (sigma / sqrt 2), v = W^T p over the W slots
        const auto& f = p->fd;
        const std::size_t n = p->st.n;
        constexpr bool f32 = std::is_same_v<T, float>;
        DeviceScope scope(p->device);
        const dctp::dev::Emit<T> even{at<int>(p->blob, f.from), at<int>(p->blob, f.to),
                                      at<T>(p->blob, f32 ? f.sign32 : f.sign64), f.n_even};
        Scratch<T> w(batch * static_cast<std::size_t>(f.L), s);
        if constexpr (!f32) {
            // the W^T product on the int8 tensor cores: the fold kernel also
            // gathers p's W slots and writes their int8 slices (no slicing pass)
            if (const int S = f.cols >= ozaki_fold_min_k(true) ? ozaki_slices(n) : 0) {
                ensure_fold_ozaki(p, 1, S, s);
                const int pm = dctp::dev::ozaki_pad_m();
                const std::size_t rows_pad = (batch + pm - 1) / pm * pm;
                Scratch<int8_t> a_sl(dctp::dev::ozaki_slice_bytes(batch, f.cols, 128, S, pm), s);
                Scratch<int> ea(rows_pad, s);
                dctp::dev::FoldSlices fs{a_sl.ptr, ea.ptr, S, (f.cols + 63) / 64, 128};
                fs.map = at<int>(p->blob, f.map);
                fs.K = f.cols;
                cuda_check(DCTP_LAUNCH("fold_idct", s,
                                       dctp::dev::idct_rows<T>(nullptr, 0, in, n, even, w.ptr, f.L,
                                                               f.L, batch, twiddles_at<T>(p->blob, f.tw64),
                                                               p->flags(s), s, fs)),
                           "fold idct kernel");
                cuda_check(DCTP_LAUNCH("fold_wt_i8", s,
                                       dctp::dev::ozaki_gemm(a_sl.ptr, ea.ptr, f.oz[1], f.oz_e[1], batch, f.L, f.cols,
                                                             S, out, n, nullptr, s, w.ptr, f.L)),
                           "int8 tensor-core product kernel");
                return;
            }
        }
        if constexpr (f32) {
            // fp32 on the persistent bf16x3 GEMM: the fold idct kernel also
            // gathers p's W slots into the GEMM's bf16 A image (no gathered split pass)
            const char* tc = std::getenv("DCTP_TC32");
            const char* bfe = std::getenv("DCTP_TC_BF16");
            if (!(tc && tc[0] == '0') && !(bfe && bfe[0] == '0') &&
                dctp::dev::tc_bf16x3_supported(f.cols, f.L, n, out, true) && f.L % 4 == 0) {
                Scratch<unsigned char> img(dctp::dev::tc_bf16x3_a_bytes(batch, f.cols), s);
                dctp::dev::FoldSlices fs;
                fs.bf = img.ptr;
                fs.map = at<int>(p->blob, f.map);
                fs.K = f.cols;
                cuda_check(DCTP_LAUNCH("fold_idct", s,
                                       dctp::dev::idct_rows<T>(nullptr, 0, in, n, even, w.ptr, f.L, f.L, batch,
                                                               twiddles_at<T>(p->blob, f.tw32), p->flags(s), s, fs)),
                           "fold idct kernel");
                cuda_check(DCTP_LAUNCH("fold_wt_bf16x3", s,
                                       dctp::dev::tc_bf16x3(nullptr, static_cast<int>(n), at<uint16_t>(p->blob, f.wt_bf),
                                                            out, n, batch, f.L, f.cols, p->flags(s), p->num_sms, s,
                                                            nullptr, nullptr, w.ptr, f.L, img.ptr)),
                           "fold bf16x3 kernel");
                return;
            }
        }
        cuda_check(DCTP_LAUNCH("fold_idct", s,
                               dctp::dev::idct_rows<T>(nullptr, 0, in, n, even, w.ptr, f.L, f.L, batch,
                                                       twiddles_at<T>(p->blob, f32 ? f.tw32 : f.tw64), p->flags(s), s)),
                   "fold idct kernel");
        if constexpr (f32) {
            const char* tc = std::getenv("DCTP_TC32");
            const float* th = at<float>(p->blob, f.wt_hi);
            const float* tl = at<float>(p->blob, f.wt_lo);
            const int ldt = (f.cols + 3) / 4 * 4;
            if (!(tc && tc[0] == '0') && f.cols % 4 == 0 &&
                dctp::dev::tc_sgemm3_supported(f.cols, f.L, 4, ldt, n, w.ptr, th, tl, out)) {
                cuda_check(DCTP_LAUNCH("fold_wt_tc32", s,
                                       dctp::dev::tc_sgemm3(in, static_cast<int>(n), th, tl, ldt, out, n, batch, f.L,
                                                            f.cols, p->flags(s), s, nullptr, at<int>(p->blob, f.map), w.ptr,
                                                            f.L, at<float>(p->blob, f.wt_sw))),
                           "fold tcgen05 kernel");
                return;
            }
        }
        cuda_check(DCTP_LAUNCH("fold_wt", s,
                               dctp::dev::rows_by_basis<T>(in, n, at<double>(p->blob, f.wt), f.ldwt, f.cols, f.L, out, n,
                                                           batch, p->flags(s), s, nullptr, at<int>(p->blob, f.map), w.ptr,
                                                           f.L)),
                   "fold product kernel");
        return;
    }
    const std::size_t n = p->st.n;
    DeviceScope scope(p->device);
    Scratch<T> d(batch * n, s);
    if (p->inv.cols > 0)
        cuda_check(DCTP_LAUNCH("cauchy_inv", s,
                               cauchy_stage<T>(in, n, d.ptr, n, p->stage_dev(std::is_same_v<T, float> ? 3 : 2), 1,
                                               p->inv.rows, p->inv.cols, batch, p->flags(s), s)),
                   "cauchy kernel");
    cuda_check(DCTP_LAUNCH("idct", s,
                           dctp::dev::idct_rows<T>(d.ptr, n, in, n, p->emit_inv<T>(), out, n, n, batch, p->tw<T>(),
                                                   p->flags(s), s)),
               "idct kernel");
}

/// Route choice for plans the NFST route can serve (fp64 forward), by
/// measurement on the plan itself: 16 seeded N(0,1) probe signals go through
/// the NFST route and through the exact route the plan would take otherwise.
/// The reference's forward() IS the NFST approximation, so where the two
/// differ by more than 1e-11 (a tenth of the fp64 parity tolerance: at n =
/// 1024, self-loop 0.5, they differ by 5e-9) the NFST route is the only one
/// that reproduces the reference and is kept.  Otherwise the faster one is
/// (tools/route_sweep.py, fully kept plans): the NFST route from
/// DCTP_FAST_MIN_N (default 1024: 0.91 vs 1.08 ms against the dense route at
/// n = 1024, 1.12 vs 2.11 ms at n = 2048) unless the plan has the folded or
/// fused route, which beat it 2-3x at every size.
static void decide_fast_route(dctp_plan& p) {
    if (!p.fs.on) return;
    static const std::size_t min_n = [] {
        const char* m = std::getenv("DCTP_FAST_MIN_N");
        return m ? static_cast<std::size_t>(std::atoll(m)) : std::size_t{1024};
    }();
    const std::size_t n = p.st.n, rows = 16;
    std::vector<double> h(rows * n), a(rows * n), b(rows * n);
    dctp::host::fill_signals(dctp::host::mix_seed(2409, n, 77), dctp::host::Dist::gaussian, 0.0, n, rows, h.data());
    double* d = nullptr;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), 3 * rows * n * sizeof(double)), "cudaMalloc(route probe)");
    std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
    cuda_check(cudaMemcpy(d, h.data(), rows * n * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(route probe)");
    p.fs.preferred = true;
    p.fs.probing = true;
    plan_forward<double>(&p, d, d + rows * n, rows, nullptr);
    p.fs.probing = false;
    p.fs.preferred = false;
    plan_forward<double>(&p, d, d + 2 * rows * n, rows, nullptr);
    cuda_check(cudaMemcpy(a.data(), d + rows * n, rows * n * sizeof(double), cudaMemcpyDeviceToHost), "route probe");
    cuda_check(cudaMemcpy(b.data(), d + 2 * rows * n, rows * n * sizeof(double), cudaMemcpyDeviceToHost),
               "route probe");
    double gap = 0.0;
    for (std::size_t r = 0; r < rows; ++r) {
        double num = 0.0, den = 0.0;
        for (std::size_t k = 0; k < n; ++k) {
            num = std::max(num, std::abs(a[r * n + k] - b[r * n + k]));
            den = std::max(den, std::abs(b[r * n + k]));
        }
        gap = std::max(gap, den > 0.0 ? num / den : num);
    }
    p.fs.probe_gap = gap;
    p.fs.preferred = !(gap <= 1e-11) || (n >= min_n && !p.fd.on && !p.small);
}

/// Page-locked host words of the calling thread for flag read-back (freed at
/// thread exit).
struct PinnedWords {
    int* p = nullptr;
    PinnedWords() {
        if (cudaHostAlloc(reinterpret_cast<void**>(&p), 2 * sizeof(int), cudaHostAllocPortable) != cudaSuccess)
            p = nullptr;
    }
    ~PinnedWords() {
        if (p) cudaFreeHost(p);
    }
};

/// Waits for `s` and raises std::domain_error if a kernel on it (or a
/// captured graph of the object) saw a non-finite sample.  The two flag words
/// are read back by copies queued behind the stream's work, so the call costs
/// one stream synchronisation.
static void sync_check(int device, const StreamFlags& flags, cudaStream_t s) {
    DeviceScope scope(device);
    int* f = flags(s);
    thread_local PinnedWords pw;
    int h = 0, g = 0;
    if (pw.p) {
        cuda_check(cudaMemcpyAsync(pw.p, f, sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(flag)");
        cuda_check(cudaMemcpyAsync(pw.p + 1, flags.graph, sizeof(int), cudaMemcpyDeviceToHost, s),
                   "cudaMemcpyAsync(flag)");
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        h = pw.p[0];
        g = pw.p[1];
    } else {
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        cuda_check(cudaMemcpy(&h, f, sizeof(int), cudaMemcpyDeviceToHost), "cudaMemcpy(flag)");
        cuda_check(cudaMemcpy(&g, flags.graph, sizeof(int), cudaMemcpyDeviceToHost), "cudaMemcpy(flag)");
    }
    if (h != 0 || g != 0) {
        if (h) cuda_check(cudaMemset(f, 0, sizeof(int)), "cudaMemset(flag)");
        if (g) cuda_check(cudaMemset(flags.graph, 0, sizeof(int)), "cudaMemset(flag)");
        throw std::domain_error("DctPlusPlan: non-finite input sample");
    }
}

/// Synchronous host-buffer apply, pipelined over three streams: a copy-in
/// stream (H2D), a compute stream and a copy-out stream (D2H), with a ring of
/// device slots, so the H2D copy of chunk c+1, the kernels of chunk c and the
/// D2H copy of chunk c-1 run at once (PCIe is full duplex; the host buffers
/// must be pinned for the copies to be asynchronous).  Events order slot reuse:
/// H2D into slot k waits for the kernels that read it, the kernels writing
/// slot k wait for the D2H that drained it.
struct HostPipe {
    int device = -1;
    cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
    std::vector<cudaEvent_t> loaded, computed, drained;
    void* buf = nullptr;
    std::size_t buf_bytes = 0;
    // tiny batches (host_tiny): page-locked staging and device rows
    void* tiny_host = nullptr;
    void* tiny_dev = nullptr;

    HostPipe() = default;
    HostPipe(const HostPipe&) = delete;
    HostPipe& operator=(const HostPipe&) = delete;
    ~HostPipe() { // at thread exit; errors ignored (the context may already be gone at process exit)
        int prev = 0;
        if (cudaGetDevice(&prev) != cudaSuccess) return;
        cudaSetDevice(device);
        if (buf) cudaFree(buf);
        if (tiny_dev) cudaFree(tiny_dev);
        if (tiny_host) cudaFreeHost(tiny_host);
        for (auto* v : {&loaded, &computed, &drained})
            for (auto ev : *v) cudaEventDestroy(ev);
        for (cudaStream_t st : {in, comp, out})
            if (st) cudaStreamDestroy(st);
        cudaSetDevice(prev);
        cudaGetLastError();
    }
};

constexpr int kMaxHostSlots = 8;

static HostPipe& host_pipe(int device) {
    thread_local std::vector<std::unique_ptr<HostPipe>> cache; // one per (thread, device), freed at thread exit
    for (auto& e : cache)
        if (e->device == device) return *e;
    auto hp = std::make_unique<HostPipe>();
    hp->device = device;
    for (cudaStream_t* st : {&hp->in, &hp->comp, &hp->out})
        cuda_check(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto* v : {&hp->loaded, &hp->computed, &hp->drained}) {
        v->resize(kMaxHostSlots);
        for (auto& ev : *v) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    }
    cache.push_back(std::move(hp));
    return *cache.back();
}

static std::size_t env_size(const char* name, std::size_t dflt) {
    const char* e = std::getenv(name);
    return e ? static_cast<std::size_t>(std::max(1, std::atoi(e))) : dflt;
}

/// Largest batch (input + output bytes) the tiny host path takes.
constexpr std::size_t kTinyBytes = 256 << 10;

/// Host-buffer apply of a tiny batch (the reference's per-signal call,
/// bench.hpp:139-169): copy into page-locked staging that the kernels read
/// and write in place over PCIe (mapped; no H2D / D2H copy operations), the
/// flag read-back queued behind them, one synchronisation (sync_check), copy
/// out — for rows up to 256 samples; longer rows (whose kernels read the input
/// more than once) stage through device memory with one H2D and one D2H
/// (tools/latency_report.py: C1 / C2 / C3 per-signal 54 / 62 / 97 us through
/// the staged pipeline -> 30 / 32 / 69 us).  DCTP_TINY=0 / copy / map forces
/// off / device staging / mapped staging.  Returns false above kTinyBytes.
template <class T, class F>
static bool host_tiny(int device, const StreamFlags& flags, std::size_t batch, std::size_t in_row,
                      std::size_t out_row, const T* h_in, T* h_out, F&& run) {
    const std::size_t in_b = batch * in_row * sizeof(T), out_b = batch * out_row * sizeof(T);
    if (in_b + out_b > kTinyBytes) return false;
    static const int forced = [] { // -1 auto, 0 off, 1 mapped staging, 2 device staging
        const char* e = std::getenv("DCTP_TINY");
        if (!e) return -1;
        return e[0] == '0' ? 0 : (e[0] == 'c' ? 2 : (e[0] == 'm' ? 1 : -1));
    }();
    if (forced == 0) return false;
    const int mode = forced > 0 ? forced : (in_row <= 256 ? 1 : 2);
    if (!h_in || !h_out) throw std::invalid_argument("host buffer is null");
    DeviceScope scope(device);
    HostPipe& hp = host_pipe(device);
    if (!hp.tiny_host) {
        cuda_check(cudaHostAlloc(&hp.tiny_host, kTinyBytes, cudaHostAllocPortable), "cudaHostAlloc(tiny)");
        cuda_check(cudaMalloc(&hp.tiny_dev, kTinyBytes), "cudaMalloc(tiny)");
    }
    const std::size_t out_off = (in_b + 255) / 256 * 256;
    if (out_off + out_b > kTinyBytes) return false;
    char* hs = static_cast<char*>(hp.tiny_host);
    char* ds = static_cast<char*>(hp.tiny_dev);
    std::memcpy(hs, h_in, in_b);
    if (mode == 1) {
        run(reinterpret_cast<const T*>(hs), reinterpret_cast<T*>(hs + out_off), batch, hp.comp);
    } else {
        cuda_check(cudaMemcpyAsync(ds, hs, in_b, cudaMemcpyHostToDevice, hp.comp), "H2D");
        run(reinterpret_cast<const T*>(ds), reinterpret_cast<T*>(ds + out_off), batch, hp.comp);
        cuda_check(cudaMemcpyAsync(hs + out_off, ds + out_off, out_b, cudaMemcpyDeviceToHost, hp.comp), "D2H");
    }
    sync_check(device, flags, hp.comp);
    std::memcpy(h_out, hs + out_off, out_b);
    return true;
}

template <class T, class F>
static void host_roundtrip(int device, std::size_t batch, std::size_t in_row, std::size_t out_row, const T* h_in,
                           T* h_out, F&& run) {
    if (!h_in || !h_out) throw std::invalid_argument("host buffer is null");
    DeviceScope scope(device);
    // defaults from tools/e2e_probe.py on the B200 box: 16 MB chunks ramping
    // from 4 MB (floor 64 rows), 4 slots — C5 e2e 3.54 -> 3.48 ms, C2 3.24 -> 3.22
    const int slots = static_cast<int>(std::min<std::size_t>(env_size("DCTP_HOST_SLOTS", 4), kMaxHostSlots));
    const std::size_t row_bytes = std::max(in_row, out_row) * sizeof(T);
    const std::size_t floor_rows = env_size("DCTP_HOST_MIN_ROWS", 64);
    const std::size_t max_rows =
        std::max<std::size_t>(floor_rows, (env_size("DCTP_HOST_CHUNK_MB", 16) << 20) / row_bytes); // tuning knobs
    const std::size_t min_rows = std::min(
        max_rows, std::max<std::size_t>(floor_rows, (env_size("DCTP_HOST_CHUNK_MIN_MB", 4) << 20) / row_bytes));
    // Chunk schedule: sizes double from min_rows up to max_rows at the head and
    // mirror that ramp at the tail, so the pipeline fills and drains with small
    // chunks while the middle runs few, large ones (every kernel launch costs a
    // fixed ~20 us while the copy engines are busy; every chunk of the fill
    // and drain costs its own PCIe time).
    std::vector<std::size_t> head, tail;
    {
        std::size_t left = batch, sz = min_rows;
        while (left > 0) {
            head.push_back(std::min(sz, left));
            left -= head.back();
            if (left == 0) break;
            tail.push_back(std::min(sz, left));
            left -= tail.back();
            sz = std::min(2 * sz, max_rows);
        }
        head.insert(head.end(), tail.rbegin(), tail.rend());
    }
    std::size_t rows = 1;
    for (std::size_t r : head) rows = std::max(rows, r);
    HostPipe& hp = host_pipe(device);
    const std::size_t in_elems = rows * in_row, out_elems = rows * out_row;
    const std::size_t slot_bytes = (in_elems + out_elems) * sizeof(T) + 256;
    if (hp.buf_bytes < slot_bytes * slots) {
        if (hp.buf) cuda_check(cudaFree(hp.buf), "cudaFree(host pipe)");
        hp.buf = nullptr;
        hp.buf_bytes = 0;
        cuda_check(cudaMalloc(&hp.buf, slot_bytes * slots), "cudaMalloc(host pipe)");
        hp.buf_bytes = slot_bytes * slots;
    }
    auto slot_in = [&](int k) {
        return reinterpret_cast<T*>(static_cast<char*>(hp.buf) + k * slot_bytes);
    };
    auto slot_out = [&](int k) { // 256-byte aligned after the input rows
        const std::size_t off = (in_elems * sizeof(T) + 255) / 256 * 256;
        return reinterpret_cast<T*>(static_cast<char*>(hp.buf) + k * slot_bytes + off);
    };
    std::size_t r0 = 0;
    for (std::size_t c = 0; c < head.size(); r0 += head[c], ++c) {
        const std::size_t nr = head[c];
        const int k = static_cast<int>(c % slots);
        const bool reuse = c >= static_cast<std::size_t>(slots);
        if (reuse) cuda_check(cudaStreamWaitEvent(hp.in, hp.computed[k], 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(slot_in(k), h_in + r0 * in_row, nr * in_row * sizeof(T), cudaMemcpyHostToDevice,
                                   hp.in),
                   "H2D");
        cuda_check(cudaEventRecord(hp.loaded[k], hp.in), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(hp.comp, hp.loaded[k], 0), "cudaStreamWaitEvent");
        if (reuse) cuda_check(cudaStreamWaitEvent(hp.comp, hp.drained[k], 0), "cudaStreamWaitEvent");
        run(slot_in(k), slot_out(k), nr, hp.comp);
        cuda_check(cudaEventRecord(hp.computed[k], hp.comp), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(hp.out, hp.computed[k], 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(h_out + r0 * out_row, slot_out(k), nr * out_row * sizeof(T),
                                   cudaMemcpyDeviceToHost, hp.out),
                   "D2H");
        cuda_check(cudaEventRecord(hp.drained[k], hp.out), "cudaEventRecord");
    }
    for (cudaStream_t st : {hp.in, hp.comp, hp.out}) cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

/// The plan's orthonormal basis X (row-major n x n: slot s = sum_i X[i][s] x_i),
/// column by column from the secular formula and one inverse DCT (the
/// reference's assemble_unsigned_basis, cauchy.hpp:84-103, with the sigma signs).
static void plan_basis(const dctp::host::Setup& st, double* x) {
    const std::size_t n = st.n;
    const dctp::host::Trig idct(dctp::host::Trig::Kind::idct2, n);
    dctp::host::parallel_for(n, [&](std::size_t s) {
        std::vector<double> buf(2 * n + idct.scratch_size() + 1);
        double* y = buf.data();
        double* col = y + n;
        dctp::host::basis_coefficients(st, s, y);
        idct.execute(y, col, col + n);
        for (std::size_t i = 0; i < n; ++i) x[i * n + s] = st.sigma[s] < 0.0 ? -col[i] : col[i];
    }, 4);
}

/// Materialises X^T and X on the device once per plan: the signed basis rows
/// in the DCT domain (the setup's a, z, nu, sigma), one batched DCT-III over
/// them (X^T row s = column s of X), and a transpose.
static void ensure_dense(const dctp_plan* p, cudaStream_t s) {
    auto& d = *p->dense;
    std::lock_guard<std::mutex> lock(d.mu);
    if (d.buf) return;
    const auto& st = p->st;
    const std::size_t n = st.n, ld = (n + 3) / 4 * 4;
    std::vector<double> tab(5 * n, 0.0); // z, lambda, nu, a, sigma
    std::vector<int> pidx(n);
    for (std::size_t q = 0; q < n; ++q) {
        tab[q] = st.z[q];
        tab[n + q] = st.lambda[q];
        const auto& sl = st.slots[q];
        pidx[q] = sl.passthrough ? static_cast<int>(sl.idx) : -1;
        tab[2 * n + q] = sl.passthrough ? 0.0 : st.sub_mu[sl.idx];
        tab[3 * n + q] = st.a[q];
        tab[4 * n + q] = st.sigma[q];
    }
    double* buf = nullptr;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&buf), 2 * n * ld * sizeof(double)), "cudaMalloc(basis)");
    Scratch<double> y(n * ld + 5 * n + (n + 1) / 2, s);
    double* dtab = y.ptr + n * ld;
    int* dp = reinterpret_cast<int*>(dtab + 5 * n);
    cuda_check(cudaMemsetAsync(buf, 0, 2 * n * ld * sizeof(double), s), "cudaMemset(basis)");
    cuda_check(cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(dp, pidx.data(), n * sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
    const int ni = static_cast<int>(n);
    cuda_check(dctp::dev::basis_coefficients(ni, ld, dtab, dtab + n, dtab + 2 * n, dp, dtab + 3 * n, dtab + 4 * n,
                                             y.ptr, s),
               "basis kernel");
    cuda_check(dctp::dev::idct_rows<double>(y.ptr, ld, y.ptr, ld, dctp::dev::Emit<double>{}, buf, ld, n, n,
                                            p->tw<double>(), p->flags(s), s),
               "basis idct kernel");
    cuda_check(dctp::dev::transpose_square(buf, ld, buf + n * ld, ld, ni, s), "transpose kernel");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(basis)");
    d.ld = ld;
    d.buf = buf;
}

/// The dense route replaces DCT + Cauchy when the structured work is close
/// to a full n x n product anyway (K A >= 0.8 n^2, e.g. general directions):
/// reading a stored X^T runs the tensor cores at ~88% against ~71% when the
/// Cauchy block is generated, and the DCT pass disappears.  X^T and X cost
/// 16 n^2 bytes of HBM.  DCTP_DENSE=0 / 1 forces the choice.
static bool dense_route(const dctp_plan* p) {
    const char* e = std::getenv("DCTP_DENSE");
    if (p->small && !(e && e[0] == '1')) return false;
    if (e && e[0] == '0') return false;
    const double n = static_cast<double>(p->st.n);
    if (16.0 * n * n > 4.0 * (1ull << 30)) return false;
    if (e && e[0] == '1') return true;
    return n * n <= 1.25 * static_cast<double>(p->fwd.rows) * static_cast<double>(p->fwd.cols);
}

/// fp64 dense products on the int8 tensor cores (ozaki.cu) from n = 1024
/// (below that the DMMA product is short and the extra slicing pass over the
/// input does not pay).  DCTP_OZAKI=0 keeps the DMMA product; the slice count
/// (DCTP_OZAKI_SLICES, 5 = default or 6) trades products (15 / 21) for
/// accuracy: 2.9e-11 / ~1e-13 norm-wise per signal on the whole C5 batch
/// against the DMMA product (fp64 tolerance 1e-10).
static int ozaki_slices(std::size_t n) {
    static const int slices = [] {
        const char* e = std::getenv("DCTP_OZAKI_SLICES");
        const int v = e ? std::atoi(e) : 5;
        return (v == 5 || v == 6) ? v : 5;
    }();
    const char* e = std::getenv("DCTP_OZAKI");
    if (e && e[0] == '0') return 0;
    if (e && e[0] == '1') return n <= 16384 ? slices : 0;
    return (n >= 1024 && n <= 16384) ? slices : 0;
}

/// int8 slices of X^T (which = 0) or X (which = 1), once per plan.
static std::pair<int8_t*, int*> slice_operand(const double* bt, std::size_t ld, std::size_t rows, int K, int S,
                                              cudaStream_t s);
static void ensure_ozaki(const dctp_plan* p, int which, int S, cudaStream_t s) {
    auto& d = *p->dense;
    std::lock_guard<std::mutex> lock(d.mu);
    if (d.oz[which] && d.oz_slices == S) return;
    for (int i = 0; i < 2; ++i) // a different slice count invalidates both
        if (d.oz[i] && d.oz_slices != S) {
            cudaFree(d.oz[i]);
            cudaFree(d.oz_e[i]);
            d.oz[i] = nullptr;
            d.oz_e[i] = nullptr;
        }
    const std::size_t n = p->st.n;
    auto [sl, ex] = slice_operand(d.buf + (which ? n * d.ld : 0), d.ld, n, static_cast<int>(n), S, s);
    d.oz[which] = sl;
    d.oz_e[which] = ex;
    d.oz_slices = S;
}

static void ensure_fold_grouped(const dctp_plan* p, int v, int S, cudaStream_t s) {
    auto& f = const_cast<dctp_plan*>(p)->fd;
    std::lock_guard<std::mutex> lock(p->dense->mu);
    if (f.g_sl[v]) return;
    auto [sl, ex] = slice_operand(at<double>(p->blob, f.g_b[v]), 2 * static_cast<std::size_t>(f.L),
                                  static_cast<std::size_t>(f.g_rows[v]), 2 * f.L, S, s);
    f.g_sl[v] = sl;
    f.g_e[v] = ex;
}

/// int8 slices of the folded route's W (which = 0, cols x L) or W^T (which =
/// 1, L x cols), once per plan.
static void ensure_fold_ozaki(const dctp_plan* p, int which, int S, cudaStream_t s) {
    auto& f = const_cast<dctp_plan*>(p)->fd;
    std::lock_guard<std::mutex> lock(p->dense->mu);
    if (f.oz[which] && f.oz_slices == S) return;
    for (int i = 0; i < 2; ++i)
        if (f.oz[i] && f.oz_slices != S) {
            cudaFree(f.oz[i]);
            cudaFree(f.oz_e[i]);
            f.oz[i] = nullptr;
            f.oz_e[i] = nullptr;
        }
    auto [sl, ex] = which == 0 ? slice_operand(at<double>(p->blob, f.w), f.ldw, f.cols, f.L, S, s)
                               : slice_operand(at<double>(p->blob, f.wt), f.ldwt, f.L, f.cols, S, s);
    f.oz[which] = sl;
    f.oz_e[which] = ex;
    f.oz_slices = S;
}

/// out[b, c] = sum_k in[b, k] bt[c, k] with bt given as int8 slices: slice
/// the signal rows (columns gathered through a_map) into stream-ordered
/// scratch, then one tcgen05 kind::i8 GEMM (col_map / fold_add epilogues as
/// in rows_by_basis).
static void rows_by_ozaki(const double* in, std::size_t ld_in, const int8_t* b_sl, const int* eb, int K, int N,
                          int S, double* out, std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t s,
                          const char* name, const int* col_map, const int* a_map, const double* fold_add,
                          std::size_t ld_add) {
    const int pm = dctp::dev::ozaki_pad_m();
    const std::size_t a_bytes = dctp::dev::ozaki_slice_bytes(batch, K, 128, S, pm);
    const std::size_t rows_pad = (batch + pm - 1) / pm * pm;
    Scratch<int8_t> a_sl(a_bytes, s);
    Scratch<int> ea(rows_pad, s);
    cuda_check(DCTP_LAUNCH("ozaki_slice", s,
                           dctp::dev::ozaki_slice<double>(in, ld_in, batch, K, a_map, 128, S, a_sl.ptr, ea.ptr, flag,
                                                          s, pm)),
               "signal slicing kernel");
    cuda_check(DCTP_LAUNCH(name, s,
                           dctp::dev::ozaki_gemm(a_sl.ptr, ea.ptr, b_sl, eb, batch, N, K, S, out, ld_out, col_map, s,
                                                 fold_add, ld_add)),
               "int8 tensor-core product kernel");
}

/// int8 slices of an operand matrix bt (rows x K, stride ld) for the B side
/// of ozaki_gemm; (slices, exponents) in device memory owned by the caller.
/// The NFST route on the int8 tensor cores: its forward (and adjoint
/// inverse) is a fixed linear map of the signal — DCT, weights, DST-I,
/// Gaussian-gridding taps, all linear — so it is materialised once per plan
/// as the n x n operator F (row i = the NFST kernel applied to e_i: the same
/// kernel, so F carries the reference's own NFST approximation and the
/// result stays on the reference's fast route, fast_transform.hpp:163-190)
/// and applied as out = in F on the kind::i8 product.  At n = 1024 / 2048
/// that is 0.26 / 0.42 ms per batch (X7 / X8) against 0.91 / 1.02 ms in the
/// one-signal-per-CTA NFST kernel, whose FFT and tap passes run at ~15% of
/// the fp64 pipe; the dense product costs n^2 per signal against the NFST's
/// n log n, so it stops paying past n = 4096 (DCTP_NFST_DENSE_MAX_N).  The
/// adjoint (which = 1) takes 6 slices: its map amplifies the product's
/// rounding (n = 2048, self-loop 5.0: 1.0e-10 from the reference with 5
/// slices, at the tolerance).  DCTP_NFST_DENSE = 0 keeps the NFST kernel.
static int nfst_dense_slices(const dctp_plan* p, int which) {
    const char* e = std::getenv("DCTP_NFST_DENSE");
    if (p->fs.probing || (e && e[0] == '0')) return 0;
    const char* m = std::getenv("DCTP_NFST_DENSE_MAX_N");
    const std::size_t max_n = m ? static_cast<std::size_t>(std::atoll(m)) : std::size_t{4096};
    const int S = p->st.n <= max_n ? ozaki_slices(p->st.n) : 0;
    return S && which == 1 ? 6 : S;
}

static void ensure_nfst_ozaki(const dctp_plan* p, int which, int S, cudaStream_t s) {
    auto& d = *p->dense;
    std::lock_guard<std::mutex> lock(d.mu);
    if (d.nf[which] && d.nf_slices[which] == S) return;
    if (d.nf[which]) {
        cudaFree(d.nf[which]);
        cudaFree(d.nf_e[which]);
        d.nf[which] = nullptr;
        d.nf_e[which] = nullptr;
    }
    const std::size_t n = p->st.n;
    Scratch<double> eye(n * n, s), img(n * n, s);
    Scratch<int> flag(1, s);
    cuda_check(cudaMemsetAsync(eye.ptr, 0, n * n * sizeof(double), s), "cudaMemset(identity)");
    cuda_check(cudaMemsetAsync(flag.ptr, 0, sizeof(int), s), "cudaMemset(flag)");
    const std::vector<double> ones(n, 1.0); // the diagonal: one strided 2-D copy
    cuda_check(cudaMemcpy2DAsync(eye.ptr, (n + 1) * sizeof(double), ones.data(), sizeof(double), sizeof(double), n,
                                 cudaMemcpyHostToDevice, s),
               "H2D(identity)");
    cuda_check(dctp::dev::nfst_apply(eye.ptr, img.ptr, n, fast_plan_dev(p), flag.ptr, which == 1, s),
               "nfst operator kernel");
    const int ni = static_cast<int>(n);
    cuda_check(dctp::dev::transpose_square(img.ptr, n, eye.ptr, n, ni, s), "transpose kernel"); // bt = F^T
    auto [sl, ex] = slice_operand(eye.ptr, n, n, ni, S, s); // synchronises s (the host vector may go)
    d.nf[which] = sl;
    d.nf_e[which] = ex;
    d.nf_slices[which] = S;
}

static std::pair<int8_t*, int*> slice_operand(const double* bt, std::size_t ld, std::size_t rows, int K, int S,
                                              cudaStream_t s) {
    const int tn = dctp::dev::ozaki_tile_n(S), pn = dctp::dev::ozaki_pad_n(S);
    int8_t* sl = nullptr;
    int* ex = nullptr;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&sl), dctp::dev::ozaki_slice_bytes(rows, K, tn, S, pn)),
               "cudaMalloc(operand slices)");
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&ex), (rows + pn - 1) / pn * pn * sizeof(int)),
               "cudaMalloc(operand exponents)");
    cuda_check(dctp::dev::ozaki_slice<double>(bt, ld, rows, K, nullptr, tn, S, sl, ex, nullptr, s, pn),
               "operand slicing kernel");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(operand slices)");
    return {sl, ex};
}

/// The dense routes of DctPlusPlan: forward_nmvp = X^T s (fast_transform.hpp:
/// 199-214) and inverse(p, fast = false) = X p (:218-260), as one product with
/// the materialised basis on the DMMA tensor cores (rows_by_basis).
template <class T>
static void plan_dense(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s, bool inverse) {
    if (!p) throw std::invalid_argument("dctp_*_nmvp: null plan");
    if (!p->blob) throw std::invalid_argument("DctPlusPlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("dctp_*_nmvp: null buffer");
    if (static_cast<const void*>(in) == static_cast<const void*>(out))
        throw std::invalid_argument("dctp_*_nmvp: in and out must not alias");
    const std::size_t n = p->st.n;
    DeviceScope scope(p->device);
    ensure_dense(p, s);
    const auto& d = *p->dense;
    const double* bt = d.buf + (inverse ? n * d.ld : 0);
    const int ni = static_cast<int>(n);
    if constexpr (std::is_same_v<T, double>) {
        if (const int S = ozaki_slices(n)) {
            ensure_ozaki(p, inverse ? 1 : 0, S, s);
            rows_by_ozaki(in, n, d.oz[inverse ? 1 : 0], d.oz_e[inverse ? 1 : 0], ni, ni, S, out, n, batch, p->flags(s),
                          s, inverse ? "dense_inv_i8" : "dense_i8");
            return;
        }
    }
    cuda_check(DCTP_LAUNCH(inverse ? "dense_inv" : "dense_nmvp", s,
                           dctp::dev::rows_by_basis<T>(in, n, bt, d.ld, ni, ni, out, n, batch, p->flags(s), s)),
               "dense basis kernel");
}
template <class T>
static void plan_nmvp(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    plan_dense<T>(p, in, out, batch, s, false);
}
template <class T>
static void plan_inverse_dense(const dctp_plan* p, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    plan_dense<T>(p, in, out, batch, s, true);
}

// --- ensemble ------------------------------------------------------------------

struct dctp_ensemble {
    std::size_t n = 0, cp = 0;
    double threshold = 0.0;
    int device = 0;
    std::vector<std::unique_ptr<dctp_plan>> members;
    void* blob = nullptr;
    StreamFlags flags;
    TwiddleOffsets tw64, tw32;
    std::size_t to = 0, from = 0, sign64 = 0, sign32 = 0, desc64 = 0, desc32 = 0;
    int n_emit = 0, max_rows = 0, max_cols = 0;
    // fp32 dense route (n <= 256): G = [D^T | X_1 | ... | X_K], n x (K+1) n
    std::size_t gmat32 = 0;
    std::size_t gt_hi = 0, gt_lo = 0; // G^T split for the tcgen05 3xTF32 GEMM, (K+1) n x n
    std::size_t gt_sw = 0;            // the same, in the kernel's swizzled shared-memory blocks
    std::size_t gt_bf = 0;            // G^T split bf16 hi / lo for the persistent bf16x3 GEMM (tc_bf16x3.cu)
    int num_sms = 0;
    bool dense32 = false;
    // pruned mode (c_p < n): [UL_r; HL_r] = T_r[:, 0:c_p] per member, K x n x c_p
    std::size_t prune64 = 0, prune32 = 0;

    ~dctp_ensemble() {
        if (blob) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            cudaFree(blob);
            cudaSetDevice(prev);
        }
    }
};

template <class T>
static void ensemble_forward_full(const dctp_ensemble* e, const T* in, T* out, std::size_t batch, cudaStream_t s);

/// forward_all (fast_transform.hpp:396-439) for a batch: every set of every
/// signal through the full progressive path, then (c_p < n) the pruned
/// signals rewritten in place; `bounds` (batch x (K+1)) and `pruned` (batch)
/// are optional outputs.
template <class T>
static void ensemble_forward(const dctp_ensemble* e, const T* in, T* out, std::size_t batch, cudaStream_t s,
                             T* bounds = nullptr, unsigned char* pruned = nullptr) {
    ensemble_forward_full<T>(e, in, out, batch, s);
    if (batch == 0 || (e->cp >= e->n && !bounds && !pruned)) return;
    DeviceScope scope(e->device);
    constexpr bool f32 = std::is_same_v<T, float>;
    const T* blocks = e->cp < e->n ? at<T>(e->blob, f32 ? e->prune32 : e->prune64) : nullptr;
    cuda_check(DCTP_LAUNCH("ensemble_prune", s,
                           dctp::dev::ensemble_prune<T>(in, out, blocks, e->n, e->cp,
                                                        static_cast<int>(e->members.size()), e->threshold, batch,
                                                        bounds, pruned, s)),
               "prune kernel");
}

template <class T>
static void ensemble_forward_full(const dctp_ensemble* e, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    if (!e) throw std::invalid_argument("dctp_ensemble_forward_all: null ensemble");
    if (!e->blob) throw std::invalid_argument("PrunedEnsemblePlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("dctp_ensemble_forward_all: null buffer");
    const std::size_t n = e->n, sets = e->members.size() + 1, ld = sets * n;
    DeviceScope scope(e->device);
    constexpr bool f32 = std::is_same_v<T, float>;
    dctp::dev::Emit<T> emit{at<int>(e->blob, e->to), at<int>(e->blob, e->from), nullptr, e->n_emit};
    dctp::dev::Twiddles<T> tw;
    if constexpr (f32) {
        emit.sign = at<float>(e->blob, e->sign32);
        tw = twiddles_at<float>(e->blob, e->tw32);
    } else {
        emit.sign = at<double>(e->blob, e->sign64);
        tw = twiddles_at<double>(e->blob, e->tw64);
    }
    if constexpr (f32) {
        // the persistent bf16x3 tensor-core GEMM (n <= 128), else the tcgen05
        // 3xTF32 GEMM, unless DCTP_TC32=0 (FFMA SGEMM) / DCTP_TC_BF16=0
        const char* tc = std::getenv("DCTP_TC32");
        const char* bfe = std::getenv("DCTP_TC_BF16");
        if (e->dense32 && !(tc && tc[0] == '0') && !(bfe && bfe[0] == '0') &&
            dctp::dev::tc_bf16x3_supported(static_cast<int>(n), static_cast<int>(ld), ld, out) &&
            reinterpret_cast<std::uintptr_t>(in) % 16 == 0) {
            cuda_check(DCTP_LAUNCH("progressive_bf16x3", s,
                                   dctp::dev::tc_bf16x3(in, static_cast<int>(n), at<uint16_t>(e->blob, e->gt_bf), out,
                                                        ld, batch, static_cast<int>(ld), static_cast<int>(n),
                                                        e->flags(s), e->num_sms, s)),
                       "progressive bf16x3 kernel");
            return;
        }
        if (e->dense32 && !(tc && tc[0] == '0') &&
            dctp::dev::tc_sgemm3_supported(static_cast<int>(n), static_cast<int>(ld), static_cast<int>(n),
                                           static_cast<int>(n), ld, in, at<float>(e->blob, e->gt_hi),
                                           at<float>(e->blob, e->gt_lo), out)) {
            cuda_check(DCTP_LAUNCH("progressive_tc32", s,
                                   dctp::dev::tc_sgemm3(in, static_cast<int>(n), at<float>(e->blob, e->gt_hi),
                                                        at<float>(e->blob, e->gt_lo), static_cast<int>(n), out, ld,
                                                        batch, static_cast<int>(ld), static_cast<int>(n), e->flags(s), s,
                                                        nullptr, nullptr, nullptr, 0,
                                                        at<float>(e->blob, e->gt_sw))),
                       "progressive tcgen05 kernel");
            return;
        }
        if (e->dense32 &&
            dctp::dev::sgemm_rows_supported(static_cast<int>(n), static_cast<int>(ld), static_cast<int>(n),
                                            static_cast<int>(ld), ld, in, at<float>(e->blob, e->gmat32), out)) {
            cuda_check(DCTP_LAUNCH("progressive_sgemm", s,
                                   dctp::dev::sgemm_rows(in, static_cast<int>(n), at<float>(e->blob, e->gmat32),
                                                         static_cast<int>(ld), out, ld, batch, static_cast<int>(ld),
                                                         static_cast<int>(n), e->flags(s), s)),
                       "progressive sgemm kernel");
            return;
        }
    }
    // Set 0 (the shared DCT, fast_transform.hpp:401-403) is written in place
    // and is the Cauchy stages' input; sets 1..K follow in each row.
    cuda_check(DCTP_LAUNCH("dct2", s, dctp::dev::dct2_rows<T>(in, n, out, ld, out, ld, emit, n, batch, tw, e->flags(s), s)),
               "dct2 kernel");
    if (!e->members.empty() && e->max_cols > 0)
        cuda_check(DCTP_LAUNCH("cauchy_progressive", s,
                               cauchy_stage<T>(out, ld, out, ld,
                                               at<dctp::dev::CauchyStage>(e->blob, f32 ? e->desc32 : e->desc64),
                                               static_cast<int>(e->members.size()), e->max_rows, e->max_cols, batch,
                                               e->flags(s), s)),
                   "cauchy kernel");
}

// ---------------------------------------------------------------------------

extern "C" {

const char* dctp_last_error(void) { return g_last_error.c_str(); }

const char* dctp_version(void) { return "dctplus_b200 0.1 (sm_100a)"; }

int dctp_plan_create(size_t n, int kind, size_t i, size_t j, double rho, const double* v, double epsilon,
                     double tau, int device, dctp_plan** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("dctp_plan_create: null output");
        *out = nullptr;
        if (n < 2) throw std::invalid_argument("DctPlusPlan: need n >= 2");
        auto p = build_plan(n, make_update(kind, i, j, rho, v, n), epsilon, tau, device);
        if (device >= 0 && dense_route(p.get())) { // the dense route's X^T and X are part of the setup
            DeviceScope scope(device);
            ensure_dense(p.get(), nullptr);
        }
        *out = p.release();
    });
}

int dctp_plan_destroy(dctp_plan* plan) {
    return guarded([&] { delete plan; });
}

int dctp_plan_info(const dctp_plan* p, size_t* n, double* epsilon, int* slow_path, size_t* n_kept,
                   size_t* n_active, int* device) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_info: null plan");
        if (n) *n = p->st.n;
        if (epsilon) *epsilon = p->st.epsilon;
        if (slow_path) *slow_path = p->st.slow_path ? 1 : 0;
        if (n_kept) *n_kept = p->st.kept.size();
        if (n_active) *n_active = p->st.sub_mu.size();
        if (device) *device = p->device;
    });
}

int dctp_plan_route(const dctp_plan* p, int* nfst, double* probe_gap) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_route: null plan");
        if (nfst) *nfst = fast_route(p) ? 1 : 0;
        if (probe_gap) *probe_gap = p->fs.probe_gap;
    });
}

int dctp_ozaki_slices(std::size_t n, int* slices) {
    return guarded([&] {
        if (!slices) throw std::invalid_argument("dctp_ozaki_slices: null output");
        *slices = ozaki_slices(n);
    });
}

int dctp_plan_setup(const dctp_plan* p, double* lambda, double* mu, double* z, double* a, double* sigma) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_setup: null plan");
        const auto& st = p->st;
        if (lambda) std::copy(st.lambda.begin(), st.lambda.end(), lambda);
        if (mu) std::copy(st.mu.begin(), st.mu.end(), mu);
        if (z) std::copy(st.z.begin(), st.z.end(), z);
        if (a) std::copy(st.a.begin(), st.a.end(), a);
        if (sigma) std::copy(st.sigma.begin(), st.sigma.end(), sigma);
    });
}

int dctp_plan_slots(const dctp_plan* p, int* passthrough, int64_t* idx) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_slots: null plan");
        for (std::size_t s = 0; s < p->st.slots.size(); ++s) {
            if (passthrough) passthrough[s] = p->st.slots[s].passthrough ? 1 : 0;
            if (idx) idx[s] = static_cast<int64_t>(p->st.slots[s].idx);
        }
    });
}

int dctp_plan_subproblem(const dctp_plan* p, size_t* k, double* sub_lambda, double* sub_z, double* sub_mu,
                         double* rho) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_subproblem: null plan");
        const auto& st = p->st;
        if (k) *k = st.kept.size();
        if (rho) *rho = st.rho;
        for (std::size_t q = 0; q < st.kept.size(); ++q) {
            if (sub_lambda) sub_lambda[q] = st.lambda[st.kept[q]];
            if (sub_z) sub_z[q] = st.z[st.kept[q]];
        }
        if (sub_mu) std::copy(st.sub_mu.begin(), st.sub_mu.end(), sub_mu);
    });
}

int dctp_plan_basis(const dctp_plan* p, double* x) {
    return guarded([&] {
        if (!p || !x) throw std::invalid_argument("dctp_plan_basis: null argument");
        plan_basis(p->st, x);
    });
}

int dctp_forward_f64(const dctp_plan* p, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { plan_forward<double>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_forward_f32(const dctp_plan* p, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { plan_forward<float>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_inverse_f64(const dctp_plan* p, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { plan_inverse<double>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_inverse_f32(const dctp_plan* p, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { plan_inverse<float>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}

int dctp_forward_nmvp_f64(const dctp_plan* p, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { plan_nmvp<double>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_forward_nmvp_f32(const dctp_plan* p, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { plan_nmvp<float>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_inverse_nmvp_f64(const dctp_plan* p, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { plan_inverse_dense<double>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_inverse_nmvp_f32(const dctp_plan* p, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { plan_inverse_dense<float>(p, in, out, batch, static_cast<cudaStream_t>(stream)); });
}

int dctp_plan_sync_check(const dctp_plan* p, void* stream) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("dctp_plan_sync_check: null plan");
        sync_check(p->device, p->flags, static_cast<cudaStream_t>(stream));
    });
}

} // extern "C"

/// True when [p, p + bytes) lies inside one page-locked host allocation that
/// device `device` can address (UVA-mapped): the same buffer id at both ends.
static bool pinned_range(const void* p, std::size_t bytes, int device) {
    cudaPointerAttributes a{}, b{};
    const void* last = static_cast<const char*>(p) + bytes - 1;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess || cudaPointerGetAttributes(&b, last) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || a.devicePointer != p || a.device != device)
        return false;
    using GetAttr = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
    static GetAttr get = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return static_cast<GetAttr>(nullptr);
        }
        return reinterpret_cast<GetAttr>(fn);
    }();
    if (!get) return false;
    unsigned long long id0 = 0, id1 = 0;
    if (get(&id0, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS ||
        get(&id1, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(last)) != CUDA_SUCCESS)
        return false;
    return id0 == id1;
}

/// Small host batches of fused plans: the kernel's TMA bulk copies read and
/// write the page-locked host rows directly over PCIe (zero copy).  For a few
/// MB this halves the latency of staged H2D / kernel / D2H (every copy and
/// stream hop costs tens of microseconds there; tools/small_e2e_probe.py);
/// above DCTP_ZC_MAX_MB (default 8) the staged pipeline moves more bytes/s.
static bool forward_zero_copy(const dctp_plan*, const float*, float*, std::size_t) { return false; }
static bool forward_zero_copy(const dctp_plan* p, const double* h_in, double* h_out, std::size_t batch) {
    if (!p->small || !h_in || !h_out) return false;
    const char* off = std::getenv("DCTP_ZERO_COPY");
    if (off && off[0] == '0') return false;
    const std::size_t bytes = batch * p->st.n * sizeof(double);
    if (bytes > (env_size("DCTP_ZC_MAX_MB", 8) << 20)) return false;
    if ((reinterpret_cast<std::uintptr_t>(h_in) | reinterpret_cast<std::uintptr_t>(h_out)) % 16 != 0) return false;
    DeviceScope scope(p->device);
    if (!pinned_range(h_in, bytes, p->device) || !pinned_range(h_out, bytes, p->device)) return false;
    HostPipe& hp = host_pipe(p->device);
    plan_forward<double>(p, h_in, h_out, batch, hp.comp);
    sync_check(p->device, p->flags, hp.comp);
    return true;
}

extern "C" {

#define DCTP_HOST_ENTRY(NAME, T, FN, ZC)                                                            \
    int NAME(const dctp_plan* p, const T* h_in, T* h_out, size_t batch) {                             \
        return guarded([&] {                                                                          \
            if (!p) throw std::invalid_argument(#NAME ": null plan");                                 \
            if (!p->blob) throw std::invalid_argument("DctPlusPlan: host-only plan (created with device < 0)"); \
            if (batch == 0) return;                                                                   \
            const std::size_t n = p->st.n;                                                           \
            if (ZC && forward_zero_copy(p, h_in, h_out, batch)) return;                               \
            auto fn = [&](const T* din, T* dout, std::size_t rows, cudaStream_t s) { FN<T>(p, din, dout, rows, s); }; \
            if (host_tiny<T>(p->device, p->flags, batch, n, n, h_in, h_out, fn)) return;              \
            host_roundtrip<T>(p->device, batch, n, n, h_in, h_out,                                    \
                              [&](const T* din, T* dout, std::size_t rows, cudaStream_t s) {         \
                                  FN<T>(p, din, dout, rows, s);                                       \
                              });                                                                     \
            sync_check(p->device, p->flags, host_pipe(p->device).comp);                                                  \
        });                                                                                           \
    }
DCTP_HOST_ENTRY(dctp_forward_host_f64, double, plan_forward, true)
DCTP_HOST_ENTRY(dctp_forward_host_f32, float, plan_forward, false)
DCTP_HOST_ENTRY(dctp_inverse_host_f64, double, plan_inverse, false)
DCTP_HOST_ENTRY(dctp_inverse_host_f32, float, plan_inverse, false)
DCTP_HOST_ENTRY(dctp_forward_nmvp_host_f64, double, plan_nmvp, false)
DCTP_HOST_ENTRY(dctp_forward_nmvp_host_f32, float, plan_nmvp, false)
DCTP_HOST_ENTRY(dctp_inverse_nmvp_host_f64, double, plan_inverse_dense, false)
DCTP_HOST_ENTRY(dctp_inverse_nmvp_host_f32, float, plan_inverse_dense, false)
#undef DCTP_HOST_ENTRY

int dctp_ensemble_create(size_t n, size_t k, const int* kinds, const size_t* is, const size_t* js, const double* rhos,
                         const double* vs, size_t cp, double threshold, double epsilon, int device,
                         dctp_ensemble** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("dctp_ensemble_create: null output");
        *out = nullptr;
        if (cp < 1 || cp > n) throw std::invalid_argument("PrunedEnsemblePlan: need 1 <= c_p <= n");
        if (k > 0 && (!kinds || !is || !js || !rhos)) throw std::invalid_argument("dctp_ensemble_create: null update arrays");
        auto e = std::make_unique<dctp_ensemble>();
        e->n = n;
        e->cp = cp;
        e->threshold = threshold;
        e->device = device;
        for (std::size_t r = 0; r < k; ++r)
            e->members.push_back(build_plan(
                n, make_update(kinds[r], is[r], js[r], rhos[r], vs ? vs + r * n : nullptr, n), epsilon, 1e-12, device));
        // Twiddles, the merged pass-through emit list and one stage per member.
        Blob blob;
        e->tw64 = add_twiddles<double>(blob, n);
        e->tw32 = add_twiddles<float>(blob, n);
        std::vector<int> to, from;
        std::vector<double> sign;
        std::vector<ApplyTables> tabs;
        for (std::size_t r = 0; r < k; ++r) {
            tabs.push_back(make_tables(e->members[r]->st));
            const auto& t = tabs.back();
            for (std::size_t q = 0; q < t.pass_slot.size(); ++q) {
                to.push_back(static_cast<int>((r + 1) * n) + t.pass_slot[q]);
                from.push_back(t.pass_src[q]);
                sign.push_back(t.pass_sign[q]);
            }
        }
        e->to = blob.add(to);
        e->from = blob.add(from);
        e->sign64 = blob.add(sign);
        e->sign32 = blob.add(to_f32(sign));
        e->n_emit = static_cast<int>(to.size());
        std::vector<StageOffsets> st(k);
        for (std::size_t r = 0; r < k; ++r) {
            const auto& t = tabs[r];
            bool contig = true;
            for (std::size_t k = 0; k < t.kept_idx.size(); ++k) contig = contig && t.kept_idx[k] == static_cast<int>(k);
            st[r] = {blob.add(t.kept_idx), blob.add(t.lam_kept), blob.add(t.z_kept), blob.add(to_f32(t.z_kept)),
                     blob.add(t.act_slot), blob.add(t.nu), blob.add(t.act_scale), blob.add(to_f32(t.act_scale)),
                     static_cast<int>(t.kept_idx.size()), static_cast<int>(t.nu.size()), contig ? 1 : 0};
            e->max_rows = std::max(e->max_rows, st[r].rows);
            e->max_cols = std::max(e->max_cols, st[r].cols);
        }
        e->desc64 = blob.add(std::vector<dctp::dev::CauchyStage>(k));
        e->desc32 = blob.add(std::vector<dctp::dev::CauchyStage>(k));
        if (cp < n) {
            // T_r rows exactly as the reference builds them (fast_transform.hpp:355-366):
            // pass-through slot -> sigma at its DCT index, active slot s ->
            // -sigma_s a_s z_j / (nu_s - lambda_j); keep the first c_p columns.
            std::vector<double> blk(k * n * cp, 0.0);
            for (std::size_t r = 0; r < k; ++r) {
                const auto& st = e->members[r]->st;
                double* b = blk.data() + r * n * cp;
                for (std::size_t slot = 0; slot < n; ++slot) {
                    const auto& ref = st.slots[slot];
                    if (ref.passthrough) {
                        if (ref.idx < cp) b[slot * cp + ref.idx] = st.sigma[slot];
                        continue;
                    }
                    const double nu = st.sub_mu[ref.idx];
                    const double sc = -st.sigma[slot] * st.a[slot];
                    for (std::size_t j = 0; j < cp; ++j)
                        if (st.z[j] != 0.0) b[slot * cp + j] = sc * st.z[j] / (nu - st.lambda[j]);
                }
            }
            e->prune64 = blob.add(blk);
            e->prune32 = blob.add(to_f32(blk));
        }
        // fp32 progressive as one SGEMM: every member is its full basis X_r and
        // set 0 the orthonormal DCT-II matrix, so out = x * [D^T | X_1 | ... | X_K]
        if (n <= 256 && n % 16 == 0 && device >= 0) {
            const std::size_t cols = (k + 1) * n;
            std::vector<double> gd(n * cols);
            const long double pi = 3.141592653589793238462643383279502884L;
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) {
                    const long double c = j == 0 ? std::sqrt(1.0L / n) : std::sqrt(2.0L / n);
                    gd[i * cols + j] = static_cast<double>(c * std::cos(pi * j * (2 * i + 1) / (2.0L * n)));
                }
            std::vector<double> xb(n * n);
            for (std::size_t r = 0; r < k; ++r) {
                plan_basis(e->members[r]->st, xb.data());
                for (std::size_t i = 0; i < n; ++i)
                    for (std::size_t sl = 0; sl < n; ++sl) gd[i * cols + (r + 1) * n + sl] = xb[i * n + sl];
            }
            std::vector<float> g(n * cols), bt_hi(cols * n), bt_lo(cols * n);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t c = 0; c < cols; ++c) {
                    const double v = gd[i * cols + c];
                    g[i * cols + c] = static_cast<float>(v);
                    // 3xTF32 operand split of G^T: the TF32 head (round to nearest,
                    // ties away, like cvt.rna.tf32.f32) and the fp32 tail
                    std::uint32_t bits;
                    const float f = static_cast<float>(v);
                    std::memcpy(&bits, &f, 4);
                    bits = (bits + 0x1000u) & 0xffffe000u;
                    float hi;
                    std::memcpy(&hi, &bits, 4);
                    bt_hi[c * n + i] = hi;
                    bt_lo[c * n + i] = static_cast<float>(v - static_cast<double>(hi));
                }
            e->gmat32 = blob.add(g);
            e->gt_hi = blob.add(bt_hi);
            e->gt_lo = blob.add(bt_lo);
            e->gt_sw = blob.add(dctp::dev::tc_swizzle_b(bt_hi.data(), bt_lo.data(), static_cast<int>(cols),
                                                        static_cast<int>(n), static_cast<int>(n)));
            {
                std::vector<double> btd(cols * n);
                for (std::size_t i = 0; i < n; ++i)
                    for (std::size_t c = 0; c < cols; ++c) btd[c * n + i] = gd[i * cols + c];
                e->gt_bf = blob.add(dctp::dev::tc_bf16x3_swizzle_b(btd.data(), static_cast<int>(cols),
                                                                   static_cast<int>(n), static_cast<int>(n)));
            }
            e->dense32 = true;
        }
        if (device < 0) {
            *out = e.release();
            return;
        }
        DeviceScope scope(device);
        e->blob = blob.upload();
        std::vector<dctp::dev::CauchyStage> d64, d32;
        for (std::size_t r = 0; r < k; ++r) {
            d64.push_back(stage_at(e->blob, st[r], false, static_cast<std::int64_t>((r + 1) * n)));
            d32.push_back(stage_at(e->blob, st[r], true, static_cast<std::int64_t>((r + 1) * n)));
        }
        if (k > 0) {
            cuda_check(cudaMemcpy(static_cast<unsigned char*>(e->blob) + e->desc64, d64.data(),
                                  k * sizeof(dctp::dev::CauchyStage), cudaMemcpyHostToDevice),
                       "cudaMemcpy(stages)");
            cuda_check(cudaMemcpy(static_cast<unsigned char*>(e->blob) + e->desc32, d32.data(),
                                  k * sizeof(dctp::dev::CauchyStage), cudaMemcpyHostToDevice),
                       "cudaMemcpy(stages)");
        }
        e->flags.init(e->device);
        cuda_check(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
        *out = e.release();
    });
}

int dctp_ensemble_destroy(dctp_ensemble* e) {
    return guarded([&] { delete e; });
}

int dctp_ensemble_info(const dctp_ensemble* e, size_t* n, size_t* ensemble_size) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("dctp_ensemble_info: null ensemble");
        if (n) *n = e->n;
        if (ensemble_size) *ensemble_size = e->members.size() + 1;
    });
}

int dctp_ensemble_member(const dctp_ensemble* e, size_t r, const dctp_plan** member) {
    return guarded([&] {
        if (!e || !member) throw std::invalid_argument("dctp_ensemble_member: null argument");
        if (r < 1 || r > e->members.size()) throw std::out_of_range("PrunedEnsemblePlan::member: index out of range");
        *member = e->members[r - 1].get();
    });
}

int dctp_ensemble_forward_all_f64(const dctp_ensemble* e, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { ensemble_forward<double>(e, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_ensemble_forward_all_f32(const dctp_ensemble* e, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { ensemble_forward<float>(e, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_ensemble_forward_all_pruned_f64(const dctp_ensemble* e, const double* in, double* out, double* bounds,
                                         unsigned char* pruned, size_t batch, void* stream) {
    return guarded([&] {
        ensemble_forward<double>(e, in, out, batch, static_cast<cudaStream_t>(stream), bounds, pruned);
    });
}
int dctp_ensemble_forward_all_pruned_f32(const dctp_ensemble* e, const float* in, float* out, float* bounds,
                                         unsigned char* pruned, size_t batch, void* stream) {
    return guarded([&] {
        ensemble_forward<float>(e, in, out, batch, static_cast<cudaStream_t>(stream), bounds, pruned);
    });
}
} // extern "C"

/// rdo_select for a batch (fast_transform.hpp:472-496, l1 cost): forward_all
/// into scratch, then the least-l1 set per signal.
template <class T>
static void ensemble_rdo(const dctp_ensemble* e, const T* in, T* chosen, int* index, unsigned char* pruned,
                         std::size_t batch, cudaStream_t s) {
    if (!e) throw std::invalid_argument("rdo_select: null ensemble");
    if (!e->blob) throw std::invalid_argument("PrunedEnsemblePlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!in || (!chosen && !index)) throw std::invalid_argument("rdo_select: null buffer");
    DeviceScope scope(e->device);
    const std::size_t n = e->n, sets = e->members.size() + 1;
    Scratch<T> all(batch * sets * n, s);
    ensemble_forward<T>(e, in, all.ptr, batch, s, nullptr, pruned);
    cuda_check(DCTP_LAUNCH("rdo_select", s,
                           dctp::dev::rdo_select_rows<T>(all.ptr, n, static_cast<int>(sets), batch, chosen, index, s)),
               "rdo_select kernel");
}

/// Host buffers, with bounds and pruned flags: H2D, forward_all, D2H on one
/// stream (meant for small batches; large ones use the pipelined entries).
template <class T>
static void ensemble_pruned_host(const dctp_ensemble* e, const T* h_in, T* h_out, T* h_bounds,
                                 unsigned char* h_pruned, std::size_t batch) {
    if (!e) throw std::invalid_argument("null ensemble");
    if (!e->blob) throw std::invalid_argument("PrunedEnsemblePlan: host-only plan (created with device < 0)");
    if (batch == 0) return;
    if (!h_in || !h_out) throw std::invalid_argument("pruned_forward_all: null buffer");
    DeviceScope scope(e->device);
    const std::size_t n = e->n, sets = e->members.size() + 1;
    HostPipe& hp = host_pipe(e->device);
    cudaStream_t s = hp.comp;
    Scratch<T> din(batch * n, s), dout(batch * sets * n, s), db(batch * sets, s);
    Scratch<unsigned char> dp(batch, s);
    cuda_check(cudaMemcpyAsync(din.ptr, h_in, batch * n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    ensemble_forward<T>(e, din.ptr, dout.ptr, batch, s, db.ptr, dp.ptr);
    cuda_check(cudaMemcpyAsync(h_out, dout.ptr, batch * sets * n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    if (h_bounds)
        cuda_check(cudaMemcpyAsync(h_bounds, db.ptr, batch * sets * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    if (h_pruned) cuda_check(cudaMemcpyAsync(h_pruned, dp.ptr, batch, cudaMemcpyDeviceToHost, s), "D2H");
    sync_check(e->device, e->flags, s);
}

extern "C" {

int dctp_ensemble_rdo_select_f64(const dctp_ensemble* e, const double* in, double* chosen, int* index,
                                 unsigned char* pruned, size_t batch, void* stream) {
    return guarded([&] { ensemble_rdo<double>(e, in, chosen, index, pruned, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_ensemble_rdo_select_f32(const dctp_ensemble* e, const float* in, float* chosen, int* index,
                                 unsigned char* pruned, size_t batch, void* stream) {
    return guarded([&] { ensemble_rdo<float>(e, in, chosen, index, pruned, batch, static_cast<cudaStream_t>(stream)); });
}

int dctp_ensemble_forward_all_pruned_host_f64(const dctp_ensemble* e, const double* h_in, double* h_out,
                                              double* h_bounds, unsigned char* h_pruned, size_t batch) {
    return guarded([&] { ensemble_pruned_host<double>(e, h_in, h_out, h_bounds, h_pruned, batch); });
}
int dctp_ensemble_forward_all_pruned_host_f32(const dctp_ensemble* e, const float* h_in, float* h_out,
                                              float* h_bounds, unsigned char* h_pruned, size_t batch) {
    return guarded([&] { ensemble_pruned_host<float>(e, h_in, h_out, h_bounds, h_pruned, batch); });
}

int dctp_ensemble_sync_check(const dctp_ensemble* e, void* stream) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("dctp_ensemble_sync_check: null ensemble");
        sync_check(e->device, e->flags, static_cast<cudaStream_t>(stream));
    });
}

int dctp_ensemble_forward_all_host_f32(const dctp_ensemble* e, const float* h_in, float* h_out, size_t batch) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("null ensemble");
        if (!e->blob) throw std::invalid_argument("PrunedEnsemblePlan: host-only plan (created with device < 0)");
        if (batch == 0) return;
        const std::size_t sets = e->members.size() + 1;
        if (host_tiny<float>(e->device, e->flags, batch, e->n, sets * e->n, h_in, h_out,
                             [&](const float* din, float* dout, std::size_t rows, cudaStream_t s) {
                                 ensemble_forward<float>(e, din, dout, rows, s);
                             }))
            return;
        host_roundtrip<float>(e->device, batch, e->n, sets * e->n, h_in, h_out,
                              [&](const float* din, float* dout, std::size_t rows, cudaStream_t s) {
                                  ensemble_forward<float>(e, din, dout, rows, s);
                              });
        sync_check(e->device, e->flags, host_pipe(e->device).comp);
    });
}
int dctp_ensemble_forward_all_host_f64(const dctp_ensemble* e, const double* h_in, double* h_out, size_t batch) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("null ensemble");
        if (!e->blob) throw std::invalid_argument("PrunedEnsemblePlan: host-only plan (created with device < 0)");
        if (batch == 0) return;
        const std::size_t sets = e->members.size() + 1;
        if (host_tiny<double>(e->device, e->flags, batch, e->n, sets * e->n, h_in, h_out,
                             [&](const double* din, double* dout, std::size_t rows, cudaStream_t s) {
                                 ensemble_forward<double>(e, din, dout, rows, s);
                             }))
            return;
        host_roundtrip<double>(e->device, batch, e->n, sets * e->n, h_in, h_out,
                               [&](const double* din, double* dout, std::size_t rows, cudaStream_t s) {
                                   ensemble_forward<double>(e, din, dout, rows, s);
                               });
        sync_check(e->device, e->flags, host_pipe(e->device).comp);
    });
}

// --- bare trig kernels ------------------------------------------------------------

} // extern "C"

// --- rank-k chains -------------------------------------------------------------

struct dctp_chain {
    dctp::host::Chain ch;
    int device = 0;
    void* blob = nullptr; // X^T in fp64 (ld even), X in fp32 for the SGEMM route
    StreamFlags flags;
    std::size_t ldt = 0, xt64 = 0, x32 = 0;
    bool sgemm32 = false;
    // int8 slices of X^T for the tcgen05 kind::i8 product (ozaki.cu), built on first use
    std::mutex oz_mu;
    int8_t* oz = nullptr;
    int* oz_e = nullptr;
    int oz_slices = 0;

    ~dctp_chain() {
        if (blob) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            cudaFree(blob);
            if (oz) cudaFree(oz);
            if (oz_e) cudaFree(oz_e);
            cudaSetDevice(prev);
        }
    }
};

/// chain_forward (cauchy.hpp:218-231) for a batch: out = in X, one product
/// with the composed basis (fp64 on DMMA; fp32 as an SGEMM when the shape
/// allows, else widened through the DMMA kernel).
template <class T>
static void chain_forward(const dctp_chain* c, const T* in, T* out, std::size_t batch, cudaStream_t s) {
    if (!c) throw std::invalid_argument("chain_forward: null chain");
    if (!c->blob) throw std::invalid_argument("ChainedFactorization: host-only chain (created with device < 0)");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("chain_forward: null buffer");
    DeviceScope scope(c->device);
    const std::size_t n = c->ch.n;
    const int ni = static_cast<int>(n);
    if constexpr (std::is_same_v<T, float>) {
        const float* x = at<float>(c->blob, c->x32);
        if (c->sgemm32 && dctp::dev::sgemm_rows_supported(ni, ni, ni, ni, n, in, x, out)) {
            cuda_check(DCTP_LAUNCH("chain_sgemm", s,
                                   dctp::dev::sgemm_rows(in, ni, x, ni, out, n, batch, ni, ni, c->flags(s), s)),
                       "chain sgemm kernel");
            return;
        }
    }
    if constexpr (std::is_same_v<T, double>) {
        if (const int S = ozaki_slices(n)) {
            {
                auto* cm = const_cast<dctp_chain*>(c);
                std::lock_guard<std::mutex> lock(cm->oz_mu);
                if (!cm->oz || cm->oz_slices != S) {
                    if (cm->oz) cudaFree(cm->oz);
                    if (cm->oz_e) cudaFree(cm->oz_e);
                    cm->oz = nullptr;
                    cm->oz_e = nullptr;
                    auto [sl, ex] = slice_operand(at<double>(c->blob, c->xt64), c->ldt, n, ni, S, s);
                    cm->oz = sl;
                    cm->oz_e = ex;
                    cm->oz_slices = S;
                }
            }
            rows_by_ozaki(in, n, c->oz, c->oz_e, ni, ni, S, out, n, batch, c->flags(s), s, "chain_i8");
            return;
        }
    }
    cuda_check(DCTP_LAUNCH("chain_dmma", s,
                           dctp::dev::rows_by_basis<T>(in, n, at<double>(c->blob, c->xt64), c->ldt, ni, ni, out, n,
                                                       batch, c->flags(s), s)),
               "chain dmma kernel");
}

extern "C" {

int dctp_chain_create(size_t n, size_t k, const int* kinds, const size_t* is, const size_t* js, const double* rhos,
                      const double* vs, const double* base_lambda, const double* base_u, double tau, int device,
                      dctp_chain** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("dctp_chain_create: null output");
        *out = nullptr;
        if (k > 0 && (!kinds || !is || !js || !rhos)) throw std::invalid_argument("dctp_chain_create: null update arrays");
        if (!base_lambda != !base_u) throw std::invalid_argument("dctp_chain_create: give both base arrays or neither");
        if (n > (std::size_t{1} << 14)) throw std::invalid_argument("dctp_chain_create: n above 16384");
        std::vector<dctp::host::Update> ups;
        for (std::size_t r = 0; r < k; ++r) {
            try {
                ups.push_back(make_update(kinds[r], is[r], js[r], rhos[r], vs ? vs + r * n : nullptr, n));
            } catch (const std::exception& ex) {
                throw std::runtime_error("compose_rank_k: stage " + std::to_string(r + 1) + ": " + ex.what());
            }
        }
        auto c = std::make_unique<dctp_chain>();
        c->device = device;
        c->ch = dctp::host::compose_rank_k(
            n, ups, base_lambda ? std::vector<double>(base_lambda, base_lambda + n) : std::vector<double>{},
            base_u ? std::vector<double>(base_u, base_u + n * n) : std::vector<double>{}, tau);
        if (device >= 0) {
            c->ldt = (n + 3) / 4 * 4;
            std::vector<double> xt(n * c->ldt, 0.0);
            std::vector<float> x32(n * n);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) {
                    xt[j * c->ldt + i] = c->ch.x[i * n + j];
                    x32[i * n + j] = static_cast<float>(c->ch.x[i * n + j]);
                }
            c->sgemm32 = n % 16 == 0 && n <= 4096;
            Blob blob;
            c->xt64 = blob.add(xt);
            if (c->sgemm32) c->x32 = blob.add(x32);
            DeviceScope scope(device);
            prepare_pool(device);
            c->blob = blob.upload();
            c->flags.init(c->device);
        }
        *out = c.release();
    });
}

int dctp_chain_destroy(dctp_chain* c) {
    return guarded([&] { delete c; });
}

int dctp_chain_info(const dctp_chain* c, size_t* n, size_t* stages) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("dctp_chain_info: null chain");
        if (n) *n = c->ch.n;
        if (stages) *stages = c->ch.stages.size();
    });
}

int dctp_chain_spectrum(const dctp_chain* c, double* mu, double* x) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("dctp_chain_spectrum: null chain");
        if (mu) std::copy(c->ch.mu.begin(), c->ch.mu.end(), mu);
        if (x) std::copy(c->ch.x.begin(), c->ch.x.end(), x);
    });
}

int dctp_chain_stage(const dctp_chain* c, size_t r, double* base_vals, double* mu, double* sigma, int* passthrough,
                     int64_t* idx, size_t* n_rotations) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("dctp_chain_stage: null chain");
        if (r >= c->ch.stages.size()) throw std::out_of_range("dctp_chain_stage: stage index out of range");
        const auto& st = c->ch.stages[r];
        if (base_vals) std::copy(st.base_vals.begin(), st.base_vals.end(), base_vals);
        if (mu) std::copy(st.spec.mu.begin(), st.spec.mu.end(), mu);
        if (sigma) std::copy(st.sigma.begin(), st.sigma.end(), sigma);
        for (std::size_t q = 0; q < st.spec.slots.size(); ++q) {
            if (passthrough) passthrough[q] = st.spec.slots[q].passthrough ? 1 : 0;
            if (idx) idx[q] = static_cast<int64_t>(st.spec.slots[q].idx);
        }
        if (n_rotations) *n_rotations = st.spec.rotations.size();
    });
}

int dctp_chain_forward_f64(const dctp_chain* c, const double* in, double* out, size_t batch, void* stream) {
    return guarded([&] { chain_forward<double>(c, in, out, batch, static_cast<cudaStream_t>(stream)); });
}
int dctp_chain_forward_f32(const dctp_chain* c, const float* in, float* out, size_t batch, void* stream) {
    return guarded([&] { chain_forward<float>(c, in, out, batch, static_cast<cudaStream_t>(stream)); });
}

int dctp_chain_sync_check(const dctp_chain* c, void* stream) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("dctp_chain_sync_check: null chain");
        if (!c->blob) throw std::invalid_argument("ChainedFactorization: host-only chain (created with device < 0)");
        sync_check(c->device, c->flags, static_cast<cudaStream_t>(stream));
    });
}

#define DCTP_CHAIN_HOST_ENTRY(NAME, T)                                                                  \
    int NAME(const dctp_chain* c, const T* h_in, T* h_out, size_t batch) {                             \
        return guarded([&] {                                                                           \
            if (!c) throw std::invalid_argument(#NAME ": null chain");                                 \
            if (!c->blob) throw std::invalid_argument("ChainedFactorization: host-only chain (created with device < 0)"); \
            if (batch == 0) return;                                                                    \
            const std::size_t n = c->ch.n;                                                             \
            auto fn = [&](const T* din, T* dout, std::size_t rows, cudaStream_t s) { chain_forward<T>(c, din, dout, rows, s); }; \
            if (host_tiny<T>(c->device, c->flags, batch, n, n, h_in, h_out, fn)) return;               \
            host_roundtrip<T>(c->device, batch, n, n, h_in, h_out,                                     \
                              [&](const T* din, T* dout, std::size_t rows, cudaStream_t s) {          \
                                  chain_forward<T>(c, din, dout, rows, s);                             \
                              });                                                                      \
            sync_check(c->device, c->flags, host_pipe(c->device).comp);                                                   \
        });                                                                                            \
    }
DCTP_CHAIN_HOST_ENTRY(dctp_chain_forward_host_f64, double)
DCTP_CHAIN_HOST_ENTRY(dctp_chain_forward_host_f32, float)
#undef DCTP_CHAIN_HOST_ENTRY

} // extern "C"

namespace {
struct TrigCache {
    std::mutex mu;
    struct Entry {
        int device;
        std::size_t n;
        void* blob;
        TwiddleOffsets t64, t32;
        int* flag;
    };
    std::vector<Entry> entries;
    Entry get(int device, std::size_t n) {
        std::lock_guard<std::mutex> lock(mu);
        for (auto& e : entries)
            if (e.device == device && e.n == n) return e;
        Blob blob;
        Entry e{device, n, nullptr, add_twiddles<double>(blob, n), add_twiddles<float>(blob, n), nullptr};
        e.blob = blob.upload();
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&e.flag), sizeof(int)), "cudaMalloc(flag)");
        cuda_check(cudaMemset(e.flag, 0, sizeof(int)), "cudaMemset(flag)");
        entries.push_back(e);
        return e;
    }
};
TrigCache& trig_cache() {
    static TrigCache* c = new TrigCache; // never destroyed: outlives the CUDA context teardown
    return *c;
}

template <class T>
void trig_run(bool inverse, std::size_t n, const T* in, T* out, std::size_t batch, int device, cudaStream_t s) {
    if (n < 1) throw std::invalid_argument("TrigPlan: length must be positive");
    if (batch == 0) return;
    if (!in || !out) throw std::invalid_argument("trig: null buffer");
    if (!dctp::dev::dct_supported(n, std::is_same_v<T, double>))
        throw std::invalid_argument("TrigPlan: length " + std::to_string(n) + " exceeds the GPU DCT kernels");
    DeviceScope scope(device);
    const auto e = trig_cache().get(device, n);
    dctp::dev::Twiddles<T> tw;
    if constexpr (std::is_same_v<T, double>)
        tw = twiddles_at<double>(e.blob, e.t64);
    else
        tw = twiddles_at<float>(e.blob, e.t32);
    const dctp::dev::Emit<T> none{};
    if (!inverse)
        cuda_check(dctp::dev::dct2_rows<T>(in, n, out, n, out, n, none, n, batch, tw, e.flag, s), "dct2 kernel");
    else
        cuda_check(dctp::dev::idct_rows<T>(in, n, in, n, none, out, n, n, batch, tw, e.flag, s), "idct kernel");
}
} // namespace

extern "C" {

int dctp_dct2_f64(size_t n, const double* in, double* out, size_t batch, int device, void* stream) {
    return guarded([&] { trig_run<double>(false, n, in, out, batch, device, static_cast<cudaStream_t>(stream)); });
}
int dctp_idct2_f64(size_t n, const double* in, double* out, size_t batch, int device, void* stream) {
    return guarded([&] { trig_run<double>(true, n, in, out, batch, device, static_cast<cudaStream_t>(stream)); });
}
int dctp_dct2_f32(size_t n, const float* in, float* out, size_t batch, int device, void* stream) {
    return guarded([&] { trig_run<float>(false, n, in, out, batch, device, static_cast<cudaStream_t>(stream)); });
}
int dctp_idct2_f32(size_t n, const float* in, float* out, size_t batch, int device, void* stream) {
    return guarded([&] { trig_run<float>(true, n, in, out, batch, device, static_cast<cudaStream_t>(stream)); });
}

int dctp_trig_host_f64(int inverse, size_t n, const double* h_in, double* h_out, size_t batch, int device) {
    return guarded([&] {
        if (batch == 0) return;
        if (!h_in || !h_out) throw std::invalid_argument("dctp_trig_host_f64: null buffer");
        DeviceScope scope(device);
        cudaStream_t s = host_pipe(device).comp;
        Scratch<double> d(2 * batch * n, s);
        cuda_check(cudaMemcpyAsync(d.ptr, h_in, batch * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
        trig_run<double>(inverse != 0, n, d.ptr, d.ptr + batch * n, batch, device, s);
        cuda_check(cudaMemcpyAsync(h_out, d.ptr + batch * n, batch * n * sizeof(double), cudaMemcpyDeviceToHost, s),
                   "D2H");
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(trig)");
    });
}

int dctp_profile_enable(int on) {
    return guarded([&] { Profiler::get().enable(on != 0); });
}

int dctp_profile_reset(void) {
    return guarded([&] { Profiler::get().reset(); });
}

int dctp_profile_summary(char* buf, size_t len) {
    return guarded([&] {
        const std::string s = Profiler::get().summary();
        if (!buf || len <= s.size()) throw std::invalid_argument("dctp_profile_summary: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

uint64_t dctp_mix_seed(uint64_t seed, size_t size, size_t kind) { return dctp::host::mix_seed(seed, size, kind); }

int dctp_fill_signals(uint64_t seed, int dist, double r, size_t n, size_t rows, double* out) {
    return guarded([&] {
        if (!out && n * rows > 0) throw std::invalid_argument("dctp_fill_signals: null output");
        if (dist < 0 || dist > 4) throw std::invalid_argument("dctp_fill_signals: unknown distribution");
        dctp::host::fill_signals(seed, static_cast<dctp::host::Dist>(dist), r, n, rows, out);
    });
}

} // extern "C"
