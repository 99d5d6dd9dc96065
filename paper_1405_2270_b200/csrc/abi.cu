// abi.cu -- lifecycle, diagnostics and the synchronous host-level entry points
// (ls_h_*) of liblatsum_cuda.so. The host-level calls are what the drop-in
// C++ headers (include/latsum/*.hpp) and the end-to-end bench path use: host
// buffers in, host buffers out, every device buffer owned and released here
// (stream-ordered pool allocations, so repeated calls do not hit cudaMalloc).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ls {

std::string& last_error() {
    thread_local std::string msg;
    return msg;
}

std::atomic<int64_t>& launch_counter() {
    static std::atomic<int64_t> n{0};
    return n;
}

int sm_count() {
    static std::mutex mu;
    static std::vector<int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
    if (cache[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

unsigned* fault_flag() {
    static std::mutex mu;
    static std::vector<unsigned*> flags;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= static_cast<int>(flags.size())) flags.resize(dev + 1, nullptr);
    if (flags[dev] == nullptr) {
        unsigned* f = nullptr;
        if (cudaMalloc(&f, sizeof(unsigned)) != cudaSuccess) return nullptr;
        if (cudaMemset(f, 0, sizeof(unsigned)) != cudaSuccess) return nullptr;
        flags[dev] = f;
    }
    return flags[dev];
}

bool take_fault() {
    unsigned* f = fault_flag();
    if (f == nullptr) return false;
    unsigned v = 0;
    if (cudaMemcpy(&v, f, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    if (v != 0) cudaMemset(f, 0, sizeof(unsigned));
    return v != 0;
}

void ensure_pool() {
    static std::mutex mu;
    static std::vector<char> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= static_cast<int>(done.size())) done.resize(dev + 1, 0);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev] = 1;
}

namespace {

// Per-thread compute + copy streams on the current device, and a pool that
// keeps freed blocks cached between calls.
struct Streams {
    int device = -1;
    cudaStream_t compute = nullptr;
    cudaStream_t copy = nullptr;
};

int get_streams(Streams*& out) {
    thread_local Streams s;
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev));
    if (s.device != dev) {
        LS_CUDA(cudaStreamCreateWithFlags(&s.compute, cudaStreamNonBlocking));
        LS_CUDA(cudaStreamCreateWithFlags(&s.copy, cudaStreamNonBlocking));
        ensure_pool();
        s.device = dev;
    }
    out = &s;
    return LS_OK;
}

// Stream-ordered device buffer.
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    int alloc(size_t bytes, cudaStream_t stream) {
        s = stream;
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, stream);
        if (e != cudaSuccess) {
            p = nullptr;
            return cuda_fail(e, "cudaMallocAsync");
        }
        return LS_OK;
    }
    double* d() const { return static_cast<double*>(p); }
    int64_t* i() const { return static_cast<int64_t*>(p); }
};

#define LS_TRY(expr)                 \
    do {                             \
        int _rc = (expr);            \
        if (_rc != LS_OK) return _rc; \
    } while (0)

int upload(DevBuf& b, const void* host, size_t bytes, cudaStream_t s) {
    LS_TRY(b.alloc(bytes, s));
    if (bytes) LS_CUDA(cudaMemcpyAsync(b.p, host, bytes, cudaMemcpyHostToDevice, s));
    return LS_OK;
}


// Host threads the pageable copy-out uses (ls_set_host_threads); 0 = min(8, hardware).
std::atomic<int>& host_threads() {
    static std::atomic<int> n{0};
    return n;
}

// Pinned staging for pageable destinations: a bounded ring of page-locked pieces per thread
// and device (kRingSlots x kPieceBytes = 256 MiB), so a caller's ordinary (numpy, std::vector)
// buffer receives the grid at near link speed without pinning gigabytes of host memory.
constexpr int kRingSlots = 8;
constexpr int64_t kPieceBytes = 32ll << 20;

struct PinnedRing {
    int device = -1;
    void* slot[kRingSlots] = {};
    cudaEvent_t ready[kRingSlots] = {};
    ~PinnedRing() {
        for (int r = 0; r < kRingSlots; ++r) {
            if (slot[r]) cudaFreeHost(slot[r]);
            if (ready[r]) cudaEventDestroy(ready[r]);
        }
    }
};

int get_ring(PinnedRing*& out) {
    thread_local PinnedRing ring;
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev));
    if (ring.device != dev) {
        for (int r = 0; r < kRingSlots; ++r) {
            if (ring.slot[r]) cudaFreeHost(ring.slot[r]);
            ring.slot[r] = nullptr;
            LS_CUDA(cudaMallocHost(&ring.slot[r], static_cast<size_t>(kPieceBytes)));
            if (!ring.ready[r]) LS_CUDA(cudaEventCreateWithFlags(&ring.ready[r], cudaEventDisableTiming));
        }
        ring.device = dev;
    }
    out = &ring;
    return LS_OK;
}

// Copy-out workers: each job waits for its piece's D2H event, then memcpy's the pinned piece
// into the caller's buffer. Jobs run in submission order per worker (round robin), and a
// slot is reused only after its previous job has finished (done[r]).
class CopyOut {
public:
    explicit CopyOut(int n) : queues_(static_cast<size_t>(n)) {
        for (int t = 0; t < n; ++t) workers_.emplace_back([this, t] { run(t); });
    }
    ~CopyOut() { finish(); }
    void submit(int slot, cudaEvent_t ev, void* dst, const void* src, size_t bytes) {
        {
            std::lock_guard<std::mutex> lock(mu_);
            busy_[slot] = true;
            queues_[static_cast<size_t>(next_)].push_back({slot, ev, dst, src, bytes});
            next_ = (next_ + 1) % static_cast<int>(workers_.size());
        }
        cv_.notify_all();
    }
    // Blocks until the last job that used `slot` has finished copying out of it.
    void wait_slot(int slot) {
        std::unique_lock<std::mutex> lock(mu_);
        done_cv_.wait(lock, [&] { return !busy_[slot]; });
    }
    void finish() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            if (stop_) return;
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    bool failed() const { return failed_.load(); }

private:
    struct Job {
        int slot;
        cudaEvent_t ev;
        void* dst;
        const void* src;
        size_t bytes;
    };
    void run(int t) {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return stop_ || !queues_[static_cast<size_t>(t)].empty(); });
                if (queues_[static_cast<size_t>(t)].empty()) return;  // stop_ and drained
                j = queues_[static_cast<size_t>(t)].front();
                queues_[static_cast<size_t>(t)].erase(queues_[static_cast<size_t>(t)].begin());
            }
            if (cudaEventSynchronize(j.ev) != cudaSuccess) failed_ = true;
            else std::memcpy(j.dst, j.src, j.bytes);
            {
                std::lock_guard<std::mutex> lock(mu_);
                busy_[j.slot] = false;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::vector<Job>> queues_;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    bool busy_[kRingSlots] = {};
    bool stop_ = false;
    int next_ = 0;
    std::atomic<bool> failed_{false};
};

// Expands slabs [k0, k1) of a device-resident tensor into host memory. The compute stream
// fills ~1 GiB chunk buffers (two alternate, so the expansion of chunk c+1 overlaps the copy of
// chunk c); the copy stream drains them. A page-locked destination (cudaMallocHost /
// cudaHostRegister, e.g. a pinned torch tensor) receives the D2H copies directly; a pageable
// one goes through the bounded pinned ring above, piece by piece, with host threads moving
// each piece into place while the link carries the next.
int expand_to_host(const double* A, const double* B, const double* C, const double* w,
                   const int64_t d[3], int R, int64_t k0, int64_t k1, double* out_h, Streams& st) {
    const int64_t slab = d[0] * d[1];
    if (k1 <= k0 || slab == 0) return LS_OK;
    const int64_t slab_bytes = slab * static_cast<int64_t>(sizeof(double));
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, out_h) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // an unregistered pointer is not an error here
    PinnedRing* ring = nullptr;
    if (!pinned) LS_TRY(get_ring(ring));
    // ~1 GiB chunks: enough work units per launch to fill the GPU; two buffers in flight.
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(k1 - k0, (1ll << 30) / slab_bytes));
    DevBuf buf[2];
    cudaEvent_t done_compute[2], done_copy[2];
    for (int b = 0; b < 2; ++b) {
        LS_TRY(buf[b].alloc(static_cast<size_t>(chunk * slab_bytes), st.compute));
        LS_CUDA(cudaEventCreateWithFlags(&done_compute[b], cudaEventDisableTiming));
        LS_CUDA(cudaEventCreateWithFlags(&done_copy[b], cudaEventDisableTiming));
    }
    int nt = host_threads().load();
    if (nt <= 0) nt = static_cast<int>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())));
    std::unique_ptr<CopyOut> copier;
    if (!pinned) copier.reset(new CopyOut(std::min(nt, kRingSlots)));
    int rc = LS_OK;
    int64_t c = 0, piece = 0;
    for (int64_t ks = k0; ks < k1 && rc == LS_OK; ks += chunk, ++c) {
        const int b = static_cast<int>(c & 1);
        const int64_t ke = std::min(k1, ks + chunk);
        if (c >= 2) cudaStreamWaitEvent(st.compute, done_copy[b], 0);
        rc = ls_expand(A, d[0], B, d[1], C, d[2], w, d[0], d[1], d[2], R, ks, ke, buf[b].d(), 0, 0,
                       nullptr, nullptr, nullptr, nullptr, st.compute);
        if (rc != LS_OK) break;
        cudaEventRecord(done_compute[b], st.compute);
        cudaStreamWaitEvent(st.copy, done_compute[b], 0);
        const int64_t bytes = (ke - ks) * slab_bytes;
        char* dst = reinterpret_cast<char*>(out_h + (ks - k0) * slab);
        const char* src = static_cast<const char*>(buf[b].p);
        if (pinned) {
            cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost, st.copy);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync D2H");
        } else {
            for (int64_t off = 0; off < bytes && rc == LS_OK; off += kPieceBytes, ++piece) {
                const int r = static_cast<int>(piece % kRingSlots);
                const size_t n = static_cast<size_t>(std::min(kPieceBytes, bytes - off));
                copier->wait_slot(r);  // the slot's previous piece has left it
                cudaError_t e = cudaMemcpyAsync(ring->slot[r], src + off, n, cudaMemcpyDeviceToHost, st.copy);
                if (e != cudaSuccess) {
                    rc = cuda_fail(e, "cudaMemcpyAsync D2H (pinned ring)");
                    break;
                }
                cudaEventRecord(ring->ready[r], st.copy);
                copier->submit(r, ring->ready[r], dst + off, ring->slot[r], n);
            }
        }
        cudaEventRecord(done_copy[b], st.copy);
    }
    if (copier) {
        copier->finish();
        if (copier->failed() && rc == LS_OK) rc = fail(LS_ECUDA, "expand_to_host: D2H piece failed");
    }
    cudaError_t e1 = cudaStreamSynchronize(st.copy);
    cudaError_t e2 = cudaStreamSynchronize(st.compute);
    for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(done_compute[b]);
        cudaEventDestroy(done_copy[b]);
    }
    if (rc != LS_OK) return rc;
    if (e1 != cudaSuccess) return cuda_fail(e1, "copy stream");
    if (e2 != cudaSuccess) return cuda_fail(e2, "compute stream");
    if (take_fault()) return fail(LS_ECUDA, "kernel watchdog: an mbarrier wait timed out (results discarded)");
    return LS_OK;
}

}  // namespace
}  // namespace ls

using ls::DevBuf;
using ls::Streams;

extern "C" {

int ls_abi_version(void) { return 1; }

const char* ls_last_error(void) { return ls::last_error().c_str(); }

// grid.hpp:21-27 (GridSpec::validate) and lattice.hpp:33-68 (LatticeSpec::validate,
// charge_grid_index): the one host implementation of these checks, with the reference's
// messages, called by the drop-in headers, the host-level calls, the pipeline and the
// Python mirror.
int ls_charge_grid_index(double b, int64_t n, double p, int axis, int nu, int64_t* out) {
    const double h = b / static_cast<double>(n);
    const double x = (p + b / 2.0) / h;
    const double rounded = std::round(x);
    if (std::abs(x - rounded) > 1e-9 * static_cast<double>(n) || rounded < 0.0 ||
        rounded > static_cast<double>(n))
        return ls::fail(LS_EVALIDATION, "lattice: charge " + std::to_string(nu) + " coordinate " + std::to_string(p) +
                                            " on axis " + std::to_string(axis) +
                                            " does not lie on a grid point of the unit cell");
    if (out) *out = static_cast<int64_t>(rounded);
    return LS_OK;
}

int ls_validate_grid(double b, int64_t n) {
    if (!(b > 0.0) || !std::isfinite(b))
        return ls::fail(LS_EVALIDATION, "grid: box edge must be positive, got " + std::to_string(b));
    if (n < 2 || n % 2 != 0)
        return ls::fail(LS_EVALIDATION, "grid: n must be even and at least 2, got " + std::to_string(n));
    return LS_OK;
}

int ls_validate_lattice(const int64_t L[3], int64_t n, double b, const double* charges_h, int M0, int64_t* ia_out) {
    if (const int rc = ls_validate_grid(b, n)) return rc;
    for (int l = 0; l < 3; ++l)
        if (L[l] < 1) return ls::fail(LS_EVALIDATION, "lattice: cell count on axis " + std::to_string(l) + " must be >= 1");
    if (M0 < 1) return ls::fail(LS_EVALIDATION, "lattice: at least one charge required");
    for (int nu = 0; nu < M0; ++nu) {
        const double Z = charges_h[4 * nu + 3];
        if (!(Z > 0.0) || !std::isfinite(Z))
            return ls::fail(LS_EVALIDATION, "lattice: charge " + std::to_string(nu) + " must have positive finite Z");
        for (int l = 0; l < 3; ++l) {
            int64_t i = 0;
            if (const int rc = ls_charge_grid_index(b, n, charges_h[4 * nu + l], l, nu, &i)) return rc;
            if (ia_out) ia_out[static_cast<size_t>(l) * M0 + nu] = i;
        }
    }
    return LS_OK;
}

int ls_fault_status(int reset) {
    unsigned* f = ls::fault_flag();
    if (f == nullptr) return ls::fail(LS_ECUDA, "fault_status: no CUDA device");
    unsigned v = 0;
    LS_CUDA(cudaMemcpy(&v, f, sizeof(v), cudaMemcpyDeviceToHost));
    if (v != 0 && reset) LS_CUDA(cudaMemset(f, 0, sizeof(unsigned)));
    return v != 0 ? 1 : 0;
}

int ls_set_host_threads(int n) {
    if (n < 0) return ls::fail(LS_EVALIDATION, "set_host_threads: negative count");
    ls::host_threads() = n;
    return LS_OK;
}

int ls_dev_knobs_enabled(void) {
#ifdef LS_DEV_KNOBS
    return 1;
#else
    return 0;
#endif
}

int ls_set_device(int device) {
    LS_CUDA(cudaSetDevice(device));
    return LS_OK;
}

int64_t ls_launch_count(void) { return ls::launch_counter().load(); }

// quadrature.hpp:50-89 (host arithmetic; the rule is 2M+1 scalars shared by
// every stage): window [s1, s2] from the two tail bisections
// (quadrature.hpp:35-46, :62-66), then tau_j = 2 G(s_j) / a_max and
// w_j = step (4/sqrt(pi)) cosh(s_j) / (1 + e^{-min(sinh s_j, 700)}) / a_max,
// G(s) = log(1 + e^{sinh s}) (sinh s itself above 30).
}  // extern "C"
namespace {
template <class F>
double bisect_tail(F f, double target, double hi) {
    double lo = 1e-3;
    while (f(hi) > target) hi *= 1.5;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        (f(mid) <= target ? hi : lo) = mid;
    }
    return hi;
}
}  // namespace
extern "C" {

int ls_sinc_quadrature(double eps, double a_min, double a_max, int M, double C0, double* nodes,
                       double* exponents, double* weights, double* step_out) {
    if (M < 1) return ls::fail(LS_EVALIDATION, "quadrature: M must be >= 1, got " + std::to_string(M));
    if (!(eps > 0.0) || !(eps < 1.0)) return ls::fail(LS_EVALIDATION, "quadrature: eps must lie in (0, 1)");
    if (!(a_min > 0.0) || !(a_min < a_max))
        return ls::fail(LS_EVALIDATION, "quadrature: need 0 < a_min < a_max");
    const double tol = eps * std::pow(10.0, -C0);
    const double ratio = a_min / a_max;
    const double t_lo = bisect_tail([](double t) { return 2.0 * t * std::exp(-t); }, tol, 5.0);
    const double t_hi = bisect_tail([](double t) { return std::sqrt(t) * std::exp(-t); }, tol * ratio, 5.0);
    const double s_begin = -std::log(2.0 * t_lo);
    const double s_end = 0.5 * std::log(t_hi / (ratio * ratio));
    const int count = 2 * M + 1;
    const double step = (s_end - s_begin) / static_cast<double>(count - 1);
    const double c = 4.0 / std::sqrt(M_PI);
    for (int j = 0; j < count; ++j) {
        const double s = s_begin + step * static_cast<double>(j);
        const double sh = std::sinh(s);
        const double G = sh > 30.0 ? sh : std::log1p(std::exp(sh));
        if (nodes) nodes[j] = s;
        exponents[j] = 2.0 * G / a_max;
        weights[j] = step * c * std::cosh(s) / (1.0 + std::exp(-std::min(sh, 700.0))) / a_max;
    }
    if (step_out) *step_out = step;
    return LS_OK;
}

// calibrate_quadrature (newton.hpp:161-189) with every candidate's probes evaluated on the GPU
// by the fused probe_error kernel: the probe set (newton.hpp:97-132) is built once on the host
// and uploaded once; per candidate only tau/w go up and one double comes back.
int ls_h_calibrate_quadrature(double b, int64_t n, double eps, double a_min, double a_max, int m_cap, int* M_out,
                              double* C0_out, int* trace_len, int* trace_M, double* trace_C0, double* trace_err,
                              int trace_cap) {
    if (!(b > 0.0) || !std::isfinite(b) || n < 2 || n % 2 != 0)
        return ls::fail(LS_EVALIDATION, "grid: need b > 0 and even n >= 2");
    if (!(eps > 0.0 && eps < 1.0)) return ls::fail(LS_EVALIDATION, "tolerance: eps must lie in (0, 1)");
    if (!(a_min > 0.0 && a_min < a_max)) return ls::fail(LS_EVALIDATION, "tolerance: need 0 < a_min < a_max");
    const double h = b / static_cast<double>(n);
    // probe set: shell around the centre, three rays, strided lattice; sorted unique, in band
    std::vector<int64_t> keys;
    auto add = [&](int64_t i, int64_t j, int64_t k) {
        if (i >= 0 && i < n && j >= 0 && j < n && k >= 0 && k < n) keys.push_back((i * n + j) * n + k);
    };
    const int64_t c = n / 2, sh = std::min<int64_t>(8, n / 2);
    for (int64_t i = c - sh; i < c + sh; ++i)
        for (int64_t j = c - sh; j < c + sh; ++j)
            for (int64_t k = c - sh; k < c + sh; ++k) add(i, j, k);
    for (int64_t i = 0; i < n; ++i) {
        add(i, c, c);
        add(i, i, c);
        add(i, i, i);
    }
    const int64_t stride = std::max<int64_t>(1, n / 16);
    for (int64_t i = 0; i < n; i += stride)
        for (int64_t j = 0; j < n; j += stride)
            for (int64_t k = 0; k < n; k += stride) add(i, j, k);
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::vector<int64_t> idx;
    std::vector<double> rad;
    for (int64_t key : keys) {
        const int64_t i = key / (n * n), j = (key / n) % n, k = key % n;
        auto mid = [&](int64_t a) { return (static_cast<double>(a) + 0.5 - static_cast<double>(n) / 2.0) * h; };
        const double x = mid(i), y = mid(j), z = mid(k);
        const double r = std::sqrt(x * x + y * y + z * z);
        if (r >= a_min && r <= a_max) {
            idx.insert(idx.end(), {i, j, k});
            rad.push_back(r);
        }
    }
    if (rad.empty()) return ls::fail(LS_EVALIDATION, "calibrate_quadrature: no grid midpoints in [a_min, a_max]");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const cudaStream_t s = st->compute;
    const int64_t P = static_cast<int64_t>(rad.size());
    const int maxR = 2 * m_cap + 1;
    DevBuf didx, drad, dtau, dw, derr;
    LS_TRY(ls::upload(didx, idx.data(), sizeof(int64_t) * idx.size(), s));
    LS_TRY(ls::upload(drad, rad.data(), sizeof(double) * rad.size(), s));
    LS_TRY(dtau.alloc(sizeof(double) * maxR, s));
    LS_TRY(dw.alloc(sizeof(double) * maxR, s));
    LS_TRY(derr.alloc(sizeof(double) * 4, s));
    std::vector<double> tau(maxR), w(maxR), nodes(maxR);
    const double depths[4] = {1.0, 2.0, 3.0, 4.0};
    int n_trace = 0;
    double best_seen = INFINITY;
    for (int M = 2; M <= m_cap; ++M) {
        const int R = 2 * M + 1;
        double errs[4];
        for (int d = 0; d < 4; ++d) {
            double step = 0.0;
            LS_TRY(ls_sinc_quadrature(eps, a_min, a_max, M, depths[d], nodes.data(), tau.data(), w.data(), &step));
            LS_CUDA(cudaMemcpyAsync(dtau.p, tau.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s));
            LS_CUDA(cudaMemcpyAsync(dw.p, w.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s));
            LS_TRY(ls_probe_error(dtau.d(), dw.d(), R, n, h, didx.i(), drad.d(), P, derr.d() + d, s));
        }
        LS_CUDA(cudaMemcpyAsync(errs, derr.p, sizeof(errs), cudaMemcpyDeviceToHost, s));
        LS_SYNC(s);
        int pick = 0;
        for (int d = 0; d < 4; ++d) {
            if (trace_len && n_trace < trace_cap) {
                trace_M[n_trace] = M;
                trace_C0[n_trace] = depths[d];
                trace_err[n_trace] = errs[d];
            }
            ++n_trace;
            if (errs[d] < errs[pick]) pick = d;
        }
        best_seen = std::min(best_seen, errs[pick]);
        if (errs[pick] <= eps) {
            *M_out = M;
            *C0_out = depths[pick];
            if (trace_len) *trace_len = n_trace;
            return LS_OK;
        }
    }
    if (trace_len) *trace_len = n_trace;
    return ls::fail(LS_EGUARD, "calibrate_quadrature: no rule with M <= " + std::to_string(m_cap) +
                                   " meets eps = " + std::to_string(eps) + "; best achieved error " +
                                   std::to_string(best_seen));
}

int ls_h_gen_column(int mode, double t, int64_t len, double h, double* out_h) {
    if (!(t >= 0.0) || !std::isfinite(t))
        return ls::fail(LS_EVALIDATION, "generator: t must be finite and >= 0");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf tau, out;
    LS_TRY(ls::upload(tau, &t, sizeof(double), st->compute));
    LS_TRY(out.alloc(sizeof(double) * static_cast<size_t>(std::max<int64_t>(len, 1)), st->compute));
    LS_TRY(ls_gen_master(mode, tau.d(), 1, len, h, out.d(), len, st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double) * len, cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

int ls_h_newton_master(int mode, const int64_t lens[3], double h, const double* tau_h, int R, double* f0_h,
                       double* f1_h, double* f2_h) {
    if (!(h > 0.0) || !std::isfinite(h)) return ls::fail(LS_EVALIDATION, "generator: mesh h must be positive");
    for (int l = 0; l < 3; ++l)
        if (lens[l] < 2 || lens[l] % 2 != 0)
            return ls::fail(LS_EVALIDATION, "generator: axis lengths must be even and >= 2");
    for (int q = 0; q < R; ++q)
        if (!(tau_h[q] >= 0.0) || !std::isfinite(tau_h[q]))
            return ls::fail(LS_EVALIDATION, "generator: exponents must be finite and >= 0");
    if (R == 0) return LS_OK;
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf tau;
    LS_TRY(ls::upload(tau, tau_h, sizeof(double) * R, st->compute));
    double* outs[3] = {f0_h, f1_h, f2_h};
    for (int l = 0; l < 3; ++l) {
        // Axes of equal length share one factor (newton.hpp:60-69).
        int same = -1;
        for (int m = 0; m < l; ++m)
            if (lens[m] == lens[l]) same = m;
        if (same >= 0) {
            LS_SYNC(st->compute);
            std::memcpy(outs[l], outs[same], sizeof(double) * static_cast<size_t>(lens[l] * R));
            continue;
        }
        DevBuf f;
        LS_TRY(f.alloc(sizeof(double) * static_cast<size_t>(lens[l] * R), st->compute));
        LS_TRY(ls_gen_master(mode, tau.d(), R, lens[l], h, f.d(), lens[l], st->compute));
        LS_CUDA(cudaMemcpyAsync(outs[l], f.p, sizeof(double) * lens[l] * R, cudaMemcpyDeviceToHost, st->compute));
        LS_SYNC(st->compute);
    }
    return LS_OK;
}

int ls_h_functional_batch(const int64_t dims[3], int R, const double* A_h, const double* B_h, const double* C_h,
                          const double* w_h, int F, const double* X_h, const double* Y_h, const double* Z_h,
                          double scale, double* out_h) {
    if (F == 0) return LS_OK;
    if (R == 0) {
        for (int f = 0; f < F; ++f) out_h[f] = 0.0;
        return LS_OK;
    }
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf A, B, C, w, X, Y, Z, out;
    LS_TRY(ls::upload(A, A_h, sizeof(double) * dims[0] * R, st->compute));
    LS_TRY(ls::upload(B, B_h, sizeof(double) * dims[1] * R, st->compute));
    LS_TRY(ls::upload(C, C_h, sizeof(double) * dims[2] * R, st->compute));
    LS_TRY(ls::upload(w, w_h, sizeof(double) * R, st->compute));
    LS_TRY(ls::upload(X, X_h, sizeof(double) * dims[0] * F, st->compute));
    LS_TRY(ls::upload(Y, Y_h, sizeof(double) * dims[1] * F, st->compute));
    LS_TRY(ls::upload(Z, Z_h, sizeof(double) * dims[2] * F, st->compute));
    LS_TRY(out.alloc(sizeof(double) * F, st->compute));
    LS_TRY(ls_functional_batch(A.d(), dims[0], B.d(), dims[1], C.d(), dims[2], w.d(), R, dims[0], dims[1], dims[2],
                               X.d(), dims[0], Y.d(), dims[1], Z.d(), dims[2], F, scale, out.d(), st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double) * F, cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

int ls_h_max_norm_diff(const int64_t dims[3], int Ra, const double* A0_h, const double* A1_h, const double* A2_h,
                       const double* wa_h, int Rb, const double* B0_h, const double* B1_h, const double* B2_h,
                       const double* wb_h, double* max_diff_h, double* max_abs_b_h) {
    *max_diff_h = 0.0;
    *max_abs_b_h = 0.0;
    const int64_t slab = dims[0] * dims[1];
    if (slab == 0 || dims[2] == 0) return LS_OK;
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const cudaStream_t s = st->compute;
    const double* ah[3] = {A0_h, A1_h, A2_h};
    const double* bh[3] = {B0_h, B1_h, B2_h};
    DevBuf fa[3], fb[3], wa, wb, ga, gb, part;
    for (int l = 0; l < 3; ++l) {
        LS_TRY(ls::upload(fa[l], ah[l], sizeof(double) * dims[l] * Ra, s));
        LS_TRY(ls::upload(fb[l], bh[l], sizeof(double) * dims[l] * Rb, s));
    }
    LS_TRY(ls::upload(wa, wa_h, sizeof(double) * Ra, s));
    LS_TRY(ls::upload(wb, wb_h, sizeof(double) * Rb, s));
    // Both tensors expanded chunk by chunk on the device; the grids never leave HBM
    // (max_norm_diff_canonical, canonical.hpp:282-301).
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(dims[2], (256ll << 20) / (slab * 8)));
    LS_TRY(ga.alloc(sizeof(double) * chunk * slab, s));
    LS_TRY(gb.alloc(sizeof(double) * chunk * slab, s));
    const int nblocks = 4 * ls::sm_count();
    LS_TRY(part.alloc(sizeof(double) * 2 * nblocks, s));
    LS_CUDA(cudaMemsetAsync(part.p, 0, sizeof(double) * 2 * nblocks, s));
    for (int64_t k0 = 0; k0 < dims[2]; k0 += chunk) {
        const int64_t k1 = std::min(dims[2], k0 + chunk);
        LS_TRY(ls_expand(fa[0].d(), dims[0], fa[1].d(), dims[1], fa[2].d(), dims[2], wa.d(), dims[0], dims[1],
                         dims[2], Ra, k0, k1, ga.d(), 0, 0, nullptr, nullptr, nullptr, nullptr, s));
        LS_TRY(ls_expand(fb[0].d(), dims[0], fb[1].d(), dims[1], fb[2].d(), dims[2], wb.d(), dims[0], dims[1],
                         dims[2], Rb, k0, k1, gb.d(), 0, 0, nullptr, nullptr, nullptr, nullptr, s));
        LS_TRY(ls_maxdiff_accumulate(ga.d(), gb.d(), (k1 - k0) * slab, part.d(), nblocks, s));
    }
    std::vector<double> hp(2 * static_cast<size_t>(nblocks));
    LS_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s));
    LS_SYNC(s);
    for (int b = 0; b < nblocks; ++b) {
        *max_diff_h = std::max(*max_diff_h, hp[2 * b]);
        *max_abs_b_h = std::max(*max_abs_b_h, hp[2 * b + 1]);
    }
    return LS_OK;
}

int ls_h_lattice_master(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h,
                        int R, double* f0_h, double* f1_h, double* f2_h) {
    if (n < 2 || n % 2 != 0 || !(b > 0.0) || !std::isfinite(b))
        return ls::fail(LS_EVALIDATION, "grid: need b > 0 and even n >= 2");
    for (int l = 0; l < 3; ++l)
        if (L[l] < 1) return ls::fail(LS_EVALIDATION, "lattice: cell counts must be >= 1");
    for (int q = 0; q < R; ++q)
        if (!(tau_h[q] >= 0.0) || !std::isfinite(tau_h[q]))
            return ls::fail(LS_EVALIDATION, "generator: exponents must be finite and >= 0");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const double h = b / static_cast<double>(n);
    DevBuf tau;
    LS_TRY(ls::upload(tau, tau_h, sizeof(double) * R, st->compute));
    double* outs[3] = {f0_h, f1_h, f2_h};
    for (int l = 0; l < 3; ++l) {
        const int64_t len = 2 * L[l] * n;
        // Axes of equal length share one factor (newton.hpp:60-69).
        int same = -1;
        for (int m = 0; m < l; ++m)
            if (L[m] == L[l]) same = m;
        if (same >= 0) {
            LS_SYNC(st->compute);
            std::memcpy(outs[l], outs[same], sizeof(double) * static_cast<size_t>(len * R));
            continue;
        }
        DevBuf f;
        LS_TRY(f.alloc(sizeof(double) * static_cast<size_t>(len * R), st->compute));
        LS_TRY(ls_gen_master(mode, tau.d(), R, len, h, f.d(), len, st->compute));
        LS_CUDA(cudaMemcpyAsync(outs[l], f.p, sizeof(double) * len * R, cudaMemcpyDeviceToHost, st->compute));
        LS_SYNC(st->compute);
    }
    return LS_OK;
}

int ls_h_assemble_axis(const double* master_h, int64_t master_len, int R, int M0,
                       const int64_t* ia_h, int64_t n, int64_t L, int periodic, double* out_h) {
    if (master_len != 2 * L * n)
        return ls::fail(LS_EVALIDATION, "lattice: master axis length does not match the doubled target grid");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const int64_t out_len = periodic ? n : L * n;
    DevBuf m, ia, out;
    LS_TRY(ls::upload(m, master_h, sizeof(double) * master_len * R, st->compute));
    LS_TRY(ls::upload(ia, ia_h, sizeof(int64_t) * M0, st->compute));
    LS_TRY(out.alloc(sizeof(double) * out_len * M0 * R, st->compute));
    LS_TRY(ls_assemble_axis(m.d(), master_len, R, M0, ia.i(), n, L, periodic, out.d(), out_len, st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double) * out_len * M0 * R, cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

int ls_h_expand(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                const double* C_h, const double* w_h, int64_t k0, int64_t k1, double* out_h) {
    if (k0 < 0 || k1 > dims[2] || k0 > k1) return ls::fail(LS_EVALIDATION, "expand: slab range outside [0, N3]");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf A, B, C, w;
    LS_TRY(ls::upload(A, A_h, sizeof(double) * dims[0] * R, st->compute));
    LS_TRY(ls::upload(B, B_h, sizeof(double) * dims[1] * R, st->compute));
    LS_TRY(ls::upload(C, C_h, sizeof(double) * dims[2] * R, st->compute));
    LS_TRY(ls::upload(w, w_h, sizeof(double) * R, st->compute));
    return ls::expand_to_host(A.d(), B.d(), C.d(), w.d(), dims, R, k0, k1, out_h, *st);
}

int ls_h_eval_points(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                     const double* C_h, const double* w_h, const int64_t* idx_h, int64_t P,
                     double* out_h) {
    for (int64_t p = 0; p < P; ++p)
        for (int l = 0; l < 3; ++l)
            if (idx_h[3 * p + l] < 0 || idx_h[3 * p + l] >= dims[l])
                return ls::fail(LS_EVALIDATION, "eval_point: index out of range");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf A, B, C, w, idx, out;
    LS_TRY(ls::upload(A, A_h, sizeof(double) * dims[0] * R, st->compute));
    LS_TRY(ls::upload(B, B_h, sizeof(double) * dims[1] * R, st->compute));
    LS_TRY(ls::upload(C, C_h, sizeof(double) * dims[2] * R, st->compute));
    LS_TRY(ls::upload(w, w_h, sizeof(double) * R, st->compute));
    LS_TRY(ls::upload(idx, idx_h, sizeof(int64_t) * 3 * P, st->compute));
    LS_TRY(out.alloc(sizeof(double) * P, st->compute));
    LS_TRY(ls_eval_points(A.d(), dims[0], B.d(), dims[1], C.d(), dims[2], w.d(), R, idx.i(), P, out.d(), st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double) * P, cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

int ls_h_scalar_product(const int64_t dims[3], int Ra, const double* A0_h, const double* A1_h,
                        const double* A2_h, const double* wa_h, int Rb, const double* B0_h,
                        const double* B1_h, const double* B2_h, const double* wb_h, double* out_h) {
    if (Ra == 0 || Rb == 0) {
        *out_h = 0.0;  // canonical.hpp:128
        return LS_OK;
    }
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const double* ah[3] = {A0_h, A1_h, A2_h};
    const double* bh[3] = {B0_h, B1_h, B2_h};
    DevBuf a[3], bb[3], G[3], wa, wb, out;
    for (int l = 0; l < 3; ++l) {
        LS_TRY(ls::upload(a[l], ah[l], sizeof(double) * dims[l] * Ra, st->compute));
        LS_TRY(ls::upload(bb[l], bh[l], sizeof(double) * dims[l] * Rb, st->compute));
        LS_TRY(G[l].alloc(sizeof(double) * static_cast<size_t>(Ra) * Rb, st->compute));
        LS_TRY(ls_gram(a[l].d(), dims[l], Ra, bb[l].d(), dims[l], Rb, dims[l], G[l].d(), st->compute));
    }
    LS_TRY(ls::upload(wa, wa_h, sizeof(double) * Ra, st->compute));
    LS_TRY(ls::upload(wb, wb_h, sizeof(double) * Rb, st->compute));
    LS_TRY(out.alloc(sizeof(double), st->compute));
    LS_TRY(ls_gram_reduce(G[0].d(), G[1].d(), G[2].d(), wa.d(), Ra, wb.d(), Rb, out.d(), st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

int ls_h_grid_functional(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                         const double* C_h, const double* w_h, const double* r1_h,
                         const double* r2_h, const double* r3_h, int64_t k0, int64_t k1,
                         double* out_h) {
    if (k0 < 0 || k1 > dims[2] || k0 > k1) return ls::fail(LS_EVALIDATION, "functional: slab range outside [0, N3]");
    Streams* st;
    LS_TRY(ls::get_streams(st));
    DevBuf A, B, C, w, r1, r2, r3, part, out;
    LS_TRY(ls::upload(A, A_h, sizeof(double) * dims[0] * R, st->compute));
    LS_TRY(ls::upload(B, B_h, sizeof(double) * dims[1] * R, st->compute));
    LS_TRY(ls::upload(C, C_h, sizeof(double) * dims[2] * R, st->compute));
    LS_TRY(ls::upload(w, w_h, sizeof(double) * R, st->compute));
    LS_TRY(ls::upload(r1, r1_h, sizeof(double) * dims[0], st->compute));
    LS_TRY(ls::upload(r2, r2_h, sizeof(double) * dims[1], st->compute));
    LS_TRY(ls::upload(r3, r3_h, sizeof(double) * dims[2], st->compute));
    const int64_t np = ls_expand_partial_count(dims[0], dims[1], std::max(R, 4), k0, k1);
    if (np < 0) return ls::fail(LS_EGUARD, "functional: rank too large");
    LS_TRY(part.alloc(sizeof(double) * std::max<int64_t>(np, 1), st->compute));
    LS_TRY(out.alloc(sizeof(double), st->compute));
    LS_CUDA(cudaMemsetAsync(part.p, 0, sizeof(double) * std::max<int64_t>(np, 1), st->compute));
    LS_TRY(ls_expand(A.d(), dims[0], B.d(), dims[1], C.d(), dims[2], w.d(), dims[0], dims[1], dims[2], R,
                     k0, k1, nullptr, 0, 0, r1.d(), r2.d(), r3.d(), part.d(), st->compute));
    LS_TRY(ls_sum_partials(part.d(), np, out.d(), st->compute));
    LS_CUDA(cudaMemcpyAsync(out_h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st->compute));
    LS_SYNC(st->compute);
    return LS_OK;
}

}  // extern "C"

namespace {
// Generator -> assembled sum on the device, then either the expansion of slabs [k0, k1) into
// host memory (grid_h) or the fused full-grid functional of those slabs against the separable
// density rho_h (energy_h); the host-level entry points below.
int lattice_impl(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h, const double* w_h, int R,
                 const double* charges_h, int M0, int periodic, int64_t k0, int64_t k1, double* grid_h,
                 double* f0_h, double* f1_h, double* f2_h, double* wout_h, const double* const* rho_h,
                 double* energy_h) {
    // LatticeSpec::validate + charge snapping (lattice.hpp:33-68), then weights Z_nu * w_q
    // (lattice.hpp:284-287), on the host.
    std::vector<int64_t> ia(static_cast<size_t>(3 * std::max(M0, 0)));
    LS_TRY(ls_validate_lattice(L, n, b, charges_h, M0, ia.data()));
    if (R < 1) return ls::fail(LS_EVALIDATION, "lattice: master tensor has rank 0");
    std::vector<double> wt(static_cast<size_t>(M0) * R);
    for (int nu = 0; nu < M0; ++nu)
        for (int q = 0; q < R; ++q) wt[static_cast<size_t>(nu) * R + q] = charges_h[4 * nu + 3] * w_h[q];
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const cudaStream_t s = st->compute;
    const double h = b / static_cast<double>(n);
    const int Rt = M0 * R;
    int64_t d[3];
    for (int l = 0; l < 3; ++l) d[l] = periodic ? n : L[l] * n;
    if (k0 < 0 || k1 > d[2] || k0 > k1) return ls::fail(LS_EVALIDATION, "lattice potential: slab range outside the grid");
    DevBuf tau, iad, wd, master[3], fac[3];
    LS_TRY(ls::upload(tau, tau_h, sizeof(double) * R, s));
    LS_TRY(ls::upload(iad, ia.data(), sizeof(int64_t) * ia.size(), s));
    LS_TRY(ls::upload(wd, wt.data(), sizeof(double) * wt.size(), s));
    const double* fptr[3];
    double* fh[3] = {f0_h, f1_h, f2_h};
    ls::GenAsmAxis ax[3];
    int n_ax = 0;
    for (int l = 0; l < 3; ++l) {
        // Axes with equal L and equal charge indices yield bit-identical factors.
        int same = -1;
        for (int m = 0; m < l && same < 0; ++m)
            if (L[m] == L[l] &&
                std::equal(ia.begin() + m * M0, ia.begin() + (m + 1) * M0, ia.begin() + l * M0))
                same = m;
        if (same >= 0) {
            fptr[l] = fptr[same];
            continue;
        }
        const int64_t len = 2 * L[l] * n;
        LS_TRY(master[l].alloc(sizeof(double) * len * R, s));
        LS_TRY(fac[l].alloc(sizeof(double) * d[l] * Rt, s));
        ax[n_ax++] = {L[l], iad.i() + l * M0, master[l].d(), fac[l].d()};
        fptr[l] = fac[l].d();
    }
    // generator + assembled sum (one launch on small lattices)
    LS_TRY(ls::gen_assemble(mode, tau.d(), R, M0, n, h, periodic, ax, n_ax, s));
    for (int l = 0; l < 3; ++l)
        if (fh[l]) LS_CUDA(cudaMemcpyAsync(fh[l], fptr[l], sizeof(double) * d[l] * Rt, cudaMemcpyDeviceToHost, s));
    if (wout_h) std::memcpy(wout_h, wt.data(), sizeof(double) * wt.size());
    if (energy_h) {
        // <V, rho> over slabs [k0, k1) fused into the expansion (V never stored), fixed-order sum.
        DevBuf rho[3], part, out;
        for (int l = 0; l < 3; ++l) LS_TRY(ls::upload(rho[l], rho_h[l], sizeof(double) * d[l], s));
        const int64_t np = ls_expand_partial_count(d[0], d[1], Rt, k0, k1);
        if (np < 0) return ls::fail(LS_EGUARD, "lattice energy: no tile plan for this rank");
        LS_TRY(part.alloc(sizeof(double) * std::max<int64_t>(np, 1), s));
        LS_TRY(out.alloc(sizeof(double), s));
        LS_CUDA(cudaMemsetAsync(part.p, 0, sizeof(double) * std::max<int64_t>(np, 1), s));
        LS_TRY(ls_expand(fptr[0], d[0], fptr[1], d[1], fptr[2], d[2], wd.d(), d[0], d[1], d[2], Rt, k0, k1, nullptr,
                         0, 0, rho[0].d(), rho[1].d(), rho[2].d(), part.d(), s));
        LS_TRY(ls_sum_partials(part.d(), np, out.d(), s));
        LS_CUDA(cudaMemcpyAsync(energy_h, out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        LS_SYNC(s);
    } else if (grid_h) {
        LS_TRY(ls::expand_to_host(fptr[0], fptr[1], fptr[2], wd.d(), d, Rt, k0, k1, grid_h, *st));
    } else {
        LS_SYNC(s);
    }
    return LS_OK;
}
}  // namespace

extern "C" {

int ls_h_lattice_potential(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h,
                           const double* w_h, int R, const double* charges_h, int M0, int periodic,
                           int64_t k0, int64_t k1, double* grid_h, double* f0_h, double* f1_h,
                           double* f2_h, double* wout_h) {
    return lattice_impl(mode, L, n, b, tau_h, w_h, R, charges_h, M0, periodic, k0, k1, grid_h, f0_h, f1_h, f2_h,
                        wout_h, nullptr, nullptr);
}

// Host-level QTT (qtt.hpp): the columns of V_h (N x ncols, column-major) in, cores / ranks out.
int ls_h_qtt_compress(const double* V_h, int64_t N, int ncols, double eps, int rmax, double* cores_h,
                      int64_t core_stride, int* ranks_h, int* capped_h) {
    if (ncols < 0) return ls::fail(LS_EVALIDATION, "qtt_compress: negative column count");
    if (N < 2 || (N & (N - 1)) != 0)
        return ls::fail(LS_EVALIDATION, "qtt_compress: length " + std::to_string(N) + " is not a power of two >= 2");
    if (!(eps > 0.0)) return ls::fail(LS_EVALIDATION, "qtt_compress: eps must be positive");
    int L = 0;
    while ((int64_t(1) << L) < N && L < 62) ++L;
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const cudaStream_t s = st->compute;
    DevBuf v, cores, ranks, capped;
    LS_TRY(ls::upload(v, V_h, sizeof(double) * static_cast<size_t>(std::max<int64_t>(N, 0)) * ncols, s));
    LS_TRY(cores.alloc(sizeof(double) * std::max<int64_t>(core_stride, 1) * std::max(ncols, 1), s));
    LS_TRY(ranks.alloc(sizeof(int) * (L + 1) * std::max(ncols, 1), s));
    LS_TRY(capped.alloc(sizeof(int) * std::max(ncols, 1), s));
    LS_TRY(ls_qtt_compress(v.d(), N, N, ncols, eps, rmax, cores.d(), core_stride, static_cast<int*>(ranks.p),
                           static_cast<int*>(capped.p), s));
    if (ncols > 0) {
        LS_CUDA(cudaMemcpyAsync(cores_h, cores.p, sizeof(double) * core_stride * ncols, cudaMemcpyDeviceToHost, s));
        LS_CUDA(cudaMemcpyAsync(ranks_h, ranks.p, sizeof(int) * (L + 1) * ncols, cudaMemcpyDeviceToHost, s));
        LS_CUDA(cudaMemcpyAsync(capped_h, capped.p, sizeof(int) * ncols, cudaMemcpyDeviceToHost, s));
    }
    LS_SYNC(s);
    return LS_OK;
}

int ls_h_qtt_unfolding_ranks(const double* V_h, int64_t N, int ncols, double eps, int* ranks_h) {
    if (ncols < 0) return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: negative column count");
    if (N < 2 || (N & (N - 1)) != 0)
        return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: length is not a power of two >= 2");
    if (!(eps > 0.0)) return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: eps must be positive");
    int L = 0;
    while ((int64_t(1) << L) < N && L < 62) ++L;
    Streams* st;
    LS_TRY(ls::get_streams(st));
    const cudaStream_t s = st->compute;
    DevBuf v, ranks;
    LS_TRY(ls::upload(v, V_h, sizeof(double) * static_cast<size_t>(std::max<int64_t>(N, 0)) * ncols, s));
    LS_TRY(ranks.alloc(sizeof(int) * std::max(L - 1, 1) * std::max(ncols, 1), s));
    LS_TRY(ls_qtt_unfolding_ranks(v.d(), N, N, ncols, eps, static_cast<int*>(ranks.p), s));
    if (ncols > 0 && L > 1)
        LS_CUDA(cudaMemcpyAsync(ranks_h, ranks.p, sizeof(int) * (L - 1) * ncols, cudaMemcpyDeviceToHost, s));
    LS_SYNC(s);
    return LS_OK;
}

int ls_h_lattice_energy(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h, const double* w_h,
                        int R, const double* charges_h, int M0, int periodic, int64_t k0, int64_t k1,
                        const double* r1_h, const double* r2_h, const double* r3_h, double* energy_h) {
    if (!r1_h || !r2_h || !r3_h || !energy_h) return ls::fail(LS_EVALIDATION, "lattice energy: null density or output");
    const double* rho[3] = {r1_h, r2_h, r3_h};
    return lattice_impl(mode, L, n, b, tau_h, w_h, R, charges_h, M0, periodic, k0, k1, nullptr, nullptr, nullptr,
                        nullptr, nullptr, rho, energy_h);
}

}  // extern "C"
