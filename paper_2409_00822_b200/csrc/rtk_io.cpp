// rtk_io.cpp -- RTKM matrix file -> row top-k on the GPU -> RTKR result file.
//
// A streaming file-level job (include/rtk.h: rtk_topk_file_f32) replacing
// the reference chain load_matrix -> batch_topk -> save_result
// (/root/reference/pkg/src/rowtopk/io.py:46-78, batch.py:105-142).  Rows move
// in chunks through two pinned host buffers and two device buffers:
//   host thread:  pread chunk i | pwrite results of chunk i-1
//   s_h2d:        H2D chunk i
//   s_comp:       rtk_rowtopk_*_f32 on chunk i (the same C-ABI launch as the
//                 in-memory path, so the outputs are bit-identical)
//   s_d2h:        D2H values / indices of chunk i
// so disk (page cache) reads, PCIe in both directions, the kernel and the
// result writes overlap.  Values and indices go to their two regions of the
// RTKR file by offset (pwrite), in the reference byte layout.
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rtk.h"

int rtk_fail(int code, const char* fmt, ...);

namespace {

constexpr char kMatrixMagic[4] = {'R', 'T', 'K', 'M'};
constexpr char kResultMagic[4] = {'R', 'T', 'K', 'R'};
constexpr uint32_t kVersion = 1;
constexpr int64_t kHeader = 24;  // magic, u32 version, u64 n_rows, u64 n_cols

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

// A temporary output file removed on scope exit unless its path was cleared.
struct TmpFile {
    std::string path;
    ~TmpFile() {
        if (!path.empty()) unlink(path.c_str());
    }
};

bool read_full(int fd, void* buf, size_t n, int64_t off) {
    char* p = static_cast<char*>(buf);
    while (n > 0) {
        ssize_t r = pread(fd, p, n, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        p += r;
        n -= (size_t)r;
        off += r;
    }
    return true;
}

bool write_full(int fd, const void* buf, size_t n, int64_t off) {
    const char* p = static_cast<const char*>(buf);
    while (n > 0) {
        ssize_t r = pwrite(fd, p, n, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        p += r;
        n -= (size_t)r;
        off += r;
    }
    return true;
}

// pread / pwrite of one contiguous range split across `threads` host threads
// (a single thread copies the page cache at a few GB/s; the range sizes here
// are tens of MB).
template <class F>
bool parallel_io(F op, int fd, char* buf, size_t n, int64_t off, int threads) {
    const size_t min_piece = 4u << 20;
    int t = (int)std::min<size_t>((size_t)threads, std::max<size_t>(1, n / min_piece));
    if (t <= 1) return op(fd, buf, n, off);
    std::atomic<bool> ok{true};
    std::vector<std::thread> pool;
    const size_t piece = (n + t - 1) / t;
    for (int i = 0; i < t; ++i) {
        const size_t a = (size_t)i * piece, b = std::min(n, a + piece);
        if (a >= b) break;
        pool.emplace_back([&, a, b] {
            if (!op(fd, buf + a, b - a, off + (int64_t)a)) ok = false;
        });
    }
    for (auto& th : pool) th.join();
    return ok;
}

// Pinned host and device buffers of the file job, kept per device between
// jobs (cudaHostAlloc of the ~200 MB working set costs ~100 ms, more than the
// streaming itself).  One job at a time uses a device's pool; a concurrent
// job on the same device allocates private buffers.
struct Buffers {
    size_t in_bytes = 0, out_bytes = 0, nan_words = 0;
    float* pin_in[2] = {nullptr, nullptr};
    float* pin_val[2] = {nullptr, nullptr};
    int32_t* pin_idx[2] = {nullptr, nullptr};
    float* d_in[2] = {nullptr, nullptr};
    float* d_val[2] = {nullptr, nullptr};
    int32_t* d_idx[2] = {nullptr, nullptr};
    uint32_t* d_nan = nullptr;

    void release() {
        for (int i = 0; i < 2; ++i) {
            cudaFreeHost(pin_in[i]);
            cudaFreeHost(pin_val[i]);
            cudaFreeHost(pin_idx[i]);
            cudaFree(d_in[i]);
            cudaFree(d_val[i]);
            cudaFree(d_idx[i]);
            pin_in[i] = pin_val[i] = nullptr;
            pin_idx[i] = nullptr;
            d_in[i] = d_val[i] = nullptr;
            d_idx[i] = nullptr;
        }
        cudaFree(d_nan);
        d_nan = nullptr;
        in_bytes = out_bytes = nan_words = 0;
    }
    // Grow to at least the requested sizes (contents are not preserved).
    cudaError_t reserve(size_t in_b, size_t out_b, size_t words) {
        cudaError_t e = cudaSuccess;
        if (in_b > in_bytes) {
            for (int i = 0; i < 2; ++i) {
                cudaFreeHost(pin_in[i]);
                cudaFree(d_in[i]);
                pin_in[i] = nullptr;
                d_in[i] = nullptr;
            }
            for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
                e = cudaHostAlloc(reinterpret_cast<void**>(&pin_in[i]), in_b, cudaHostAllocDefault);
                if (e == cudaSuccess) e = cudaMalloc(&d_in[i], in_b);
            }
            in_bytes = e == cudaSuccess ? in_b : 0;
        }
        if (e == cudaSuccess && out_b > out_bytes) {
            for (int i = 0; i < 2; ++i) {
                cudaFreeHost(pin_val[i]);
                cudaFreeHost(pin_idx[i]);
                cudaFree(d_val[i]);
                cudaFree(d_idx[i]);
                pin_val[i] = nullptr;
                pin_idx[i] = nullptr;
                d_val[i] = nullptr;
                d_idx[i] = nullptr;
            }
            for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
                e = cudaHostAlloc(reinterpret_cast<void**>(&pin_val[i]), out_b, cudaHostAllocDefault);
                if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&pin_idx[i]), out_b, cudaHostAllocDefault);
                if (e == cudaSuccess) e = cudaMalloc(&d_val[i], out_b);
                if (e == cudaSuccess) e = cudaMalloc(&d_idx[i], out_b);
            }
            out_bytes = e == cudaSuccess ? out_b : 0;
        }
        if (e == cudaSuccess && words > nan_words) {
            cudaFree(d_nan);
            d_nan = nullptr;
            e = cudaMalloc(&d_nan, words * 4);
            nan_words = e == cudaSuccess ? words : 0;
        }
        if (e != cudaSuccess) release();
        return e;
    }
};

constexpr int kMaxDevices = 64;
std::mutex g_pool_mu[kMaxDevices];
Buffers g_pool[kMaxDevices];

// One job's CUDA resources: pooled (or private) buffers, streams, events.
struct Job {
    Buffers priv;
    Buffers* b = &priv;
    std::unique_lock<std::mutex> pool_lock;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t h2d[2] = {}, kern[2] = {}, d2h[2] = {};
    explicit Job(int dev) {
        if (dev >= 0 && dev < kMaxDevices) {
            std::unique_lock<std::mutex> lk(g_pool_mu[dev], std::try_to_lock);
            if (lk.owns_lock()) {
                pool_lock = std::move(lk);
                b = &g_pool[dev];
            }
        }
    }
    ~Job() {
        for (auto st : s)
            if (st) cudaStreamSynchronize(st);
        priv.release();
        for (int i = 0; i < 2; ++i) {
            if (h2d[i]) cudaEventDestroy(h2d[i]);
            if (kern[i]) cudaEventDestroy(kern[i]);
            if (d2h[i]) cudaEventDestroy(d2h[i]);
        }
        for (auto st : s)
            if (st) cudaStreamDestroy(st);
    }
};

#define CU(call)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) return rtk_fail(RTK_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

namespace {
// RTK_IO_TRACE=1: phase timestamps on stderr (diagnostics for the file job).
struct Trace {
    bool on = std::getenv("RTK_IO_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void operator()(const char* what) const {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[rtk_io] %9.3f ms  %s\n", ms, what);
    }
};
}  // namespace

extern "C" int rtk_topk_file_f32(const char* matrix_path, const char* result_path, int32_t k, int32_t mode,
                                 double eps_rel, int32_t hard_cap, int32_t max_iter, int64_t chunk_rows,
                                 int64_t* dims) {
    if (!matrix_path || !result_path) return rtk_fail(RTK_EINVAL, "NULL path");
    if (mode != 0 && mode != 1) return rtk_fail(RTK_EINVAL, "mode must be 0 (exact) or 1 (early stop), got %d", mode);
    Fd in;
    in.fd = open(matrix_path, O_RDONLY | O_CLOEXEC);
    if (in.fd < 0) return rtk_fail(RTK_EIO, "%s: %s", matrix_path, strerror(errno));
    // header (io.py:32-43): magic, version, non-empty payload
    unsigned char hdr[kHeader];
    struct stat st;
    if (fstat(in.fd, &st) != 0) return rtk_fail(RTK_EIO, "%s: %s", matrix_path, strerror(errno));
    if (st.st_size < kHeader || !read_full(in.fd, hdr, kHeader, 0))
        return rtk_fail(RTK_ETRUNC, "unexpected end of file while reading header");
    if (std::memcmp(hdr, kMatrixMagic, 4) != 0)
        return rtk_fail(RTK_EFORMAT, "%s: expected magic b'RTKM', found b'%.4s'", matrix_path, (const char*)hdr);
    uint32_t version;
    uint64_t n64, m64;
    std::memcpy(&version, hdr + 4, 4);
    std::memcpy(&n64, hdr + 8, 8);
    std::memcpy(&m64, hdr + 16, 8);
    if (version != kVersion) return rtk_fail(RTK_EFORMAT, "%s: unsupported format version %u", matrix_path, version);
    if (n64 < 1 || m64 < 1)
        return rtk_fail(RTK_ETRUNC, "%s: header declares empty payload %llux%llu", matrix_path,
                        (unsigned long long)n64, (unsigned long long)m64);
    if (m64 >= (1ull << 30) || n64 >= 0xffffffffull || n64 * m64 > (1ull << 60))
        return rtk_fail(RTK_EINVAL, "%s: matrix %llux%llu is too large", matrix_path, (unsigned long long)n64,
                        (unsigned long long)m64);
    const int64_t n = (int64_t)n64, m = (int64_t)m64;
    if (dims) {
        dims[0] = n;
        dims[1] = m;
        dims[2] = -1;
    }
    if ((uint64_t)st.st_size < (uint64_t)kHeader + n64 * m64 * 4)
        return rtk_fail(RTK_ETRUNC, "unexpected end of file while reading matrix payload");
    const bool k_ok = k >= 1 && k <= m;  // checked after the NaN scan (batch.py:107-111)
    const int64_t kk = k_ok ? k : 1;

    if (chunk_rows <= 0) chunk_rows = (64ll << 20) / (4 * m);
    if (chunk_rows < 1) chunk_rows = 1;
    if (chunk_rows > n) chunk_rows = n;
    const int64_t n_chunks = (n + chunk_rows - 1) / chunk_rows;

    Trace trace;
    trace("header checked");
    int dev = 0;
    CU(cudaGetDevice(&dev));
    Job j(dev);
    for (int i = 0; i < 3; ++i) CU(cudaStreamCreateWithFlags(&j.s[i], cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CU(cudaEventCreateWithFlags(&j.h2d[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&j.kern[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&j.d2h[i], cudaEventDisableTiming));
    }
    CU(j.b->reserve((size_t)chunk_rows * m * 4, k_ok ? (size_t)chunk_rows * kk * 4 : 0, (size_t)n_chunks));
    Buffers& B = *j.b;
    trace("buffers allocated");

    // The result goes to a temporary file next to result_path, renamed over it
    // only once every row is written and the NaN check has passed: a failing
    // job leaves an existing result_path untouched and no partial file, as
    // the reference (load_matrix -> batch_topk raise before save_result).
    Fd out;
    TmpFile tmp;
    if (k_ok) {
        tmp.path = std::string(result_path) + ".rtk-tmp." + std::to_string((long long)getpid());
        out.fd = open(tmp.path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
        if (out.fd < 0) {
            tmp.path.clear();
            return rtk_fail(RTK_EIO, "%s: %s", result_path, strerror(errno));
        }
        unsigned char rh[kHeader];
        const uint64_t kk64 = (uint64_t)kk;
        std::memcpy(rh, kResultMagic, 4);
        std::memcpy(rh + 4, &kVersion, 4);
        std::memcpy(rh + 8, &n64, 8);
        std::memcpy(rh + 16, &kk64, 8);
        if (!write_full(out.fd, rh, kHeader, 0)) return rtk_fail(RTK_EIO, "%s: %s", result_path, strerror(errno));
    }
    const int64_t val_off = kHeader, idx_off = kHeader + n * kk * 4;
    const int io_threads = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
    auto write_back = [&](int64_t c) -> int {
        const int sl = (int)(c % 2);
        const int64_t a = c * chunk_rows, rows = (a + chunk_rows <= n ? chunk_rows : n - a);
        cudaError_t e = cudaEventSynchronize(j.d2h[sl]);
        if (e != cudaSuccess) return rtk_fail(RTK_ECUDA, "D2H: %s", cudaGetErrorString(e));
        if (!parallel_io(write_full, out.fd, reinterpret_cast<char*>(B.pin_val[sl]), (size_t)rows * kk * 4,
                         val_off + a * kk * 4, io_threads) ||
            !parallel_io(write_full, out.fd, reinterpret_cast<char*>(B.pin_idx[sl]), (size_t)rows * kk * 4,
                         idx_off + a * kk * 4, io_threads))
            return rtk_fail(RTK_EIO, "%s: %s", result_path, strerror(errno));
        return RTK_OK;
    };

    // The result writes of chunk c-1 run on a writer thread while the host
    // thread reads chunk c+1; the writer is joined before its pinned output
    // buffers are reused (the D2H of chunk c+1).
    std::thread writer;
    std::atomic<int> wrc{RTK_OK};
    std::string werr;  // the writer thread's error message (rtk_fail's buffer is thread-local)
    auto join_writer = [&] {
        if (writer.joinable()) writer.join();
        const int rc = wrc.load();
        return rc == RTK_OK ? rc : rtk_fail(rc, "%s", werr.c_str());
    };
    struct JoinAtExit {
        std::thread& t;
        ~JoinAtExit() {
            if (t.joinable()) t.join();
        }
    } join_at_exit{writer};
    for (int64_t c = 0; c < n_chunks; ++c) {
        const int sl = (int)(c % 2);
        const int64_t a = c * chunk_rows, rows = (a + chunk_rows <= n ? chunk_rows : n - a);
        if (c >= 2) CU(cudaEventSynchronize(j.h2d[sl]));  // the pinned buffer's last H2D has drained
        if (!parallel_io(read_full, in.fd, reinterpret_cast<char*>(B.pin_in[sl]), (size_t)rows * m * 4,
                         kHeader + a * m * 4, io_threads))
            return rtk_fail(RTK_ETRUNC, "unexpected end of file while reading matrix payload");
        if (trace.on && c < 3) trace("chunk read");
        if (c >= 2) CU(cudaStreamWaitEvent(j.s[0], j.kern[sl], 0));  // device input free again
        CU(cudaMemcpyAsync(B.d_in[sl], B.pin_in[sl], (size_t)rows * m * 4, cudaMemcpyHostToDevice, j.s[0]));
        CU(cudaEventRecord(j.h2d[sl], j.s[0]));
        CU(cudaStreamWaitEvent(j.s[1], j.h2d[sl], 0));
        if (c >= 2) CU(cudaStreamWaitEvent(j.s[1], j.d2h[sl], 0));  // device outputs copied out
        int rc;
        if (!k_ok)
            rc = rtk_nan_scan_f32(B.d_in[sl], rows, m, m, B.d_nan + c, j.s[1]);
        else if (mode == 0)
            rc = rtk_rowtopk_exact_f32(B.d_in[sl], rows, m, m, k, eps_rel, hard_cap, B.d_val[sl], B.d_idx[sl], k,
                                       nullptr, nullptr, B.d_nan + c, j.s[1]);
        else
            rc = rtk_rowtopk_early_f32(B.d_in[sl], rows, m, m, k, max_iter, B.d_val[sl], B.d_idx[sl], k, nullptr,
                                       nullptr, B.d_nan + c, j.s[1]);
        if (rc != RTK_OK) return rc;
        CU(cudaEventRecord(j.kern[sl], j.s[1]));
        if (k_ok) {
            if ((rc = join_writer()) != RTK_OK) return rc;  // chunk c-2's pinned outputs are free
            CU(cudaStreamWaitEvent(j.s[2], j.kern[sl], 0));
            CU(cudaMemcpyAsync(B.pin_val[sl], B.d_val[sl], (size_t)rows * kk * 4, cudaMemcpyDeviceToHost, j.s[2]));
            CU(cudaMemcpyAsync(B.pin_idx[sl], B.d_idx[sl], (size_t)rows * kk * 4, cudaMemcpyDeviceToHost, j.s[2]));
            CU(cudaEventRecord(j.d2h[sl], j.s[2]));
            if (c >= 1)
                writer = std::thread([&, c] {
                    const int rc = write_back(c - 1);
                    if (rc != RTK_OK) werr = rtk_last_error();
                    wrc = rc;
                });
        }
    }
    if (k_ok) {
        int rc = join_writer();
        if (rc == RTK_OK) rc = write_back(n_chunks - 1);
        if (rc != RTK_OK) return rc;
    }
    trace("all chunks written");
    CU(cudaStreamSynchronize(j.s[1]));
    std::vector<uint32_t> nan((size_t)n_chunks);
    CU(cudaMemcpy(nan.data(), B.d_nan, (size_t)n_chunks * 4, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < n_chunks; ++c) {
        if (nan[(size_t)c] != 0xffffffffu) {
            const int64_t row = c * chunk_rows + nan[(size_t)c];
            if (dims) dims[2] = row;
            return rtk_fail(RTK_ENAN, "matrix contains NaN (first offending row: %lld)", (long long)row);
        }
    }
    if (!k_ok) return rtk_fail(RTK_EINVAL, "k must be in [1, %lld], got %d", (long long)m, k);
    if (close(out.fd) != 0) {
        out.fd = -1;
        return rtk_fail(RTK_EIO, "%s: %s", result_path, strerror(errno));
    }
    out.fd = -1;
    if (rename(tmp.path.c_str(), result_path) != 0) return rtk_fail(RTK_EIO, "%s: %s", result_path, strerror(errno));
    tmp.path.clear();  // renamed: nothing to remove
    return RTK_OK;
}
