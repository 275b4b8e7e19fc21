// engine.cpp -- the streaming engine behind ss_engine_* (include/specsense_b200.h).
//
// GPU form of runtime::run's data plane (proj/src/runtime.cpp:221-487) and
// frontend::PingPongBuffer (proj/include/specsense/frontend.hpp:86-135):
//
//   push()  : F-sample chunks -> the HBM bank of their window (w % n_banks),
//             one async H2D per run of consecutive rows on the copy stream.
//             The reference FFTs rows as they arrive; here the rows wait in
//             HBM and the whole window is transformed at once (K1 over T rows
//             is ~10-100 us), so a window's latency covers its FFT as well.
//   window complete: an event on the copy stream gates K1..K6 for that window
//             on the compute stream (its own ss_ctx, exact-pool CCL: no host
//             synchronisation anywhere on this path), then a D2H of the
//             boxes into the bank's pinned record and a `done` event.  A
//             completion thread spin-polls the done events in launch order,
//             stamps the completion time and queues the bank for poll()
//             (a cudaLaunchHostFunc callback showed 10-40 ms delivery
//             outliers at P rates; the spinning waiter is busy only while a
//             window is in flight).
//   poll()  : hands records out in completion order and releases the bank.
//
// Bank rules follow PingPongBuffer: rows of a window whose bank is still held
// are dropped and the window counts as one overrun (paced sources) or the
// writer waits for release (unpaced); rows of stale windows are ignored;
// lost ranges drop their windows.
#include "specsense_b200.h"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace ssb {
ss_status engine_ctx_open(int device, ss_ctx** out);
cudaStream_t engine_ctx_stream(ss_ctx* ctx);
ss_status engine_check(ss_ctx* ctx, int n_fft, int rows, ss_fmt fmt, double fs, const ss_detector_cfg& cfg);
ss_status engine_sense(ss_ctx* ctx, const void* diq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                       uint64_t start_seq, double fs, const ss_detector_cfg& cfg, float* tf, const ss_batch_out& dev,
                       const unsigned long long* seq_dev);
ss_status engine_check_stft(ss_ctx* ctx, int n_fft, int hop, int window, ss_fmt fmt);
void engine_add_launches(ss_ctx* ctx, int64_t n);
void engine_stage_events(ss_ctx* ctx, cudaEvent_t* ev16, bool* used8);
} // namespace ssb

namespace {

using Clock = std::chrono::steady_clock;

enum class BankState { Free, Filling, Busy };

struct Bank {
    BankState state = BankState::Free;
    uint64_t window = 0;
    uint64_t samples_in = 0;  // of the window's span
    // device
    unsigned char* iq = nullptr;
    float* tf = nullptr;
    float* psd_raw = nullptr;
    float* psd_smoothed = nullptr;
    float* floor_thr = nullptr;
    int32_t* active = nullptr;
    int32_t* n_active = nullptr;
    ss_box* boxes = nullptr;
    ss_bin_box* bin_boxes = nullptr;
    int32_t* n_boxes = nullptr;
    // pinned host record
    struct Host {
        unsigned long long seq;  // the window's start_seq, copied to d_seq before the graph runs
        int32_t n_boxes;
        int32_t n_active;
        float floor_thr[2];
    }* host = nullptr;
    unsigned long long* d_seq = nullptr;
    // pinned host staging for small / pageable pushes: window samples
    // [st_lo, st_hi) are staged, not yet copied; one H2D per kFlushRows chunks
    unsigned char* h_stage = nullptr;
    uint64_t st_lo = 0, st_hi = 0;
    cudaGraphExec_t graph = nullptr;  // K1..K6 + record D2H of this bank, captured once
    int64_t graph_launches = 0;
    ss_box* h_boxes = nullptr;
    ss_bin_box* h_bin_boxes = nullptr;
    cudaEvent_t rows_ready = nullptr;
    cudaEvent_t start_ev = nullptr;  // compute stream, before the window's first kernel
    cudaEvent_t done_ev = nullptr;   // compute stream, after the boxes' D2H
    cudaEvent_t stage_ev[16] = {};    // begin/end of each stage (K1..K6), event nodes of the graph
    bool stage_used[8] = {};
    double stage_s[8] = {};
    double gpu_s = 0.0;
    cudaError_t fault = cudaSuccess;  // the done event's query status, reported by poll
    bool poisoned = false;            // the filling window lost rows upstream: it can never complete
    Clock::time_point complete_at{};
    Clock::time_point done_at{};
};

} // namespace

struct ss_engine {
    ss_engine_cfg cfg{};
    ss_detector_cfg det{};
    ss_ctx* ctx = nullptr;
    cudaStream_t compute = nullptr;
    cudaStream_t copy = nullptr;
    int device = 0;
    size_t sbytes = 8;
    double deadline_s = 0.0;
    int hop = 0, window = 0;
    uint64_t stride = 0, span = 0;  // samples between window starts; samples per window
    uint64_t shards = 1, shard = 0;  // this engine owns windows w % shards == shard

    bool owns(uint64_t w) const { return w % shards == shard; }
    Clock::time_point t0{};
    std::vector<Bank> banks;

    std::mutex mu;
    std::condition_variable released;  // a bank went Free (writers waiting)
    std::condition_variable ready;     // a record is ready (poller waiting)
    std::deque<int> done;              // banks with records, completion order
    std::deque<int> inflight;          // banks launched, not yet complete (launch order)
    std::condition_variable launched_cv;
    std::thread waiter;
    bool stop = false;
    uint64_t completed = 0, overruns = 0, rows_retired = 0, launched = 0, polled = 0;
    // per bank slot: highest window counted as dropped, +1 (frontend.cpp:206-223
    // dropped_upto / count_drop: each window counted at most once, and rows of a
    // counted window are ignored)
    std::vector<uint64_t> dropped_upto;
    uint64_t newest_window = 0;        // highest window seen (rows of older, recycled windows are stale)
    bool finished = false;
    std::string err;

    double secs(Clock::time_point t) const { return std::chrono::duration<double>(t - t0).count(); }
};

namespace {

// pushes of at least this many rows from pinned / device memory go straight
// to HBM; smaller or pageable ones are staged in the bank's pinned buffer and
// leave in runs of kFlushRows rows (and at window completion)
constexpr int kDirectRows = 64;
constexpr int kFlushRows = 64;

ss_status efail(ss_engine* e, ss_status s, const std::string& msg) {
    e->err = msg;
    return s;
}

#define EN_CK(e, expr)                                                                                  \
    do {                                                                                                \
        cudaError_t c_ = (expr);                                                                        \
        if (c_ != cudaSuccess) return efail((e), SS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(c_)); \
    } while (0)

// Completion thread: waits for each launched window's done event in launch
// order (spin on cudaEventQuery, yield between polls), then publishes it.
void waiter_main(ss_engine* e) {
    cudaSetDevice(e->device);
    for (;;) {
        int bi;
        {
            std::unique_lock<std::mutex> lk(e->mu);
            e->launched_cv.wait(lk, [&] { return e->stop || !e->inflight.empty(); });
            if (e->inflight.empty()) return;  // stop requested and nothing in flight
            bi = e->inflight.front();
        }
        Bank& b = e->banks[static_cast<size_t>(bi)];
        cudaError_t st;
        while ((st = cudaEventQuery(b.done_ev)) == cudaErrorNotReady) std::this_thread::yield();
        const Clock::time_point now = Clock::now();
        float ms = 0.f;
        double stage_s[8] = {};
        if (st == cudaSuccess) {
            cudaEventElapsedTime(&ms, b.start_ev, b.done_ev);
            for (int i = 0; i < 8; ++i) {
                float t = 0.f;
                if (b.stage_used[i] && cudaEventElapsedTime(&t, b.stage_ev[2 * i], b.stage_ev[2 * i + 1]) == cudaSuccess)
                    stage_s[i] = 1e-3 * t;
            }
        }
        {
            std::lock_guard<std::mutex> lk(e->mu);
            e->inflight.pop_front();
            b.done_at = now;
            b.gpu_s = 1e-3 * ms;
            for (int i = 0; i < 8; ++i) b.stage_s[i] = stage_s[i];
            b.fault = st;
            e->done.push_back(bi);
        }
        e->ready.notify_all();
    }
}

ss_batch_out dev_out(const Bank& b, int cap) {
    ss_batch_out o{};
    o.psd_raw = b.psd_raw;
    o.psd_smoothed = b.psd_smoothed;
    o.floor_thr = b.floor_thr;
    o.active = b.active;
    o.n_active = b.n_active;
    o.boxes = b.boxes;
    o.bin_boxes = b.bin_boxes;
    o.n_boxes = b.n_boxes;
    o.box_capacity = cap;
    return o;
}

// Window of bank b is complete: launch its sensing.  Called with mu held.
ss_status launch_window(ss_engine* e, int bi) {
    Bank& b = e->banks[static_cast<size_t>(bi)];
    const int T = e->cfg.plot_rows;
    b.complete_at = Clock::now();
    EN_CK(e, cudaEventRecord(b.rows_ready, e->copy));
    EN_CK(e, cudaStreamWaitEvent(e->compute, b.rows_ready, 0));
    EN_CK(e, cudaEventRecord(b.start_ev, e->compute));
    b.host->seq = b.window * static_cast<uint64_t>(T);
    EN_CK(e, cudaMemcpyAsync(b.d_seq, &b.host->seq, sizeof(unsigned long long), cudaMemcpyHostToDevice, e->compute));
    EN_CK(e, cudaGraphLaunch(b.graph, e->compute));
    ssb::engine_add_launches(e->ctx, b.graph_launches);
    EN_CK(e, cudaEventRecord(b.done_ev, e->compute));
    b.state = BankState::Busy;
    e->inflight.push_back(bi);
    e->launched_cv.notify_one();
    ++e->completed;
    ++e->launched;
    return SS_OK;
}

// Bank for window w, or -1 when its rows must be dropped.  Called with lk held.
// w is a window this engine owns; its banks cycle over the owned windows
// (w / shards) so a sharded engine sees consecutive bank indices.
int bank_slot(const ss_engine* e, uint64_t w) {
    return static_cast<int>((w / e->shards) % static_cast<uint64_t>(e->cfg.n_banks));
}

bool already_dropped(const ss_engine* e, uint64_t w) {
    return w + 1 <= e->dropped_upto[static_cast<size_t>(bank_slot(e, w))];
}

// Counts window w as one overrun, at most once (windows needing drops arrive in
// nondecreasing order per bank slot).  mu held.
void count_drop(ss_engine* e, uint64_t w) {
    uint64_t& up = e->dropped_upto[static_cast<size_t>(bank_slot(e, w))];
    if (w + 1 > up) {
        up = w + 1;
        ++e->overruns;
    }
}

int claim_bank(ss_engine* e, uint64_t w, std::unique_lock<std::mutex>& lk) {
    if (already_dropped(e, w)) return -1;  // rows of a shed or lost window
    if (w + static_cast<uint64_t>(e->cfg.n_banks) * e->shards <= e->newest_window) return -1;  // stale row
    const int bi = bank_slot(e, w);
    for (;;) {
        Bank& b = e->banks[static_cast<size_t>(bi)];
        if (b.state == BankState::Filling && b.window == w) return b.poisoned ? -1 : bi;
        if (b.state == BankState::Filling && b.window < w) {
            // an older window never completed (rows lost upstream): shed it
            count_drop(e, b.window);
            b.state = BankState::Free;
        }
        if (b.state == BankState::Free) {
            b.state = BankState::Filling;
            b.window = w;
            b.samples_in = 0;
            b.st_lo = b.st_hi = 0;
            b.poisoned = false;
            e->newest_window = std::max(e->newest_window, w);
            return bi;
        }
        // Busy: held by the reader (or a newer window is filling it)
        if (b.state == BankState::Filling && b.window > w) return -1;
        if (e->cfg.paced) {
            count_drop(e, w);
            e->newest_window = std::max(e->newest_window, w);
            return -1;
        }
        e->released.wait(lk);
        if (e->finished) return -1;  // finish() / abort while waiting: drop the rows
    }
}

} // namespace

extern "C" {

ss_status ss_engine_open(int device, const ss_engine_cfg* cfg, const ss_detector_cfg* det, ss_engine** out) {
    if (!cfg || !det || !out) return SS_EVALIDATION;
    *out = nullptr;
    ss_engine* e = new ss_engine();
    e->cfg = *cfg;
    e->det = *det;
    e->device = device;
    if (e->cfg.n_banks == 0) e->cfg.n_banks = 2;
    if (e->cfg.box_capacity <= 0) e->cfg.box_capacity = 1024;
    ss_status s = ssb::engine_ctx_open(device, &e->ctx);
    if (s != SS_OK) {
        delete e;
        return s;
    }
    auto bad = [&](ss_status st, const std::string& m) {
        // keep the message reachable through the half-built engine
        e->err = m;
        *out = e;
        return st;
    };
    s = ssb::engine_check(e->ctx, cfg->n_fft, cfg->plot_rows, cfg->fmt, cfg->sample_rate_hz, *det);
    if (s != SS_OK) return bad(s, ss_last_error(e->ctx));
    if (e->cfg.n_banks < 2) return bad(SS_EVALIDATION, "n_banks must be >= 2");
    if (cfg->deadline_s < 0.0) return bad(SS_EVALIDATION, "deadline_s must be >= 0");
    const int F = cfg->n_fft, T = cfg->plot_rows, K = e->cfg.box_capacity;
    e->hop = cfg->hop > 0 ? cfg->hop : F;
    e->window = cfg->window;
    if (cfg->shard_count < 0 || (cfg->shard_count > 0 && (cfg->shard_index < 0 || cfg->shard_index >= cfg->shard_count)))
        return bad(SS_EVALIDATION, "shard_index must be in [0, shard_count)");
    e->shards = cfg->shard_count > 0 ? static_cast<uint64_t>(cfg->shard_count) : 1;
    e->shard = cfg->shard_count > 0 ? static_cast<uint64_t>(cfg->shard_index) : 0;
    s = ssb::engine_check_stft(e->ctx, F, e->hop, e->window, cfg->fmt);
    if (s != SS_OK) return bad(s, ss_last_error(e->ctx));
    e->sbytes = cfg->fmt == SS_FMT_F32 ? 8 : 4;
    e->stride = static_cast<uint64_t>(T) * e->hop;
    e->span = static_cast<uint64_t>(T - 1) * e->hop + F;
    e->deadline_s = cfg->deadline_s > 0.0 ? cfg->deadline_s : static_cast<double>(e->stride) / cfg->sample_rate_hz;
    e->compute = ssb::engine_ctx_stream(e->ctx);
    if (cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking) != cudaSuccess) return bad(SS_ECUDA, "copy stream");
    e->banks.resize(static_cast<size_t>(e->cfg.n_banks));
    e->dropped_upto.assign(static_cast<size_t>(e->cfg.n_banks), 0);
    const size_t cells = static_cast<size_t>(T) * F;  // TF plot
    const size_t iq_n = static_cast<size_t>(e->span);  // IQ samples per window
    for (Bank& b : e->banks) {
        bool ok = cudaMalloc(&b.iq, iq_n * e->sbytes) == cudaSuccess && cudaMalloc(&b.tf, cells * sizeof(float)) == cudaSuccess &&
                  cudaMalloc(&b.psd_raw, sizeof(float) * F) == cudaSuccess &&
                  cudaMalloc(&b.psd_smoothed, sizeof(float) * F) == cudaSuccess &&
                  cudaMalloc(&b.floor_thr, sizeof(float) * 2) == cudaSuccess &&
                  cudaMalloc(&b.active, sizeof(int32_t) * F) == cudaSuccess &&
                  cudaMalloc(&b.n_active, sizeof(int32_t)) == cudaSuccess &&
                  cudaMalloc(&b.boxes, sizeof(ss_box) * K) == cudaSuccess &&
                  cudaMalloc(&b.bin_boxes, sizeof(ss_bin_box) * K) == cudaSuccess &&
                  cudaMalloc(&b.n_boxes, sizeof(int32_t)) == cudaSuccess &&
                  cudaMallocHost(&b.host, sizeof(Bank::Host)) == cudaSuccess &&
                  cudaMalloc(&b.d_seq, sizeof(unsigned long long)) == cudaSuccess &&
                  cudaMallocHost(&b.h_stage, iq_n * e->sbytes) == cudaSuccess &&
                  cudaMallocHost(&b.h_boxes, sizeof(ss_box) * K) == cudaSuccess &&
                  cudaMallocHost(&b.h_bin_boxes, sizeof(ss_bin_box) * K) == cudaSuccess &&
                  cudaEventCreateWithFlags(&b.rows_ready, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreate(&b.start_ev) == cudaSuccess && cudaEventCreate(&b.done_ev) == cudaSuccess;
        if (!ok) return bad(SS_ECUDA, "engine bank allocation failed");
    }
    // warm-up: one window of zeros through the whole chain, so workspace,
    // twiddles and weights exist before the first real window is timed
    Bank& b0 = e->banks[0];
    if (cudaMemsetAsync(b0.iq, 0, iq_n * e->sbytes, e->compute) != cudaSuccess) return bad(SS_ECUDA, "memset");
    s = ssb::engine_sense(e->ctx, b0.iq, cfg->fmt, F, e->hop, e->window, T, 0, cfg->sample_rate_hz, *det, b0.tf,
                          dev_out(b0, K), nullptr);
    if (s != SS_OK) return bad(s, ss_last_error(e->ctx));
    if (cudaStreamSynchronize(e->compute) != cudaSuccess) return bad(SS_ECUDA, "warm-up failed");
    // capture each bank's window chain + record copies once: a window then
    // costs one H2D of its start_seq and one graph launch on the host
    for (Bank& b : e->banks) {
        if (cudaStreamBeginCapture(e->compute, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            return bad(SS_ECUDA, "graph capture");
        cudaGraph_t g = nullptr;
        for (cudaEvent_t& ev : b.stage_ev)
            if (cudaEventCreate(&ev) != cudaSuccess) return bad(SS_ECUDA, "event");
        if (cfg->stage_timing) ssb::engine_stage_events(e->ctx, b.stage_ev, nullptr);
        const ss_status cs = ssb::engine_sense(e->ctx, b.iq, cfg->fmt, F, e->hop, e->window, T, 0, cfg->sample_rate_hz,
                                               *det, b.tf, dev_out(b, K), b.d_seq);
        if (cfg->stage_timing) ssb::engine_stage_events(e->ctx, nullptr, b.stage_used);
        bool ok = cs == SS_OK &&
                  cudaMemcpyAsync(&b.host->n_boxes, b.n_boxes, sizeof(int32_t), cudaMemcpyDeviceToHost, e->compute) == cudaSuccess &&
                  cudaMemcpyAsync(&b.host->n_active, b.n_active, sizeof(int32_t), cudaMemcpyDeviceToHost, e->compute) == cudaSuccess &&
                  cudaMemcpyAsync(b.host->floor_thr, b.floor_thr, 2 * sizeof(float), cudaMemcpyDeviceToHost, e->compute) == cudaSuccess &&
                  cudaMemcpyAsync(b.h_boxes, b.boxes, sizeof(ss_box) * K, cudaMemcpyDeviceToHost, e->compute) == cudaSuccess &&
                  cudaMemcpyAsync(b.h_bin_boxes, b.bin_boxes, sizeof(ss_bin_box) * K, cudaMemcpyDeviceToHost, e->compute) == cudaSuccess;
        const cudaError_t ce = cudaStreamEndCapture(e->compute, &g);
        if (!ok || ce != cudaSuccess || !g) {
            if (g) cudaGraphDestroy(g);
            return bad(cs != SS_OK ? cs : SS_ECUDA, cs != SS_OK ? std::string(ss_last_error(e->ctx)) : "graph capture failed");
        }
        size_t nodes = 0;
        cudaGraphGetNodes(g, nullptr, &nodes);
        std::vector<cudaGraphNode_t> nv(nodes);
        cudaGraphGetNodes(g, nv.data(), &nodes);
        b.graph_launches = 0;
        for (cudaGraphNode_t nd : nv) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++b.graph_launches;
        }
        const cudaError_t ie = cudaGraphInstantiate(&b.graph, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return bad(SS_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    }
    if (cudaGraphUpload(e->banks[0].graph, e->compute) != cudaSuccess) return bad(SS_ECUDA, "graph upload");
    e->t0 = Clock::now();
    e->waiter = std::thread(waiter_main, e);
    *out = e;
    return SS_OK;
}

void ss_engine_close(ss_engine* e) {
    if (!e) return;
    if (e->waiter.joinable()) {
        {
            std::lock_guard<std::mutex> lk(e->mu);
            e->stop = true;
        }
        e->launched_cv.notify_all();
        e->waiter.join();
    }
    if (e->compute) cudaStreamSynchronize(e->compute);
    if (e->copy) {
        cudaStreamSynchronize(e->copy);
        cudaStreamDestroy(e->copy);
    }
    for (Bank& b : e->banks) {
        cudaFree(b.iq);
        cudaFree(b.tf);
        cudaFree(b.psd_raw);
        cudaFree(b.psd_smoothed);
        cudaFree(b.floor_thr);
        cudaFree(b.active);
        cudaFree(b.n_active);
        cudaFree(b.boxes);
        cudaFree(b.bin_boxes);
        cudaFree(b.n_boxes);
        cudaFreeHost(b.host);
        cudaFreeHost(b.h_boxes);
        cudaFreeHost(b.h_bin_boxes);
        if (b.rows_ready) cudaEventDestroy(b.rows_ready);
        if (b.graph) cudaGraphExecDestroy(b.graph);
        cudaFreeHost(b.h_stage);
        cudaFree(b.d_seq);
        if (b.start_ev) cudaEventDestroy(b.start_ev);
        if (b.done_ev) cudaEventDestroy(b.done_ev);
        for (cudaEvent_t ev : b.stage_ev)
            if (ev) cudaEventDestroy(ev);
    }
    if (e->ctx) ss_close(e->ctx);
    delete e;
}

const char* ss_engine_last_error(const ss_engine* e) { return e ? e->err.c_str() : "no engine"; }

static ss_status flush_stage(ss_engine* e, Bank& b) {
    if (b.st_hi > b.st_lo) {
        const size_t o = static_cast<size_t>(b.st_lo) * e->sbytes;
        EN_CK(e, cudaMemcpyAsync(b.iq + o, b.h_stage + o, static_cast<size_t>(b.st_hi - b.st_lo) * e->sbytes,
                                 cudaMemcpyHostToDevice, e->copy));
    }
    b.st_lo = b.st_hi;
    return SS_OK;
}

// Windows whose sample span meets the sample range [a0, a1).
static void windows_of(const ss_engine* e, uint64_t a0, uint64_t a1, uint64_t* w_lo, uint64_t* w_hi) {
    *w_lo = a0 >= e->span ? (a0 - e->span) / e->stride + 1 : 0;  // first w with w*stride + span > a0
    *w_hi = (a1 - 1) / e->stride;                               // last w with w*stride < a1
}

static ss_status push_impl(ss_engine* e, const void* samples, int64_t n_chunks, uint64_t first_seq, bool sync) {
    if (!e || (!samples && n_chunks > 0) || n_chunks < 0) return SS_EVALIDATION;
    if (n_chunks == 0) return SS_OK;
    const uint64_t F = static_cast<uint64_t>(e->cfg.n_fft);
    const unsigned char* src = static_cast<const unsigned char*>(samples);
    bool dma_ok = false;  // source is pinned or device memory
    if (n_chunks >= kDirectRows) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, samples) == cudaSuccess) dma_ok = a.type != cudaMemoryTypeUnregistered;
        else cudaGetLastError();
    }
    std::unique_lock<std::mutex> lk(e->mu);
    if (e->finished) return efail(e, SS_EVALIDATION, "push after finish");
    bool direct = false;  // a DMA straight from the caller's buffer was queued
    e->rows_retired += static_cast<uint64_t>(n_chunks);
    // the push's samples: [a0, a1); every window they meet gets its part
    const uint64_t a0 = first_seq * F, a1 = (first_seq + static_cast<uint64_t>(n_chunks)) * F;
    uint64_t w_lo, w_hi;
    windows_of(e, a0, a1, &w_lo, &w_hi);
    for (uint64_t w = w_lo; w <= w_hi; ++w) {
        if (!e->owns(w)) continue;  // another shard's window
        const uint64_t base = w * e->stride;
        const uint64_t s0 = std::max(a0, base), s1 = std::min(a1, base + e->span);
        if (s0 >= s1) continue;
        const int bi = claim_bank(e, w, lk);
        if (bi < 0) continue;
        Bank& b = e->banks[static_cast<size_t>(bi)];
        const uint64_t o0 = s0 - base, n = s1 - s0;  // window offset and count, samples
        const unsigned char* from = src + static_cast<size_t>(s0 - a0) * e->sbytes;
        if (dma_ok && n >= static_cast<uint64_t>(kDirectRows) * F) {
            ss_status s = flush_stage(e, b);
            if (s != SS_OK) return s;
            EN_CK(e, cudaMemcpyAsync(b.iq + static_cast<size_t>(o0) * e->sbytes, from, static_cast<size_t>(n) * e->sbytes,
                                     cudaMemcpyDefault, e->copy));
            direct = true;
        } else {
            if (o0 != b.st_hi) {  // not contiguous with the staged run
                ss_status s = flush_stage(e, b);
                if (s != SS_OK) return s;
                b.st_lo = b.st_hi = o0;
            }
            std::memcpy(b.h_stage + static_cast<size_t>(o0) * e->sbytes, from, static_cast<size_t>(n) * e->sbytes);
            b.st_hi = o0 + n;
            if (b.st_hi - b.st_lo >= static_cast<uint64_t>(kFlushRows) * F) {
                ss_status s = flush_stage(e, b);
                if (s != SS_OK) return s;
            }
        }
        b.samples_in += n;
        if (b.samples_in >= e->span) {
            ss_status s = flush_stage(e, b);
            if (s != SS_OK) return s;
            s = launch_window(e, bi);
            if (s != SS_OK) return s;
        }
    }
    if (direct && sync) {
        // The reference's push is synchronous: the caller may reuse its buffer
        // as soon as push returns, so wait for the DMA out of it (not for the
        // window's sensing).  Waited on outside the lock.
        cudaEvent_t ev;
        EN_CK(e, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        const cudaError_t r = cudaEventRecord(ev, e->copy);
        lk.unlock();
        const cudaError_t w = r == cudaSuccess ? cudaEventSynchronize(ev) : r;
        cudaEventDestroy(ev);
        if (w != cudaSuccess) {
            std::lock_guard<std::mutex> g(e->mu);
            return efail(e, SS_ECUDA, std::string("push copy: ") + cudaGetErrorString(w));
        }
    }
    return SS_OK;
}

ss_status ss_engine_push(ss_engine* e, const void* samples, int64_t n_chunks, uint64_t first_seq) {
    return push_impl(e, samples, n_chunks, first_seq, true);
}

// The caller keeps `samples` unchanged until ss_engine_push_fence (or the
// engine's finish / close): consecutive pushes' DMAs queue back to back.
ss_status ss_engine_push_async(ss_engine* e, const void* samples, int64_t n_chunks, uint64_t first_seq) {
    return push_impl(e, samples, n_chunks, first_seq, false);
}

ss_status ss_engine_push_fence(ss_engine* e) {
    if (!e) return SS_EVALIDATION;
    cudaEvent_t ev;
    EN_CK(e, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaError_t r;
    {
        std::lock_guard<std::mutex> lk(e->mu);
        r = cudaEventRecord(ev, e->copy);
    }
    const cudaError_t w = r == cudaSuccess ? cudaEventSynchronize(ev) : r;
    cudaEventDestroy(ev);
    if (w != cudaSuccess) {
        std::lock_guard<std::mutex> g(e->mu);
        return efail(e, SS_ECUDA, std::string("push fence: ") + cudaGetErrorString(w));
    }
    return SS_OK;
}

ss_status ss_engine_mark_lost(ss_engine* e, uint64_t first, uint64_t last) {
    if (!e) return SS_EVALIDATION;
    if (last <= first) return SS_OK;
    const uint64_t F = static_cast<uint64_t>(e->cfg.n_fft);
    std::lock_guard<std::mutex> lk(e->mu);
    e->rows_retired += last - first;
    uint64_t w_lo, w_hi;
    windows_of(e, first * F, last * F, &w_lo, &w_hi);
    for (uint64_t w = w_lo; w <= w_hi; ++w) {
        if (!e->owns(w)) continue;
        // every window the lost samples belong to drops once (with hop < F a
        // lost chunk can belong to several); a window already filling keeps its
        // bank, poisoned, until a newer window reclaims it (frontend.cpp:321-330)
        count_drop(e, w);
        Bank& b = e->banks[static_cast<size_t>(bank_slot(e, w))];
        if (b.state == BankState::Filling && b.window == w) b.poisoned = true;
        e->newest_window = std::max(e->newest_window, w);
    }
    return SS_OK;
}

ss_status ss_engine_finish(ss_engine* e) {
    if (!e) return SS_EVALIDATION;
    cudaStreamSynchronize(e->copy);  // copies out of ss_engine_push_async buffers are done
    {
        std::lock_guard<std::mutex> lk(e->mu);
        e->finished = true;
        for (Bank& b : e->banks)
            if (b.state == BankState::Filling) b.state = BankState::Free;  // partial tail window
    }
    e->ready.notify_all();
    e->released.notify_all();  // a push blocked on a held bank (reader gone) returns
    return SS_OK;
}

ss_status ss_engine_poll(ss_engine* e, int wait_ms, ss_plot_record* rec, ss_box* boxes, ss_bin_box* bin_boxes, int cap,
                         int* got) {
    if (!e || !got) return SS_EVALIDATION;
    *got = 0;
    std::unique_lock<std::mutex> lk(e->mu);
    auto has = [&] { return !e->done.empty() || (e->finished && e->polled == e->launched); };
    if (wait_ms < 0) e->ready.wait(lk, has);
    else if (wait_ms > 0) e->ready.wait_for(lk, std::chrono::milliseconds(wait_ms), has);
    if (e->done.empty()) return SS_OK;
    const int bi = e->done.front();
    e->done.pop_front();
    Bank& b = e->banks[static_cast<size_t>(bi)];
    const int K = e->cfg.box_capacity;
    const int nb = b.host->n_boxes;
    const int keep = std::min({nb, K, std::max(cap, 0)});
    if (rec) {
        rec->plot_index = b.window;
        rec->start_seq = b.window * static_cast<uint64_t>(e->cfg.plot_rows);
        rec->latency_s = std::chrono::duration<double>(b.done_at - b.complete_at).count();
        rec->deadline_s = e->deadline_s;
        rec->met = rec->latency_s <= e->deadline_s ? 1 : 0;
        rec->n_boxes = nb;
        rec->n_active = b.host->n_active;
        rec->noise_floor = b.host->floor_thr[0];
        rec->threshold = b.host->floor_thr[1];
        rec->complete_s = e->secs(b.complete_at);
        rec->done_s = e->secs(b.done_at);
        rec->gpu_s = b.gpu_s;
        for (int i = 0; i < 8; ++i) rec->stage_s[i] = b.stage_s[i];
    }
    if (boxes && keep > 0) std::memcpy(boxes, b.h_boxes, sizeof(ss_box) * static_cast<size_t>(keep));
    if (bin_boxes && keep > 0) std::memcpy(bin_boxes, b.h_bin_boxes, sizeof(ss_bin_box) * static_cast<size_t>(keep));
    b.state = BankState::Free;
    ++e->polled;
    *got = 1;
    const cudaError_t fault = b.fault;
    b.fault = cudaSuccess;
    if (fault != cudaSuccess) {
        // a device fault inside the window's graph: its record is not delivered as a result
        e->err = std::string("window ") + std::to_string(b.window) + ": " + cudaGetErrorString(fault);
        lk.unlock();
        e->released.notify_all();
        return SS_ECUDA;
    }
    lk.unlock();
    e->released.notify_all();
    if (nb > K) return efail(e, SS_ECAPACITY, "box capacity too small: " + std::to_string(nb));
    return SS_OK;
}

ss_status ss_engine_stats(ss_engine* e, uint64_t* completed, uint64_t* overruns, uint64_t* rows_retired,
                          uint64_t* pending) {
    if (!e) return SS_EVALIDATION;
    std::lock_guard<std::mutex> lk(e->mu);
    if (completed) *completed = e->completed;
    if (overruns) *overruns = e->overruns;
    if (rows_retired) *rows_retired = e->rows_retired;
    if (pending) *pending = e->launched - e->polled;
    return SS_OK;
}

} // extern "C"
