// Serving scheduler. See scheduler.hpp for the design; the decision rules cited
// below are the reference's (proj/src/engine.cpp line numbers), restated over a
// flat per-request table with explicit device work items.
#include "scheduler.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <ostream>
#include <stdexcept>

#include "cronus/balancer.hpp"
#include "cronus/costmodel.hpp"

namespace cronus {
namespace sched {

bool BlockPool::alloc(int32_t& id) {
    if (in_use_ >= cap_) return false;
    if (!free_.empty()) {
        id = free_.top();
        free_.pop();
    } else {
        id = static_cast<int32_t>(minted_++);
    }
    ++in_use_;
    return true;
}

void BlockPool::release(int32_t id) {
    free_.push(id);
    --in_use_;
}

namespace {

constexpr double kTol = 1e-9;  // reference engine.cpp:21

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// Split ablation: CRONUS_FIXED_SPLIT=f in (0, 1] replaces the balancer's L_p by ceil(f * input)
// (the free-block and saturation guards still apply). Unset (the default): the reference rule.
double fixed_split_fraction() {
    static const double f = [] {
        const char* e = std::getenv("CRONUS_FIXED_SPLIT");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0.0 && v <= 1.0 ? v : 0.0;
    }();
    return f;
}

enum class Kind : uint8_t { Arrival, SerialDone, IterDone, TransferDone, Notify };

const char* kind_name(Kind k) {
    switch (k) {
        case Kind::Arrival: return "arrival";
        case Kind::SerialDone: return "serial-done";
        case Kind::IterDone: return "iter-done";
        case Kind::TransferDone: return "transfer-done";
        case Kind::Notify: return "notify";
    }
    return "?";
}

struct Event {
    double t;
    uint64_t seq;
    Kind kind;
    int arg;
};

// Min-heap order on (t, seq): equal times resolve by enqueue order.
struct Later {
    bool operator()(const Event& a, const Event& b) const {
        return a.t != b.t ? a.t > b.t : a.seq > b.seq;
    }
};

// Everything the scheduler tracks about one trace request.
struct Req {
    Request rq;
    // balancer output
    int lp = 0;
    bool full_on_ppi = false;
    int assigned = -1;
    // lifecycle
    double first_tok = -1.0;
    std::vector<double> tok_t;
    bool failed = false;
    bool done = false;
    // state on the chunked instance currently serving it
    long long need = 0;
    long long done_tok = 0;
    int emitted = 0;
    long long reserved = 0;
    std::vector<int32_t> kv;      // block table on the chunked instance
    std::vector<int32_t> ppi_kv;  // block table on the serial instance (until handoff)
};

struct Chunked {
    int idx = 0;
    std::string name;
    Role role = Role::DpEngine;
    const GpuProfile* prof = nullptr;
    int B = 512;
    long long cap = 0, reserved = 0, alloc = 0;
    BlockPool pool;
    std::deque<int> waiting;  // admission queue (dp / pure decode)
    std::deque<int> pending;  // cronus CPI: handed off by the PPI, transfer not started
    int in_transfer = 0;
    std::vector<int> running;  // admission order
    // iteration in flight
    bool busy = false;
    int chunk_rid = -1;
    long long chunk = 0;
    std::vector<int> decoders, finishers;
    double iter_t0 = 0.0;
    double iter_dur = 0.0;
    // counters
    uint64_t iters = 0;
    long long prefill_tok = 0, decode_tok = 0;
    int completions = 0;
    double busy_ms = 0.0;
};

struct Serial {
    int idx = 0;
    std::string name;
    Role role = Role::PPI;
    const GpuProfile* prof = nullptr;
    long long cap = 0, alloc = 0;
    BlockPool pool;
    std::deque<int> waiting;
    int cur = -1;
    long long cur_blocks = 0;
    bool busy = false;
    std::map<int, long long> held;  // rid -> blocks kept until the handoff completes
    double t0 = 0.0, dur = 0.0;
    uint64_t iters = 0;
    long long prefill_tok = 0;
    int completions = 0;
    double busy_ms = 0.0;
};

struct LinkXfer {
    int rid;
    long long tokens;
    double start, end;
};

class Core {
  public:
    Core(const ClusterConfig& cfg, const Trace& trace, const RunOptions& opts,
         const SchedulerHooks& hooks)
        : cfg_(cfg), trace_(trace), opts_(opts), hooks_(hooks), exec_(hooks.executor),
          wall_(exec_ && exec_->wall_clock()) {}

    RunReport run();

  private:
    const ClusterConfig& cfg_;
    const Trace& trace_;
    const RunOptions& opts_;
    const SchedulerHooks& hooks_;
    Executor* exec_;
    const bool wall_;

    std::vector<Req> req_;
    std::vector<Chunked> chunked_;
    std::vector<Serial> serial_;
    std::priority_queue<Event, std::vector<Event>, Later> events_;
    uint64_t seq_ = 0;
    double now_ = 0.0;
    std::vector<std::string> violations_;
    std::deque<int> frontend_;
    int dp_cursor_ = 0;
    int n_done_ = 0, n_failed_ = 0;
    double link_free_ = 0.0;
    std::vector<LinkXfer> xfers_;
    // wall clock: ticket -> event to raise on completion
    std::unordered_map<uint64_t, std::pair<Kind, int>> inflight_;

    // ---- infrastructure -----------------------------------------------------
    void violation(const std::string& m) {
        if (violations_.size() < 100) violations_.push_back(m);
    }
    void log(const char* who, Kind k, int rid) {
        if (!opts_.event_log) return;
        char line[192];
        std::snprintf(line, sizeof(line), "%.6f %s %s %d\n", now_, who, kind_name(k),
                      req_[rid].rq.id);
        *opts_.event_log << line;
    }
    void log_id(const char* who, Kind k, int id) {
        if (!opts_.event_log) return;
        char line[192];
        std::snprintf(line, sizeof(line), "%.6f %s %s %d\n", now_, who, kind_name(k), id);
        *opts_.event_log << line;
    }
    void post(double t, Kind k, int arg) { events_.push(Event{t, seq_++, k, arg}); }
    // Device work completes at now + modelled duration (virtual clock) or when the
    // device says so (wall clock).
    void complete_later(double dur, Kind k, int arg, uint64_t ticket) {
        if (wall_)
            inflight_.emplace(ticket, std::make_pair(k, arg));
        else
            post(now_ + dur, k, arg);
    }
    long long lifetime_blocks(const Req& r, const GpuProfile& g) const {
        return cdiv(r.rq.input_len + r.rq.output_len, g.kv_block_size);
    }

    // ---- KV block tables ----------------------------------------------------
    void grow(Chunked& ci, Req& r, long long blocks) {
        while (static_cast<long long>(r.kv.size()) < blocks) {
            int32_t id;
            if (!ci.pool.alloc(id)) {
                violation(ci.name + ": KV pool exhausted");
                return;
            }
            r.kv.push_back(id);
        }
    }
    void drop_kv(Chunked& ci, int rid) {
        Req& r = req_[rid];
        for (int32_t b : r.kv) ci.pool.release(b);
        r.kv.clear();
        if (exec_) exec_->release(ci.idx, rid);
    }
    void drop_ppi_kv(Serial& si, int rid) {
        Req& r = req_[rid];
        for (int32_t b : r.ppi_kv) si.pool.release(b);
        r.ppi_kv.clear();
        if (exec_) exec_->release(1000 + si.idx, rid);
    }

    // ---- request lifecycle --------------------------------------------------
    void first_token(int rid) {
        req_[rid].first_tok = now_;
        req_[rid].tok_t.push_back(now_);
    }
    void next_token(int rid) { req_[rid].tok_t.push_back(now_); }
    void fail(int rid, const std::string& where) {
        req_[rid].failed = true;
        ++n_failed_;
        log(where.c_str(), Kind::Arrival, rid);
    }
    void complete(int rid) {
        req_[rid].done = true;
        ++n_done_;
    }

    // ---- policy steps -------------------------------------------------------
    void build();
    void on_arrival(int rid);
    void handle(const Event& e);
    void settle();
    void idle_check();
    bool admit_cronus();
    bool admit_dp();
    bool start_handoffs(Chunked& ci);
    bool admit_chunked(Chunked& ci);
    bool start_iteration(Chunked& ci);
    void end_iteration(Chunked& ci);
    void refresh_ledger(Chunked& ci);
    bool start_prefill(Serial& si);
    void end_prefill(Serial& si);
    void begin_link(int rid, long long tokens);
    void end_link(int xfer);
    RunReport report();
};

void Core::build() {
    const PolicyBinding binding = bind_policy(cfg_);
    for (const InstanceSpec& spec : binding.instances) {
        const GpuProfile* prof = spec.on_high_gpu ? &cfg_.high_gpu : &cfg_.low_gpu;
        if (spec.role == Role::PPI || spec.role == Role::PurePrefill) {
            Serial s;
            s.idx = static_cast<int>(serial_.size());
            s.name = spec.name;
            s.role = spec.role;
            s.prof = prof;
            s.cap = prof->kv_blocks_capacity;
            s.pool = BlockPool(s.cap);
            serial_.push_back(std::move(s));
        } else if (spec.role == Role::PpStage) {
            throw std::invalid_argument(
                "policy pp: the pipeline-parallel baseline is not part of the B200 serving "
                "path (see DESIGN.md, out of scope)");
        } else {
            Chunked c;
            c.idx = static_cast<int>(chunked_.size());
            c.name = spec.name;
            c.role = spec.role;
            c.prof = prof;
            c.B = spec.max_batched_tokens;
            c.cap = prof->kv_blocks_capacity;
            c.pool = BlockPool(c.cap);
            chunked_.push_back(std::move(c));
        }
    }
    req_.resize(trace_.requests.size());
    for (size_t i = 0; i < trace_.requests.size(); ++i) {
        req_[i].rq = trace_.requests[i];
        post(trace_.requests[i].arrival_ms, Kind::Arrival, static_cast<int>(i));
    }
}

void Core::on_arrival(int rid) {
    log_id("frontend", Kind::Arrival, req_[rid].rq.id);
    switch (cfg_.policy) {
        case Policy::Cronus:
        case Policy::DpChunked: frontend_.push_back(rid); break;
        case Policy::DisaggHighLow:
        case Policy::DisaggLowHigh: serial_[0].waiting.push_back(rid); break;
        case Policy::PpChunked: break;  // rejected in build()
    }
}

// Frontend -> balancer -> PPI queue (paper steps 1-3; engine.cpp:331-358). The
// PPI accepts a new request only while its queue is empty and fewer than
// ppi_max_inflight requests are queued or running; the CPI snapshot is taken at
// that moment.
bool Core::admit_cronus() {
    Serial& ppi = serial_[0];
    Chunked& cpi = chunked_[0];
    bool moved = false;
    while (!frontend_.empty() && ppi.waiting.empty() &&
           (ppi.cur >= 0 ? 1 : 0) + static_cast<int>(ppi.waiting.size()) < cfg_.ppi_max_inflight) {
        const int rid = frontend_.front();
        frontend_.pop_front();
        CpiStats snap;
        snap.max_batched_tokens = cpi.B;
        snap.free_kv_blocks = cpi.cap - cpi.reserved;
        for (int r : cpi.running) {
            const Req& q = req_[r];
            if (q.done_tok == q.need && q.emitted >= 1) {
                ++snap.n_decode;
                snap.decode_ctx_sum += q.need + q.emitted;
            }
        }
        SplitDecision d = choose_split(cfg_.low_gpu, cfg_.high_gpu, snap, req_[rid].rq.input_len);
        if (const double f = fixed_split_fraction(); f > 0.0 && !d.full_on_ppi && !d.cpi_saturated) {
            // ablation (CRONUS_FIXED_SPLIT): a fixed fraction of the prompt instead of the balancer's L_p
            const int n = req_[rid].rq.input_len;
            d.partial_len = std::max(1, std::min(n, static_cast<int>(std::ceil(f * n))));
        }
        req_[rid].lp = d.partial_len;
        req_[rid].full_on_ppi = d.full_on_ppi;
        ppi.waiting.push_back(rid);
        moved = true;
    }
    return moved;
}

// Weighted round robin over the two DP engines with per-engine queue caps
// (engine.cpp:360-377).
bool Core::admit_dp() {
    bool moved = false;
    const int cycle = cfg_.dp_weight_high + cfg_.dp_weight_low;
    while (!frontend_.empty()) {
        const bool high = dp_cursor_ < cfg_.dp_weight_high;
        Chunked& eng = chunked_[high ? 0 : 1];
        const int qcap = high ? cfg_.dp_queue_cap_high : cfg_.dp_queue_cap_low;
        if (static_cast<int>(eng.waiting.size()) >= qcap) break;
        const int rid = frontend_.front();
        frontend_.pop_front();
        req_[rid].assigned = high ? 0 : 1;
        eng.waiting.push_back(rid);
        dp_cursor_ = (dp_cursor_ + 1) % cycle;
        moved = true;
    }
    return moved;
}

// CPI side of the handoff (paper steps 5-7; engine.cpp:379-403): reserve the
// request's lifetime KV on the CPI, then start the link transfer of its L_p
// prefix. Destination blocks are allocated now so the copy has somewhere to land.
bool Core::start_handoffs(Chunked& ci) {
    Serial& ppi = serial_[0];
    bool moved = false;
    while (!ci.pending.empty()) {
        const int rid = ci.pending.front();
        Req& r = req_[rid];
        const long long life = lifetime_blocks(r, *ci.prof);
        if (life > ci.cap) {
            ci.pending.pop_front();
            ppi.alloc -= ppi.held[rid];
            ppi.held.erase(rid);
            drop_ppi_kv(ppi, rid);
            fail(rid, ci.name);
            moved = true;
            continue;
        }
        if (static_cast<long long>(ci.running.size()) + ci.in_transfer >= ci.B) break;
        if (ci.reserved + life > ci.cap) break;
        ci.reserved += life;
        ci.in_transfer++;
        ci.pending.pop_front();
        r.reserved = life;
        grow(ci, r, cdiv(r.lp, ci.prof->kv_block_size));
        begin_link(rid, r.lp);
        moved = true;
    }
    return moved;
}

// Admission for DP engines and the disaggregated decode instance (engine.cpp:405-435).
bool Core::admit_chunked(Chunked& ci) {
    bool moved = false;
    const long long N = ci.prof->kv_block_size;
    while (!ci.waiting.empty()) {
        const int rid = ci.waiting.front();
        Req& r = req_[rid];
        const long long life = lifetime_blocks(r, *ci.prof);
        if (cdiv(r.rq.input_len, N) > ci.cap || life > ci.cap) {
            ci.waiting.pop_front();
            fail(rid, ci.name);
            moved = true;
            continue;
        }
        if (static_cast<long long>(ci.running.size()) >= ci.B) break;
        if (ci.reserved + life > ci.cap) break;
        ci.reserved += life;
        r.need = r.rq.input_len;
        r.reserved = life;
        r.done_tok = 0;
        r.emitted = 0;
        if (ci.role == Role::PureDecode) {  // KV arrived over the link; first token already out
            r.done_tok = r.rq.input_len;
            r.emitted = 1;
        }
        ci.running.push_back(rid);
        ci.waiting.pop_front();
        moved = true;
    }
    if (moved) refresh_ledger(ci);
    return moved;
}

// Compose and launch one chunked iteration (engine.cpp:437-480): every decoder
// contributes one token; the first entry still prefilling gets a chunk of
// min(B - n_decode, remaining); zero-remaining handoff finishers ride along free.
bool Core::start_iteration(Chunked& ci) {
    if (ci.busy) return false;
    ci.decoders.clear();
    ci.finishers.clear();
    ci.chunk_rid = -1;
    ci.chunk = 0;
    long long ctx_sum = 0;
    int head = -1;
    for (int rid : ci.running) {
        const Req& r = req_[rid];
        if (r.done_tok == r.need) {
            if (r.emitted >= 1) {
                ci.decoders.push_back(rid);
                ctx_sum += r.need + r.emitted;
            } else {
                ci.finishers.push_back(rid);
            }
        } else if (head < 0) {
            head = rid;
        }
    }
    const int n_d = static_cast<int>(ci.decoders.size());
    const long long budget = ci.B - n_d;
    if (head >= 0 && budget > 0) {
        ci.chunk = std::min(budget, req_[head].need - req_[head].done_tok);
        ci.chunk_rid = head;
    }
    if (n_d == 0 && ci.chunk == 0 && ci.finishers.empty()) return false;
    double pctx = 0.0;
    if (ci.chunk > 0)
        pctx = static_cast<double>(req_[head].done_tok + ci.chunk);
    else if (!ci.finishers.empty())
        pctx = static_cast<double>(req_[ci.finishers.front()].rq.input_len);
    if (n_d + ci.chunk > ci.B)
        violation(ci.name + ": batched tokens " + std::to_string(n_d + ci.chunk) + " > B");
    const double dur = chunked_iter_time(*ci.prof, pctx, static_cast<double>(ctx_sum));

    uint64_t ticket = 0;
    if (ci.chunk_rid >= 0) grow(ci, req_[ci.chunk_rid], cdiv(req_[ci.chunk_rid].done_tok + ci.chunk,
                                                             ci.prof->kv_block_size));
    if (exec_) {
        IterWork w;
        w.instance = ci.idx;
        w.decoders.reserve(ci.decoders.size());
        for (int rid : ci.decoders) {
            const Req& r = req_[rid];
            w.decoders.push_back(DecodeRow{rid, r.need + r.emitted, &r.kv});
        }
        if (ci.chunk_rid >= 0) {
            const Req& r = req_[ci.chunk_rid];
            w.chunk_rid = ci.chunk_rid;
            w.chunk_start = r.done_tok;
            w.chunk_len = ci.chunk;
            w.chunk_samples = r.done_tok + ci.chunk == r.need;
            w.chunk_blocks = &r.kv;
        }
        w.finishers = ci.finishers;
        ticket = exec_->iteration(w);
    }
    ci.busy = true;
    ci.iters++;
    ci.iter_t0 = now_;
    ci.iter_dur = dur;
    if (!wall_) ci.busy_ms += dur;
    log_id(ci.name.c_str(), Kind::IterDone, ci.chunk_rid >= 0 ? req_[ci.chunk_rid].rq.id : -1);
    complete_later(dur, Kind::IterDone, ci.idx, ticket);
    if (hooks_.iterations) {
        IterRecord rec;
        rec.instance = ci.idx;
        rec.t_start = now_;
        rec.n_decode = n_d;
        rec.decode_ctx_sum = ctx_sum;
        rec.chunk_rid = ci.chunk_rid;
        rec.chunk_start = ci.chunk_rid >= 0 ? req_[ci.chunk_rid].done_tok : 0;
        rec.chunk_len = ci.chunk;
        rec.n_finishers = static_cast<int>(ci.finishers.size());
        hooks_.iterations->push_back(rec);
    }
    return true;
}

// Iteration completion (engine.cpp:482-520), in the oracle's order: advance the
// chunk, decoders emit, finishers emit their first token, completions release
// their lifetime reservation and leave `running` (order preserved), ledger update.
void Core::end_iteration(Chunked& ci) {
    if (wall_) ci.busy_ms += now_ - ci.iter_t0;
    if (ci.chunk_rid >= 0) {
        Req& r = req_[ci.chunk_rid];
        r.done_tok += ci.chunk;
        ci.prefill_tok += ci.chunk;
        if (r.done_tok == r.need) ci.finishers.push_back(ci.chunk_rid);
    }
    bool any_done = false;
    for (int rid : ci.decoders) {
        Req& r = req_[rid];
        r.emitted++;
        ci.decode_tok++;
        next_token(rid);
        if (r.emitted == r.rq.output_len) {
            r.done = true;  // provisional mark; counted below
            any_done = true;
        }
    }
    for (int rid : ci.finishers) {
        Req& r = req_[rid];
        r.emitted = 1;
        first_token(rid);
        if (r.rq.output_len == 1) {
            r.done = true;
            any_done = true;
        }
    }
    if (any_done) {
        size_t keep = 0;
        for (size_t i = 0; i < ci.running.size(); ++i) {
            const int rid = ci.running[i];
            Req& r = req_[rid];
            if (r.done) {
                ci.reserved -= r.reserved;
                ci.completions++;
                r.done = false;
                complete(rid);
                drop_kv(ci, rid);
            } else {
                ci.running[keep++] = rid;
            }
        }
        ci.running.resize(keep);
    }
    ci.busy = false;
    ci.chunk_rid = -1;
    ci.chunk = 0;
    refresh_ledger(ci);
    if (hooks_.iterations && !hooks_.iterations->empty()) {
        // the record opened by this instance's start_iteration is the latest one of it
        for (auto it = hooks_.iterations->rbegin(); it != hooks_.iterations->rend(); ++it)
            if (it->instance == ci.idx) {
                it->t_end = now_;
                it->alloc_blocks = ci.alloc;
                break;
            }
    }
}

// Ledger (engine.cpp:522-531): alloc = sum ceil((done_tok + emitted) / N); the
// physical block tables are grown to exactly that.
void Core::refresh_ledger(Chunked& ci) {
    const long long N = ci.prof->kv_block_size;
    long long total = 0;
    for (int rid : ci.running) {
        Req& r = req_[rid];
        const long long want = cdiv(r.done_tok + r.emitted, N);
        // The in-flight chunk already holds the blocks its rows are writing.
        const long long held = ci.busy && rid == ci.chunk_rid ? std::max(want, cdiv(r.done_tok + ci.chunk, N)) : want;
        grow(ci, r, held);
        if (hooks_.check_ledger && static_cast<long long>(r.kv.size()) != held)
            violation(ci.name + ": block table of request " + std::to_string(r.rq.id) +
                      " holds " + std::to_string(r.kv.size()) + " blocks, ledger " +
                      std::to_string(want));
        total += want;
    }
    ci.alloc = total;
    if (ci.alloc > ci.cap)
        violation(ci.name + ": KV allocation " + std::to_string(ci.alloc) + " > capacity");
    if (ci.reserved > ci.cap)
        violation(ci.name + ": KV reservation " + std::to_string(ci.reserved) + " > capacity");
}

// Serial prefill (engine.cpp:533-562): one request at a time; its KV stays
// resident on this instance until the handoff completes.
bool Core::start_prefill(Serial& si) {
    if (si.busy) return false;
    while (!si.waiting.empty()) {
        const int rid = si.waiting.front();
        Req& r = req_[rid];
        const long long len = si.role == Role::PPI ? r.lp : r.rq.input_len;
        const long long blocks = cdiv(len, si.prof->kv_block_size);
        if (blocks > si.cap) {
            si.waiting.pop_front();
            fail(rid, si.name);
            continue;  // reported as a change by the caller's next pass
        }
        if (si.alloc + blocks > si.cap) return false;  // wait for held KV to drain
        si.waiting.pop_front();
        si.cur = rid;
        si.cur_blocks = blocks;
        si.alloc += blocks;
        r.ppi_kv.clear();
        for (long long b = 0; b < blocks; ++b) {
            int32_t id;
            if (!si.pool.alloc(id)) {
                violation(si.name + ": KV pool exhausted");
                break;
            }
            r.ppi_kv.push_back(id);
        }
        const double dur = prefill_time(*si.prof, static_cast<double>(len));
        uint64_t ticket = 0;
        if (exec_) {
            PrefillWork w;
            w.instance = si.idx;
            w.rid = rid;
            w.tokens = len;
            w.sample_last = len == r.rq.input_len;
            w.blocks = &r.ppi_kv;
            ticket = exec_->prefill(w);
        }
        si.busy = true;
        si.iters++;
        si.t0 = now_;
        si.dur = dur;
        if (!wall_) si.busy_ms += dur;
        si.prefill_tok += len;
        log(si.name.c_str(), Kind::SerialDone, rid);
        complete_later(dur, Kind::SerialDone, si.idx, ticket);
        if (hooks_.prefills) hooks_.prefills->push_back({si.idx, rid, len, now_, now_ + dur});
        return true;
    }
    return false;
}

void Core::end_prefill(Serial& si) {
    const int rid = si.cur;
    if (wall_) {
        si.busy_ms += now_ - si.t0;
        if (hooks_.prefills)
            for (auto it = hooks_.prefills->rbegin(); it != hooks_.prefills->rend(); ++it)
                if (it->rid == rid) {
                    it->t_end = now_;
                    break;
                }
    }
    si.cur = -1;
    si.busy = false;
    si.completions++;
    si.held[rid] = si.cur_blocks;
    log(si.name.c_str(), Kind::SerialDone, rid);
    if (si.role == Role::PPI)
        post(now_, Kind::Notify, rid);  // frontend forwards it to the CPI (step 4)
    else
        begin_link(rid, req_[rid].rq.input_len);
}

// Single FIFO link (engine.cpp:578-585).
void Core::begin_link(int rid, long long tokens) {
    const double begin = std::max(now_, link_free_);
    const double end = begin + transfer_time(cfg_.link, tokens);
    link_free_ = end;
    xfers_.push_back(LinkXfer{rid, tokens, begin, end});
    const int idx = static_cast<int>(xfers_.size()) - 1;
    uint64_t ticket = 0;
    if (exec_) {
        TransferWork w;
        w.rid = rid;
        w.tokens = tokens;
        w.src_instance = 0;
        w.dst_instance = 0;
        w.src_blocks = &req_[rid].ppi_kv;
        w.dst_blocks = &req_[rid].kv;
        ticket = exec_->transfer(w);
    }
    log("link", Kind::TransferDone, rid);
    if (hooks_.transfers) hooks_.transfers->push_back({rid, tokens, begin, end});
    if (wall_)
        inflight_.emplace(ticket, std::make_pair(Kind::TransferDone, idx));
    else
        post(end, Kind::TransferDone, idx);
}

// Handoff completion (engine.cpp:587-611): the PPI copy is released; under
// Cronus the request joins the CPI's running set with done_tok = L_p (the
// transferred prefix is never recomputed).
void Core::end_link(int xi) {
    const int rid = xfers_[xi].rid;
    if (wall_) {
        xfers_[xi].end = now_;
        if (hooks_.transfers) (*hooks_.transfers)[xi].t_end = now_;
    }
    log("link", Kind::TransferDone, rid);
    Serial& src = serial_[0];
    src.alloc -= src.held[rid];
    src.held.erase(rid);
    drop_ppi_kv(src, rid);
    Req& r = req_[rid];
    if (cfg_.policy == Policy::Cronus) {
        Chunked& cpi = chunked_[0];
        cpi.in_transfer--;
        r.need = r.rq.input_len;
        r.done_tok = r.lp;
        r.emitted = 0;
        r.reserved = lifetime_blocks(r, *cpi.prof);
        cpi.running.push_back(rid);
        refresh_ledger(cpi);
    } else {
        first_token(rid);  // disaggregated: TTFT includes the transfer
        if (r.rq.output_len == 1)
            complete(rid);
        else
            chunked_[0].waiting.push_back(rid);
    }
}

// Fixed point after every event (engine.cpp:809-824): frontend, serial starts,
// then per chunked instance handoffs -> admission -> iteration start.
void Core::settle() {
    for (bool again = true; again;) {
        again = false;
        if (cfg_.policy == Policy::Cronus) again |= admit_cronus();
        if (cfg_.policy == Policy::DpChunked) again |= admit_dp();
        for (Serial& si : serial_) {
            const size_t before = si.waiting.size();
            const bool started = start_prefill(si);
            again |= started || si.waiting.size() != before;
        }
        for (Chunked& ci : chunked_) {
            if (ci.role == Role::CPI) again |= start_handoffs(ci);
            again |= admit_chunked(ci);
            again |= start_iteration(ci);
        }
    }
}

// Work-conservation audit when time advances (engine.cpp:826-862).
void Core::idle_check() {
    for (const Chunked& ci : chunked_) {
        if (ci.busy) continue;
        bool runnable = !ci.running.empty();
        if (!runnable && !ci.waiting.empty()) {
            const long long life = lifetime_blocks(req_[ci.waiting.front()], *ci.prof);
            runnable = static_cast<long long>(ci.running.size()) < ci.B &&
                       ci.reserved + life <= ci.cap && life <= ci.cap;
        }
        if (runnable) violation(ci.name + ": idle at t=" + std::to_string(now_) + " with runnable work");
    }
    for (const Serial& si : serial_) {
        if (si.busy || si.waiting.empty()) continue;
        const Req& r = req_[si.waiting.front()];
        const long long len = si.role == Role::PPI ? r.lp : r.rq.input_len;
        const long long blocks = cdiv(len, si.prof->kv_block_size);
        if (blocks <= si.cap && si.alloc + blocks <= si.cap)
            violation(si.name + ": idle at t=" + std::to_string(now_) + " with runnable work");
    }
}

void Core::handle(const Event& e) {
    switch (e.kind) {
        case Kind::Arrival: on_arrival(e.arg); break;
        case Kind::SerialDone: end_prefill(serial_[e.arg]); break;
        case Kind::IterDone: end_iteration(chunked_[e.arg]); break;
        case Kind::TransferDone: end_link(e.arg); break;
        case Kind::Notify:
            log("frontend", Kind::Notify, e.arg);
            chunked_[0].pending.push_back(e.arg);
            break;
    }
}

RunReport Core::run() {
    const auto errs = validate_config(cfg_);
    if (!errs.empty()) {
        std::string all;
        for (const auto& m : errs) all += m + "; ";
        throw std::invalid_argument("invalid config: " + all);
    }
    if (trace_.requests.empty()) throw std::invalid_argument("empty trace");
    build();
    if (exec_) exec_->start();
    while (true) {
        if (wall_) {
            // Fold every finished device operation into the event queue with its
            // device timestamp, then release events whose time has come.
            Completion c;
            while (exec_->poll(c)) {
                auto it = inflight_.find(c.ticket);
                if (it == inflight_.end()) throw std::logic_error("unknown completion ticket");
                post(c.t_ms, it->second.first, it->second.second);
                inflight_.erase(it);
            }
            if (events_.empty()) {
                if (inflight_.empty()) break;
                exec_->wait(std::numeric_limits<double>::infinity());
                continue;
            }
            const double due = events_.top().t;
            if (due > exec_->now_ms()) {
                exec_->wait(due);
                if (exec_->now_ms() < due) continue;  // woke on a completion
            }
        } else if (events_.empty()) {
            break;
        }
        const Event e = events_.top();
        events_.pop();
        if (!wall_ && e.t + kTol < now_) violation("event time regression at t=" + std::to_string(e.t));
        if (e.t > now_ + kTol) idle_check();
        now_ = std::max(now_, e.t);
        handle(e);
        settle();
    }
    if (exec_) exec_->finish();
    return report();
}

RunReport Core::report() {
    RunReport rep;
    rep.policy = policy_name(cfg_.policy);
    rep.trace_name = trace_.name;
    rep.trace_hash = trace_hash(trace_);
    rep.n_requests = static_cast<int>(trace_.requests.size());
    double t0 = trace_.requests.front().arrival_ms;
    for (const Request& q : trace_.requests) t0 = std::min(t0, q.arrival_ms);
    rep.t_start_ms = t0;
    rep.t_end_ms = t0;
    for (const Req& r : req_) {
        if (r.failed) {
            rep.failed_ids.push_back(r.rq.id);
            continue;
        }
        if (!r.done) continue;
        RequestRecord rec;
        rec.id = r.rq.id;
        rec.ttft_ms = r.first_tok - r.rq.arrival_ms;
        rec.completion_ms = r.tok_t.back();
        rec.partial_prefill_len = r.lp;
        rec.assigned_instance = r.assigned;
        rec.tbt_samples_ms.reserve(r.tok_t.size());
        for (size_t i = 1; i < r.tok_t.size(); ++i) rec.tbt_samples_ms.push_back(r.tok_t[i] - r.tok_t[i - 1]);
        if (static_cast<int>(r.tok_t.size()) != r.rq.output_len)
            violation("request " + std::to_string(r.rq.id) + ": emitted " + std::to_string(r.tok_t.size()) +
                      " tokens, expected " + std::to_string(r.rq.output_len));
        if (rec.ttft_ms > rec.completion_ms - r.rq.arrival_ms + kTol)
            violation("request " + std::to_string(r.rq.id) + ": ttft after completion");
        rep.records.push_back(std::move(rec));
    }
    if (n_done_ + n_failed_ < rep.n_requests) {
        std::string ids;
        int shown = 0;
        for (const Req& r : req_)
            if (!r.done && !r.failed && shown++ < 10) ids += " " + std::to_string(r.rq.id);
        violation("deadlock: no runnable event with pending requests:" + ids);
    }
    for (const Chunked& ci : chunked_) {
        if (ci.reserved != 0 || ci.alloc != 0) violation(ci.name + ": KV ledger not drained at quiescence");
        rep.instances.push_back(InstanceSummary{ci.name, role_name(ci.role), ci.iters, ci.prefill_tok,
                                                ci.decode_tok, ci.completions, ci.busy_ms});
    }
    for (const Serial& si : serial_) {
        if (si.alloc != 0 || !si.held.empty()) violation(si.name + ": KV buffer not drained at quiescence");
        rep.instances.push_back(
            InstanceSummary{si.name, role_name(si.role), si.iters, si.prefill_tok, 0, si.completions, si.busy_ms});
    }
    rep.violations = violations_;
    finalize_report(rep);
    if (opts_.compute_utilization && rep.n_completed > 0) {
        const int Bh = cfg_.max_batched_tokens_high, Bl = cfg_.max_batched_tokens_low;
        switch (cfg_.policy) {
            case Policy::DisaggHighLow:
                rep.util_high = relative_utilization(rep.throughput_rps, standalone_prefill_rps(cfg_.high_gpu, trace_));
                rep.util_low =
                    relative_utilization(rep.throughput_rps, standalone_decode_rps(cfg_.low_gpu, Bl, trace_));
                break;
            case Policy::DisaggLowHigh:
                rep.util_low = relative_utilization(rep.throughput_rps, standalone_prefill_rps(cfg_.low_gpu, trace_));
                rep.util_high =
                    relative_utilization(rep.throughput_rps, standalone_decode_rps(cfg_.high_gpu, Bh, trace_));
                break;
            case Policy::Cronus:
                rep.util_high =
                    relative_utilization(rep.throughput_rps, standalone_chunked_rps(cfg_.high_gpu, Bh, trace_));
                rep.util_low = relative_utilization(rep.throughput_rps, standalone_prefill_rps(cfg_.low_gpu, trace_));
                break;
            default: break;
        }
    }
    return rep;
}

}  // namespace

RunReport run_scheduler(const ClusterConfig& cfg, const Trace& trace, const RunOptions& opts,
                        const SchedulerHooks& hooks) {
    Core core(cfg, trace, opts, hooks);
    return core.run();
}

}  // namespace sched
}  // namespace cronus
