// timing.cpp -- per-launch CUDA-event timing by kernel class (qcs_timing_*).
//
// bench.py needs the average duration of the dominant kernel measured on the launching stream
// inside the timed region, plus the algorithmic bytes of each launch (32 B per touched
// amplitude, rounded to 32-byte sectors): the roofline's "achieved" figure.
#include <string>
#include <utility>
#include <vector>

#include "engine.hpp"

namespace qcs {

struct LaunchTimer {
    struct Rec {
        std::string cls;
        cudaEvent_t a, b;
        double bytes;
        cudaStream_t s;
    };
    struct Agg {
        u64 launches = 0;
        double ms = 0.0;
        double bytes = 0.0;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, Agg>> agg;

    cudaEvent_t take() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        QCS_CUDA(cudaEventCreate(&e));
        return e;
    }
    void resolve() {
        for (Rec& r : pending) {
            QCS_CUDA(cudaEventSynchronize(r.b));
            float ms = 0.f;
            QCS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            Agg* a = nullptr;
            for (auto& kv : agg)
                if (kv.first == r.cls) a = &kv.second;
            if (!a) {
                agg.emplace_back(r.cls, Agg{});
                a = &agg.back().second;
            }
            a->launches += 1;
            a->ms += ms;
            a->bytes += r.bytes;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    ~LaunchTimer() {
        for (Rec& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

namespace {
thread_local LaunchTimer* t_sink = nullptr;
}

TimerScope::TimerScope(qcs_state* s) : prev(t_sink) { t_sink = s ? s->timer : nullptr; }
TimerScope::~TimerScope() { t_sink = prev; }

TimedLaunch::TimedLaunch(const char* cls, double bytes, cudaStream_t s) {
    if (!t_sink) return;
    t = t_sink;
    LaunchTimer::Rec r{cls, t->take(), t->take(), bytes, s};
    QCS_CUDA(cudaEventRecord(r.a, s));
    t->pending.push_back(r);
    slot = int(t->pending.size()) - 1;
}

TimedLaunch::~TimedLaunch() {
    if (t) cudaEventRecord(t->pending[std::size_t(slot)].b, t->pending[std::size_t(slot)].s);
}

void timing_enable(qcs_state* s, bool on) {
    if (on && !s->timer) s->timer = new LaunchTimer;
    if (!on && s->timer) {
        delete s->timer;
        s->timer = nullptr;
    }
}

void timing_reset(qcs_state* s) {
    if (!s->timer) return;
    s->timer->resolve();
    s->timer->agg.clear();
}

int timing_count(qcs_state* s) {
    if (!s->timer) return 0;
    s->timer->resolve();
    return int(s->timer->agg.size());
}

void timing_entry(qcs_state* s, int i, const char** name, u64* launches, double* ms, double* bytes) {
    if (!s->timer || i < 0 || i >= int(s->timer->agg.size())) raise(QCS_ERR_ARG, "timing entry out of range");
    const auto& kv = s->timer->agg[std::size_t(i)];
    *name = kv.first.c_str();
    *launches = kv.second.launches;
    *ms = kv.second.ms;
    *bytes = kv.second.bytes;
}

void destroy_timer(LaunchTimer* t) { delete t; }

}  // namespace qcs
