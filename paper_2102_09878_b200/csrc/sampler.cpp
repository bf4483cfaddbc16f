// Minimal in-process sampling profiler for the host side of the engine
// (the GPU box has no perf).  SPQR_SAMPLE=<path> turns it on for one
// factorization: SIGPROF every 100 us of CPU time (SPQR_SAMPLE_MASTER=1: of
// wall time, engine thread only) records the call stack;
// on stop, each frame is written as "<object> <offset>" so it can be
// symbolised offline (addr2line -f -C -e <object> <offset>).
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <sys/syscall.h>
#include <sys/time.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace spqr {

namespace {
constexpr int kDepth = 6;
constexpr int kMax = 400000;
void* g_buf[kMax][kDepth];
std::atomic<int> g_n{0};
bool g_on = false;
bool g_master = false;
timer_t g_timer;

void on_prof(int) {
    const int i = g_n.fetch_add(1);
    if (i >= kMax) return;
    void* tmp[kDepth + 2];
    const int d = backtrace(tmp, kDepth + 2);
    for (int k = 0; k < kDepth; ++k) g_buf[i][k] = (k + 2 < d) ? tmp[k + 2] : nullptr;
}
}  // namespace

void sampler_start() {
    if (!std::getenv("SPQR_SAMPLE") || g_on) return;
    void* warm[4];
    backtrace(warm, 4);  // load libgcc before the first signal
    g_n = 0;
    struct sigaction sa;
    std::memset(&sa, 0, sizeof sa);
    sa.sa_handler = on_prof;
    sa.sa_flags = SA_RESTART;
    sigaction(SIGPROF, &sa, nullptr);
    g_master = std::getenv("SPQR_SAMPLE_MASTER") != nullptr;
    if (g_master) {  // wall-clock samples of the calling (engine) thread only
        sigevent se;
        std::memset(&se, 0, sizeof se);
        se.sigev_notify = SIGEV_THREAD_ID;
        se.sigev_signo = SIGPROF;
        se._sigev_un._tid = static_cast<pid_t>(syscall(SYS_gettid));
        timer_create(CLOCK_MONOTONIC, &se, &g_timer);
        itimerspec its{{0, 100000}, {0, 100000}};
        timer_settime(g_timer, 0, &its, nullptr);
    } else {
        itimerval tv{{0, 100}, {0, 100}};
        setitimer(ITIMER_PROF, &tv, nullptr);
    }
    g_on = true;
}

void sampler_stop() {
    if (!g_on) return;
    if (g_master) {
        timer_delete(g_timer);
    } else {
        itimerval tv{{0, 0}, {0, 0}};
        setitimer(ITIMER_PROF, &tv, nullptr);
    }
    g_on = false;
    const char* path = std::getenv("SPQR_SAMPLE");
    FILE* f = std::fopen(path, "w");
    if (!f) return;
    const int n = std::min(g_n.load(), kMax);
    std::map<void*, std::pair<std::string, long>> cache;
    auto name = [&](void* a) -> std::string {
        auto it = cache.find(a);
        if (it != cache.end()) return it->second.first + " " + std::to_string(it->second.second);
        Dl_info di;
        std::string obj = "?";
        long off = 0;
        if (a && dladdr(a, &di) && di.dli_fname) {
            obj = di.dli_fname;
            off = static_cast<long>(static_cast<char*>(a) - static_cast<char*>(di.dli_fbase));
        }
        cache[a] = {obj, off};
        return obj + " " + std::to_string(off);
    };
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < kDepth; ++k) {
            if (!g_buf[i][k]) break;
            std::fprintf(f, "%s%s", k ? " | " : "", name(g_buf[i][k]).c_str());
        }
        std::fprintf(f, "\n");
    }
    std::fclose(f);
}

}  // namespace spqr
