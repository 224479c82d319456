// Per-rule join kernels: the compiler half of the paper's design ("rules are
// translated into a staged pipeline of CUDA kernels rather than interpreted
// at runtime"), done at run time on the host with NVRTC.
//
// For a plan descriptor, the static part of its shape (depth, atoms, the
// index columns each atom binds at each level, negations, the head
// projection, the plan class) is printed as a C++ type whose accessors are
// constexpr; wcoj_kernel.cuh is compiled for that type and sm_100a, so the
// shape loops unroll and every atom property is an immediate. The index
// pointers, row ranges and segment counts stay run-time data in the same
// srdl_plan, so one compiled kernel serves every iteration and every
// relation version of the rule instance.
//
// Caching: per process (shape key + mode -> kernel handle), and on disk as
// cubin under $SRDL_JIT_CACHE (default ~/.cache/srdl-jit), keyed by a hash
// of the generated source, the kernel header sources and the options. NVRTC
// is opened with dlopen, so the library loads without it.
//
// Modes (SRDL_JIT, srdl_wcoj_jit_set_mode): async (default) — a plan runs
// on the generic kernel of its class until its own kernel has been built by
// the background compiler (the engine schedules a program's plans when it is
// created); sync — compile on first use; 0 — generic kernels only. Both
// kernels walk the same slices in the same order, so results, counts and
// output order are identical whichever runs.
#include <dlfcn.h>
#include <stdlib.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "wcoj_jit.h"
#include "wcoj_kernel.cuh"

namespace srdl {
namespace {

// ----------------------------------------------------------- NVRTC (dlopen)

typedef int nvrtcResult_;
typedef struct _nvrtcProgram *nvrtcProgram_;

struct Nvrtc {
    bool ok = false;
    nvrtcResult_ (*create)(nvrtcProgram_ *, const char *, const char *, int, const char *const *,
                           const char *const *) = nullptr;
    nvrtcResult_ (*compile)(nvrtcProgram_, int, const char *const *) = nullptr;
    nvrtcResult_ (*log_size)(nvrtcProgram_, size_t *) = nullptr;
    nvrtcResult_ (*log)(nvrtcProgram_, char *) = nullptr;
    nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t *) = nullptr;
    nvrtcResult_ (*cubin)(nvrtcProgram_, char *) = nullptr;
    nvrtcResult_ (*destroy)(nvrtcProgram_ *) = nullptr;
};

const Nvrtc &nvrtc() {
    static Nvrtc N = [] {
        Nvrtc n;
        void *h = nullptr;
        for (const char *name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
            h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (h) break;
        }
        if (!h) return n;
        n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
        n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
        n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
        n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
        n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
        n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
        n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
        return n;
    }();
    return N;
}

// ------------------------------------------------------------- sources

std::string dir_of(const std::string &path) {
    const size_t k = path.rfind('/');
    return k == std::string::npos ? std::string(".") : path.substr(0, k);
}

// csrc/ and include/ next to libsrdl.so (the in-tree build), or SRDL_SOURCE_DIR
struct Paths {
    std::string csrc, include;
};

const Paths &paths() {
    static Paths P = [] {
        Paths p;
        const char *env = getenv("SRDL_SOURCE_DIR");
        std::string pkg;
        if (env && *env) {
            pkg = env;
        } else {
            Dl_info info;
            if (dladdr((void *)&jit_kernel, &info) && info.dli_fname) pkg = dir_of(info.dli_fname);
        }
        p.csrc = pkg + "/csrc";
        p.include = dir_of(pkg) + "/include";
        return p;
    }();
    return P;
}

std::string read_file(const std::string &path) {
    std::ifstream f(path, std::ios::binary);
    std::ostringstream o;
    o << f.rdbuf();
    return o.str();
}

uint64_t fnv1a(const std::string &s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

// ------------------------------------------------------------- shapes

// The static part of a plan (everything the kernel reads from srdl_plan
// except pointers, row ranges and segment counts), as a compact key.
std::string shape_key(const srdl_plan *P, int mode) {
    std::ostringstream k;
    k << "m" << mode << "d" << P->depth << "a" << P->natoms << "o" << P->outer << "i" << P->inner << "h"
      << P->head_arity << "n" << P->nmid << ":";
    for (uint32_t h = 0; h < P->head_arity; ++h) k << P->head_level[h] << ",";
    k << ":";
    for (uint32_t L = 0; L < P->depth; ++L) {
        k << P->nspec[L] << "[";
        for (uint32_t j = 0; j < P->nspec[L]; ++j) k << (int)P->spec[L][j] << ",";
        k << "]";
    }
    k << ":";
    for (uint32_t a = 0; a < P->natoms; ++a) {
        const srdl_atom &A = P->atom[a];
        k << (int)P->leaf_slot[a] << "/" << (int)P->mid_slot[a] << "/" << A.negated << "/" << A.check_level << "(";
        for (uint32_t L = 0; L < P->depth; ++L) k << (int)A.lvl_col[L] << "." << (int)A.lvl_ncol[L] << ",";
        k << ")";
    }
    return k.str();
}

// constexpr table lookup as nested conditionals (folds when the indices are
// constants, a short compare chain otherwise)
template <class F>
std::string table(const char *i, uint32_t n, F value) {
    std::ostringstream o;
    for (uint32_t x = 0; x < n; ++x) o << "(" << i << " == " << x << "u) ? " << value(x) << " : ";
    o << "0";
    return o.str();
}

std::string shape_source(const srdl_plan *P, int mode) {
    const int kind = plan_class(P->depth, P->nmid);
    std::ostringstream o;
    o << "// generated: per-plan WCOJ kernel (csrc/wcoj_jit.cu)\n"
      << "#define SRDL_JIT 1\n#include \"wcoj_kernel.cuh\"\nnamespace srdl {\nstruct JitShape {\n"
      << "#define F static __device__ __forceinline__ constexpr\n";
    o << "F uint32_t depth(const srdl_plan &) { return " << P->depth << "u; }\n";
    o << "F uint32_t natoms(const srdl_plan &) { return " << P->natoms << "u; }\n";
    o << "F uint32_t outer(const srdl_plan &) { return " << P->outer << "u; }\n";
    o << "F uint32_t inner(const srdl_plan &) { return " << P->inner << "u; }\n";
    o << "F uint32_t head_arity(const srdl_plan &) { return " << P->head_arity << "u; }\n";
    o << "F uint32_t nmid(const srdl_plan &) { return " << P->nmid << "u; }\n";
    o << "F int head_level(const srdl_plan &, uint32_t h) { return "
      << table("h", P->head_arity, [&](uint32_t h) { return std::to_string(P->head_level[h]); }) << "; }\n";
    o << "F uint32_t nspec(const srdl_plan &, int L) { return "
      << table("(uint32_t)L", P->depth, [&](uint32_t L) { return std::to_string(P->nspec[L]) + "u"; }) << "; }\n";
    o << "F uint32_t spec(const srdl_plan &, int L, uint32_t j) { return "
      << table("(uint32_t)L", P->depth,
               [&](uint32_t L) {
                   return "(" + table("j", P->nspec[L], [&](uint32_t j) {
                              return std::to_string((int)P->spec[L][j]) + "u";
                          }) + ")";
               })
      << "; }\n";
    o << "F uint32_t leaf_slot(const srdl_plan &, uint32_t a) { return "
      << table("a", P->natoms, [&](uint32_t a) { return std::to_string((int)P->leaf_slot[a]) + "u"; }) << "; }\n";
    o << "F uint32_t mid_slot(const srdl_plan &, uint32_t a) { return "
      << table("a", P->natoms, [&](uint32_t a) { return std::to_string((int)P->mid_slot[a]) + "u"; }) << "; }\n";
    o << "F bool negated(const srdl_plan &, uint32_t a) { return "
      << table("a", P->natoms, [&](uint32_t a) { return P->atom[a].negated ? std::string("true") : std::string("false"); })
      << "; }\n";
    o << "F int check_level(const srdl_plan &, uint32_t a) { return "
      << table("a", P->natoms, [&](uint32_t a) { return std::to_string(P->atom[a].check_level); }) << "; }\n";
    for (const char *which : {"lvl_col", "lvl_ncol"}) {
        const bool col = which[4] == 'c';
        o << "F uint32_t " << which << "(const srdl_plan &, uint32_t a, int L) { return "
          << table("a", P->natoms,
                   [&](uint32_t a) {
                       return "(" + table("(uint32_t)L", P->depth, [&](uint32_t L) {
                                  return std::to_string(col ? (int)P->atom[a].lvl_col[L] : (int)P->atom[a].lvl_ncol[L]) +
                                         "u";
                              }) + ")";
                   })
          << "; }\n";
    }
    o << "#undef F\n};\n}  // namespace srdl\n"
      << "extern \"C\" __global__ void __launch_bounds__(srdl::kJoinWarps * 32, srdl::kMinBlocks)\n"
      << "srdl_jit_wcoj(const __grid_constant__ srdl_plan P, const __grid_constant__ srdl_exec X,\n"
      << "              const __grid_constant__ srdl_spec Q) {\n"
      << "    srdl::wcoj_body<" << mode << ", " << kind << ", srdl::JitShape>(P, X, Q);\n}\n";
    return o.str();
}

const std::vector<std::string> &compile_options() {
    static std::vector<std::string> opts = [] {
        std::vector<std::string> o = {
            "--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-default-device",
            "-I" + paths().csrc,          "-I" + paths().include,
        };
        // extra -D options (tuning sweeps, e.g. -DSRDL_MERGE_RATIO=4), space-separated
        if (const char *e = getenv("SRDL_JIT_DEFINES")) {
            std::istringstream in(e);
            std::string tok;
            while (in >> tok) o.push_back(tok);
        }
        return o;
    }();
    return opts;
}

// hash of everything the cubin depends on besides the generated source
uint64_t sources_hash() {
    static uint64_t h = [] {
        uint64_t x = fnv1a(read_file(paths().csrc + "/wcoj_kernel.cuh"));
        x = fnv1a(read_file(paths().csrc + "/common.cuh"), x);
        x = fnv1a(read_file(paths().include + "/srdl.h"), x);
        for (const auto &o : compile_options()) x = fnv1a(o, x);
        return x;
    }();
    return h;
}

std::string cache_dir() {
    const char *env = getenv("SRDL_JIT_CACHE");
    if (env) return env;  // "" disables the disk cache
    const char *home = getenv("HOME");
    return home ? std::string(home) + "/.cache/srdl-jit" : std::string();
}

bool compile_cubin(const std::string &src, std::string *cubin, std::string *log) {
    const Nvrtc &N = nvrtc();
    nvrtcProgram_ prog = nullptr;
    if (N.create(&prog, src.c_str(), "srdl_jit_wcoj.cu", 0, nullptr, nullptr) != 0) {
        *log = "nvrtcCreateProgram failed";
        return false;
    }
    std::vector<const char *> argv;
    for (const auto &o : compile_options()) argv.push_back(o.c_str());
    const int rc = N.compile(prog, (int)argv.size(), argv.data());
    size_t n = 0;
    N.log_size(prog, &n);
    log->assign(n, '\0');
    if (n) N.log(prog, &(*log)[0]);
    bool ok = rc == 0;
    if (ok) {
        N.cubin_size(prog, &n);
        cubin->assign(n, '\0');
        ok = N.cubin(prog, &(*cubin)[0]) == 0;
    }
    N.destroy(&prog);
    return ok;
}

struct Entry {
    std::mutex mu;
    int state = 0;  // 0 new, 1 compiling, 2 done (kernel, or nullptr after a failure)
    srdl_plan plan{};
    int mode = 0;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    uint64_t attr_devices = 0;  // devices with the shared-memory attribute raised
};

std::mutex g_mu;
std::unordered_map<std::string, std::shared_ptr<Entry>> g_cache;
std::atomic<uint64_t> g_compiled{0}, g_disk_hits{0}, g_failures{0};

// 0 off, 1 async (default: plans run on the generic kernels until their own
// kernel is compiled in the background), 2 sync (compile on first use)
std::atomic<int> g_mode{[] {
    const char *e = getenv("SRDL_JIT");
    if (!e || !*e) return 1;
    if (e[0] == '0') return 0;
    if (e[0] == 's') return 2;
    return 1;
}()};

void build_entry(Entry &E) {
    const std::string src = shape_source(&E.plan, E.mode);
    const uint64_t h = fnv1a(src, sources_hash());
    char name[32];
    snprintf(name, sizeof(name), "%016llx.cubin", (unsigned long long)h);
    const std::string dir = cache_dir();
    std::string cubin;
    if (!dir.empty()) {
        cubin = read_file(dir + "/" + name);
        if (!cubin.empty()) g_disk_hits++;
    }
    if (cubin.empty()) {
        std::string log;
        if (!compile_cubin(src, &cubin, &log)) {
            g_failures++;
            fprintf(stderr, "[srdl] per-plan kernel compile failed, the generic kernel runs instead:\n%.2000s\n",
                    log.c_str());
            return;
        }
        g_compiled++;
        if (!dir.empty()) {  // best effort: write to a temp name, rename into place
            mkdir(dir.c_str(), 0755);
            const std::string tmp = dir + "/" + name + ".tmp" + std::to_string((long)getpid());
            std::ofstream(tmp, std::ios::binary).write(cubin.data(), (std::streamsize)cubin.size());
            rename(tmp.c_str(), (dir + "/" + name).c_str());
        }
    }
    if (cudaLibraryLoadData(&E.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&E.kernel, E.lib, "srdl_jit_wcoj") != cudaSuccess) {
        cudaGetLastError();
        g_failures++;
        E.kernel = nullptr;
        fprintf(stderr, "[srdl] per-plan kernel load failed, the generic kernel runs instead\n");
    }
}

// background compiler: a queue drained by up to kWorkers threads
struct Pool {
    std::mutex mu;
    std::condition_variable cv, idle;
    std::vector<std::shared_ptr<Entry>> queue;
    int device = 0;
    unsigned running = 0, busy = 0;
};
Pool g_pool;

void run_entry(const std::shared_ptr<Entry> &e) {
    std::lock_guard<std::mutex> lock(e->mu);
    if (e->state != 2) {
        build_entry(*e);
        e->state = 2;
    }
}

void worker(int dev) {
    cudaSetDevice(dev);
    std::unique_lock<std::mutex> lock(g_pool.mu);
    while (!g_pool.queue.empty()) {
        auto e = g_pool.queue.back();
        g_pool.queue.pop_back();
        g_pool.busy++;
        lock.unlock();
        run_entry(e);
        lock.lock();
        g_pool.busy--;
    }
    g_pool.running--;
    g_pool.idle.notify_all();
}

void enqueue(const std::shared_ptr<Entry> &e) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_pool.mu);
    g_pool.queue.push_back(e);
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned cap = hw ? (hw < 32 ? hw : 32) : 4;
    if (g_pool.running < cap) {
        g_pool.running++;
        std::thread(worker, dev).detach();
    }
}

std::shared_ptr<Entry> entry_for(const srdl_plan *P, int mode) {
    const std::string key = shape_key(P, mode);
    std::lock_guard<std::mutex> lock(g_mu);
    auto &slot = g_cache[key];
    if (!slot) {
        slot = std::make_shared<Entry>();
        slot->plan = *P;
        slot->mode = mode;
    }
    return slot;
}

}  // namespace

const void *jit_kernel(const srdl_plan *P, int mode) {
    const int m = g_mode.load();
    if (m == 0 || !nvrtc().ok) return nullptr;
    std::shared_ptr<Entry> e = entry_for(P, mode);
    {
        std::unique_lock<std::mutex> lock(e->mu, std::defer_lock);
        if (m == 2) {
            lock.lock();
            if (e->state != 2) {
                build_entry(*e);
                e->state = 2;
            }
        } else {
            if (!lock.try_lock()) return nullptr;  // being compiled in the background
            if (e->state == 0) {
                e->state = 1;
                lock.unlock();
                enqueue(e);
                return nullptr;
            }
            if (e->state != 2) return nullptr;
        }
    }
    if (!e->kernel) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lock(e->mu);
    if (!(e->attr_devices & bit)) {
        SRDL_CUDA(cudaFuncSetAttribute((const void *)e->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
        e->attr_devices |= bit;
    }
    return (const void *)e->kernel;
}

}  // namespace srdl

using namespace srdl;

extern "C" {

// Schedule the per-plan kernels of n plans in `mode` (0 count, 1
// materialize, 2 speculative count) for compilation (or a disk-cache load)
// on the background compiler, so they are ready before the plans' first
// iterations. wait != 0: block until every scheduled kernel is built.
// Returns the number of these plans that have a per-plan kernel ready.
int srdl_wcoj_jit_prepare(const srdl_plan *plans, uint32_t n, int mode, int wait) {
    if (g_mode.load() == 0 || !nvrtc().ok) return 0;
    std::vector<std::shared_ptr<Entry>> es;
    for (uint32_t i = 0; i < n; ++i) {
        auto e = entry_for(&plans[i], mode);
        es.push_back(e);
        std::lock_guard<std::mutex> lock(e->mu);
        if (e->state == 0) {
            e->state = 1;
            enqueue(e);
        }
    }
    if (wait) {
        std::unique_lock<std::mutex> lock(g_pool.mu);
        g_pool.idle.wait(lock, [] { return g_pool.queue.empty() && g_pool.busy == 0; });
    }
    int ready = 0;
    for (auto &e : es) {
        std::lock_guard<std::mutex> lock(e->mu);
        ready += e->state == 2 && e->kernel;
    }
    return ready;
}

// Block until the background compiler is idle.
void srdl_wcoj_jit_wait(void) {
    std::unique_lock<std::mutex> lock(g_pool.mu);
    g_pool.idle.wait(lock, [] { return g_pool.queue.empty() && g_pool.busy == 0; });
}

// Drop the kernels still queued for the background compiler and wait for
// the ones being compiled (process exit: no worker may outlive the CUDA
// runtime and NVRTC).
void srdl_wcoj_jit_shutdown(void) {
    std::unique_lock<std::mutex> lock(g_pool.mu);
    for (auto &e : g_pool.queue) {
        std::lock_guard<std::mutex> el(e->mu);
        e->state = 0;  // never built; a later request schedules it again
    }
    g_pool.queue.clear();
    g_pool.idle.wait(lock, [] { return g_pool.busy == 0; });
}

// Set the per-plan kernel mode (0 off, 1 background, 2 compile on first
// use); returns the previous mode. Default: SRDL_JIT (0 / async / sync).
int srdl_wcoj_jit_set_mode(int mode) { return g_mode.exchange(mode); }

// The generated source of the per-plan kernel (NUL-terminated, truncated to
// cap bytes); returns its full length. For inspection and tests.
uint64_t srdl_wcoj_jit_source(const srdl_plan *plan, int mode, char *buf, uint64_t cap) {
    const std::string src = shape_source(plan, mode);
    if (buf && cap) {
        const size_t k = src.size() < cap - 1 ? src.size() : (size_t)cap - 1;
        memcpy(buf, src.data(), k);
        buf[k] = 0;
    }
    return src.size();
}

// Compile the per-plan kernel with NVRTC without loading it (no GPU
// needed): 0 = compiled (cubin size in *cubin_bytes), 1 = compile error (the
// log in srdl_last_error), 2 = NVRTC unavailable.
int srdl_wcoj_jit_compile_check(const srdl_plan *plan, int mode, uint64_t *cubin_bytes) {
    if (!nvrtc().ok) return 2;
    std::string cubin, log;
    if (!compile_cubin(shape_source(plan, mode), &cubin, &log)) {
        set_error("%.480s", log.c_str());
        return 1;
    }
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return 0;
}

// [kernels compiled, disk-cache hits, failures, mode (0 when NVRTC is missing)]
void srdl_wcoj_jit_stats(uint64_t *out) {
    out[0] = g_compiled.load();
    out[1] = g_disk_hits.load();
    out[2] = g_failures.load();
    out[3] = nvrtc().ok ? (uint64_t)g_mode.load() : 0;
}

}  // extern "C"
