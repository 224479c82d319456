// Multi-core C++ restatement of the oracle's generic join + semi-naive
// fixpoint (checker / CPU baseline only; TEST INFRASTRUCTURE — the engine
// never links or calls this).
//
// It evaluates exactly what oracle/gj.py evaluates — same rule grouping,
// same per-instance variable order and per-atom column orders, same
// semi-naive protocol — so both are pinned by the same golden fixtures
// (tests/test_oracle_golden.py runs the reference's 154 fixpoints through
// both). The algorithm follows the reference:
//   * generic join, one variable at a time over relations sorted under a
//     per-atom column order: candidates from the positive source with the
//     smallest narrowed range, every source narrowed by binary search,
//     negated atoms probed when their last variable binds
//     (reference pkg/src/flatlog/executor.py:342-431 _root_setup/_descend,
//     pkg/src/flatlog/storage.py:113-216 narrow/intersections);
//   * stratified semi-naive loop: delta := full on entry of a recursive
//     stratum, each round joins every instance with one delta atom,
//     delta := dedup(new) - full, full |= delta, stop on an empty delta
//     (reference pkg/src/flatlog/runtime.py:259-315, storage.py:311-324).
// Differences are in the mechanics only: the first join level is cut into
// chunks that OpenMP threads walk depth-first (outputs concatenated in
// chunk order, so the emitted sequence is deterministic), sorted indexes of
// full relations are cached per column order and kept up to date by merging
// each delta in (O(n) per round instead of a re-sort), and sort / merge /
// difference run on packed fixed-width keys.
//
// Program encoding (int32 words, built by oracle/native.py):
//   nrel, arity[nrel], ncomp,
//   per component: recursive, nheads, heads[nheads], ninst, instances...
//   instance: head_rel, head_arity, (kind, value) x head_arity  [kind 0 =
//     variable level, 1 = constant id], depth, natoms, atoms...
//   atom: rel, version (0 full, 1 delta), negated, arity, perm[arity],
//     nconst, const_id[nconst] (-1 = unknown constant), nbound,
//     level[nbound] (levels of the bound columns nconst.., nondecreasing)
#include <omp.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <parallel/algorithm>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using Rows = std::vector<uint32_t>;  // row-major, `arity` words per row (join output)
using u128 = unsigned __int128;

thread_local std::string g_error;

struct Row8 {  // key for arity 5..8 (32 bytes)
    uint32_t c[8];
    bool operator<(const Row8 &o) const {
        for (int k = 0; k < 8; ++k)
            if (c[k] != o.c[k]) return c[k] < o.c[k];
        return false;
    }
    bool operator==(const Row8 &o) const { return memcmp(c, o.c, sizeof(c)) == 0; }
};

// Packed row keys, column 0 most significant: numeric order of the keys is
// the lexicographic order of the rows. kind 0: u64 (arity <= 2), 1: u128
// (arity <= 4), 2: Row8.
inline int kind_of(int arity) { return arity <= 2 ? 0 : arity <= 4 ? 1 : 2; }
inline size_t words_of(int kind) { return kind == 0 ? 1 : kind == 1 ? 2 : 4; }

template <class K>
inline K pack(const uint32_t *r, int arity) {
    K k = 0;
    for (int c = 0; c < arity; ++c) k = (k << 32) | r[c];
    return k;
}
template <>
inline Row8 pack<Row8>(const uint32_t *r, int arity) {
    Row8 k{};
    for (int c = 0; c < arity; ++c) k.c[c] = r[c];
    return k;
}
template <class K>
inline uint32_t col_of(const K &k, int arity, int c) {
    return (uint32_t)(k >> (32 * (arity - 1 - c)));
}
template <>
inline uint32_t col_of<Row8>(const Row8 &k, int, int c) {
    return k.c[c];
}

template <class F>
auto dispatch(int kind, F &&f) {
    if (kind == 0) return f(uint64_t{});
    if (kind == 1) return f(u128{});
    return f(Row8{});
}

// A sorted, distinct set of packed rows.
struct KeyVec {
    int arity = 1;
    std::vector<uint64_t> buf;  // words_of(kind) words per row
    size_t n = 0;
    int kind() const { return kind_of(arity); }
    template <class K>
    const K *as() const {
        return reinterpret_cast<const K *>(buf.data());
    }
    template <class K>
    K *as() {
        return reinterpret_cast<K *>(buf.data());
    }
    void resize(size_t rows) {
        n = rows;
        buf.resize(rows * words_of(kind()));
    }
    uint32_t at(size_t r, int c) const {
        switch (kind()) {
            case 0: return col_of(as<uint64_t>()[r], arity, c);
            case 1: return col_of(as<u128>()[r], arity, c);
            default: return as<Row8>()[r].c[c];
        }
    }
};

template <class K>
bool sorted_strict(const K *k, size_t n) {
    bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (size_t i = 1; i < n; ++i) ok = ok && (k[i - 1] < k[i]);
    return ok;
}

// row-major rows (maybe unsorted / duplicated), columns taken in `perm`
// order -> sorted distinct keys
KeyVec build(const uint32_t *rows, size_t n, int arity, const int *perm) {
    KeyVec out;
    out.arity = arity;
    out.resize(n);
    dispatch(out.kind(), [&](auto tag) {
        using K = decltype(tag);
        K *k = out.as<K>();
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < n; ++i) {
            uint32_t tmp[8];
            const uint32_t *r = rows + i * (size_t)arity;
            for (int c = 0; c < arity; ++c) tmp[c] = r[perm ? perm[c] : c];
            k[i] = pack<K>(tmp, arity);
        }
        if (!sorted_strict(k, n)) {
            __gnu_parallel::sort(k, k + n);
            out.resize(std::unique(k, k + n) - k);
        }
        return 0;
    });
    return out;
}

// rows of a set, row-major (columns in the set's order)
Rows unpack_rows(const KeyVec &a) {
    Rows out(a.n * (size_t)a.arity);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < a.n; ++i)
        for (int c = 0; c < a.arity; ++c) out[i * a.arity + c] = a.at(i, c);
    return out;
}

// the same set under another column order
KeyVec reindex(const KeyVec &a, const int *perm) {
    const Rows rows = unpack_rows(a);
    return build(rows.data(), a.n, a.arity, perm);
}

// a \ b: per chunk of a, a galloping walk through b from the chunk's first
// position (O(|a| log(|b| / |a|)) comparisons)
KeyVec difference(const KeyVec &a, const KeyVec &b) {
    if (a.n == 0 || b.n == 0) return a;
    return dispatch(a.kind(), [&](auto tag) {
        using K = decltype(tag);
        const K *ka = a.as<K>(), *kb = b.as<K>();
        std::vector<uint8_t> keep(a.n);
        const size_t chunk = 1 << 14;
        const size_t nch = (a.n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 1)
        for (size_t q = 0; q < nch; ++q) {
            const size_t lo = q * chunk, hi = std::min(a.n, lo + chunk);
            size_t pos = std::lower_bound(kb, kb + b.n, ka[lo]) - kb;
            for (size_t i = lo; i < hi; ++i) {
                size_t step = 1, end = pos;
                while (end < b.n && kb[end] < ka[i]) {  // gallop
                    pos = end + 1;
                    end = pos + step;
                    step <<= 1;
                }
                end = std::min(end, b.n);
                pos = std::lower_bound(kb + pos, kb + end, ka[i]) - kb;
                keep[i] = !(pos < b.n && kb[pos] == ka[i]);
            }
        }
        KeyVec out;
        out.arity = a.arity;
        out.resize(a.n);
        K *ko = out.as<K>();
        size_t m = 0;
        for (size_t i = 0; i < a.n; ++i)
            if (keep[i]) ko[m++] = ka[i];
        out.resize(m);
        return out;
    });
}

// sorted union of disjoint sets
KeyVec merge(const KeyVec &a, const KeyVec &b) {
    if (b.n == 0) return a;
    if (a.n == 0) return b;
    return dispatch(a.kind(), [&](auto tag) {
        using K = decltype(tag);
        KeyVec out;
        out.arity = a.arity;
        out.resize(a.n + b.n);
        K *pa = const_cast<K *>(a.as<K>()), *pb = const_cast<K *>(b.as<K>());  // libstdc++ wants mutable
        __gnu_parallel::merge(pa, pa + a.n, pb, pb + b.n, out.as<K>());
        return out;
    });
}

// ------------------------------------------------------------------ program

struct AtomSpec {
    int rel, version, negated, arity;
    std::vector<int> perm;
    std::vector<int64_t> consts;  // -1: unknown constant
    std::vector<int> levels;      // level of bound column nconst + i
};

struct Instance {
    int head_rel, head_arity;
    std::vector<std::pair<int, int64_t>> head;  // (kind, value)
    int depth;
    std::vector<AtomSpec> atoms;
};

struct Component {
    bool recursive;
    std::vector<int> heads;
    std::vector<Instance> inst;
};

struct Relation {
    int arity = 0;
    Rows loaded;                                // EDB rows before the first solve (row-major)
    KeyVec full;                                // sorted, identity order
    KeyVec delta;                               // sorted, identity order
    std::map<std::vector<int>, KeyVec> fcache;  // full sorted under perm
    std::map<std::vector<int>, KeyVec> dcache;  // delta sorted under perm
    size_t n() const { return full.n; }
};

struct Engine {
    std::vector<Relation> rel;
    std::vector<Component> comp;
    std::vector<int> rounds;
    std::vector<uint32_t> level0_keep;  // optional sorted filter on level-0 values
    int chunks_per_thread = 64;
};

struct Reader {
    const int32_t *p, *end;
    int32_t next() {
        if (p >= end) throw std::runtime_error("program encoding truncated");
        return *p++;
    }
};

// ------------------------------------------------------------------ join

struct Src {
    const KeyVec *d;
    int arity;
    bool neg;
    int maxlvl;
    std::vector<std::vector<int>> cols;  // per level: columns bound there
};

inline size_t lower_col(const KeyVec *d, int, int c, size_t lo, size_t hi, uint32_t v) {
    while (lo < hi) {
        size_t mid = lo + ((hi - lo) >> 1);
        if (d->at(mid, c) < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
inline size_t upper_col(const KeyVec *d, int, int c, size_t lo, size_t hi, uint32_t v) {
    while (lo < hi) {
        size_t mid = lo + ((hi - lo) >> 1);
        if (d->at(mid, c) <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

struct Walker {
    const Instance *I;
    const std::vector<Src> *S;
    std::vector<std::vector<int>> specs;  // per level: atoms with columns there
    std::vector<std::vector<int>> cands;  // per level: positive ones
    const std::vector<uint32_t> *keep0;
    std::vector<uint32_t> vals;
    std::vector<size_t> lo, hi;  // [level][atom] flattened
    int na;
    Rows *out;

    void emit() {
        for (int k = 0; k < I->head_arity; ++k) {
            const auto &h = I->head[k];
            out->push_back(h.first == 0 ? vals[h.second] : (uint32_t)h.second);
        }
    }

    // narrow atom a at level L with value v from the ranges of level L into
    // level L+1; false when a positive source empties / a negated one matches
    bool narrow_all(int L, uint32_t v) {
        size_t *l0 = &lo[(size_t)L * na], *h0 = &hi[(size_t)L * na];
        size_t *l1 = &lo[(size_t)(L + 1) * na], *h1 = &hi[(size_t)(L + 1) * na];
        for (int a = 0; a < na; ++a) {
            l1[a] = l0[a];
            h1[a] = h0[a];
        }
        for (int a : specs[L]) {
            const Src &s = (*S)[a];
            size_t x = l1[a], y = h1[a];
            for (int c : s.cols[L]) {
                if (x >= y) break;
                size_t nx = lower_col(s.d, s.arity, c, x, y, v);
                y = upper_col(s.d, s.arity, c, nx, y, v);
                x = nx;
            }
            if (x > y) y = x;
            l1[a] = x;
            h1[a] = y;
            if (!s.neg) {
                if (x >= y) return false;
            } else if (s.maxlvl == L && x < y) {
                return false;
            }
        }
        return true;
    }

    int driver(int L) const {
        int best = -1;
        size_t bl = 0;
        for (int a : cands[L]) {
            size_t len = hi[(size_t)L * na + a] - lo[(size_t)L * na + a];
            if (best < 0 || len < bl) {
                best = a;
                bl = len;
            }
        }
        return best;
    }

    void walk(int L) {
        if (L == I->depth) {
            emit();
            return;
        }
        const int a = driver(L);
        const Src &s = (*S)[a];
        const int c = s.cols[L][0];
        size_t r = lo[(size_t)L * na + a];
        const size_t e = hi[(size_t)L * na + a];
        while (r < e) {
            const uint32_t v = s.d->at(r, c);
            const size_t next = upper_col(s.d, s.arity, c, r, e, v);
            vals[L] = v;
            if (narrow_all(L, v)) walk(L + 1);
            r = next;
        }
    }

    // level 0 restricted to driver rows [r, e)
    void walk_root(size_t r, size_t e) {
        const int a = driver(0);
        const Src &s = (*S)[a];
        const int c = s.cols[0][0];
        while (r < e) {
            const uint32_t v = s.d->at(r, c);
            const size_t next = upper_col(s.d, s.arity, c, r, e, v);
            vals[0] = v;
            bool ok = !keep0 || keep0->empty() || std::binary_search(keep0->begin(), keep0->end(), v);
            if (ok && narrow_all(0, v)) walk(1);
            r = next;
        }
    }
};

bool is_identity(const std::vector<int> &perm) {
    for (int c = 0; c < (int)perm.size(); ++c)
        if (perm[c] != c) return false;
    return true;
}

// the relation version sorted under `perm` (identity: the relation itself)
const KeyVec &index_of(Relation &R, int version, const std::vector<int> &perm) {
    if (is_identity(perm)) return version == 0 ? R.full : R.delta;
    auto &cache = version == 0 ? R.fcache : R.dcache;
    auto it = cache.find(perm);
    if (it != cache.end()) return it->second;
    KeyVec sorted = reindex(version == 0 ? R.full : R.delta, perm.data());
    return cache.emplace(perm, std::move(sorted)).first->second;
}

// All head tuples (with duplicates) of one instance.
Rows join(Engine &E, const Instance &I) {
    const int na = (int)I.atoms.size();
    std::vector<Src> S(na);
    std::vector<size_t> lo0(na), hi0(na);
    for (int a = 0; a < na; ++a) {
        const AtomSpec &A = I.atoms[a];
        Relation &R = E.rel[A.rel];
        const KeyVec &rows = index_of(R, A.version, A.perm);
        Src &s = S[a];
        s.d = &rows;
        s.arity = A.arity;
        s.neg = A.negated != 0;
        s.cols.assign(I.depth + 1, {});
        s.maxlvl = -1;
        const int nc = (int)A.consts.size();
        for (int i = 0; i < (int)A.levels.size(); ++i) {
            s.cols[A.levels[i]].push_back(nc + i);
            s.maxlvl = std::max(s.maxlvl, A.levels[i]);
        }
        size_t lo = 0, hi = rows.n;
        for (int c = 0; c < nc && lo < hi; ++c) {
            if (A.consts[c] < 0) {
                lo = hi = 0;
                break;
            }
            const uint32_t v = (uint32_t)A.consts[c];
            size_t x = lower_col(s.d, s.arity, c, lo, hi, v);
            hi = upper_col(s.d, s.arity, c, x, hi, v);
            lo = x;
        }
        lo0[a] = lo;
        hi0[a] = hi;
        if (!s.neg && lo >= hi) return {};
        if (s.neg && A.levels.empty() && lo < hi) return {};
    }
    Walker proto;
    proto.I = &I;
    proto.S = &S;
    proto.na = na;
    proto.keep0 = &E.level0_keep;
    proto.specs.assign(I.depth + 1, {});
    proto.cands.assign(I.depth + 1, {});
    for (int L = 0; L < I.depth; ++L)
        for (int a = 0; a < na; ++a)
            if (!S[a].cols[L].empty()) {
                proto.specs[L].push_back(a);
                if (!S[a].neg) proto.cands[L].push_back(a);
            }
    proto.vals.assign(I.depth + 1, 0);
    proto.lo.assign((size_t)(I.depth + 1) * na, 0);
    proto.hi.assign((size_t)(I.depth + 1) * na, 0);
    for (int a = 0; a < na; ++a) {
        proto.lo[a] = lo0[a];
        proto.hi[a] = hi0[a];
    }
    Rows out;
    if (I.depth == 0) {
        proto.out = &out;
        proto.emit();
        return out;
    }
    // level-0 driver rows cut into chunks at value boundaries
    const int a0 = proto.driver(0);
    const Src &s0 = S[a0];
    const int c0 = s0.cols[0][0];
    const size_t r0 = lo0[a0], e0 = hi0[a0];
    const int threads = omp_get_max_threads();
    const size_t want = (size_t)threads * E.chunks_per_thread;
    std::vector<size_t> cuts{r0};
    const size_t step = std::max<size_t>(1, (e0 - r0) / std::max<size_t>(want, 1));
    for (size_t r = r0 + step; r < e0; r += step) {
        const uint32_t v = s0.d->at(r - 1, c0);
        const size_t b = upper_col(s0.d, s0.arity, c0, r - 1, e0, v);
        if (b > cuts.back() && b < e0) cuts.push_back(b);
    }
    cuts.push_back(e0);
    const size_t nchunks = cuts.size() - 1;
    std::vector<Rows> parts(nchunks);
#pragma omp parallel
    {
        Walker w = proto;
#pragma omp for schedule(dynamic, 1)
        for (size_t k = 0; k < nchunks; ++k) {
            w.out = &parts[k];
            w.walk_root(cuts[k], cuts[k + 1]);
        }
    }
    size_t total = 0;
    for (auto &p : parts) total += p.size();
    out.reserve(total);
    for (auto &p : parts) {
        out.insert(out.end(), p.begin(), p.end());
        Rows().swap(p);
    }
    return out;
}

void set_full(Relation &R, KeyVec rows) {
    R.full = std::move(rows);
    R.fcache.clear();
}

// full |= fresh (disjoint, sorted): every cached index gets the fresh rows
// merged in under its order
void add_fresh(Relation &R, const KeyVec &fresh) {
    for (auto &kv : R.fcache) kv.second = merge(kv.second, reindex(fresh, kv.first.data()));
    R.full = merge(R.full, fresh);
}

void set_delta(Relation &R, KeyVec rows) {
    R.delta = std::move(rows);
    R.dcache.clear();
}

KeyVec from_rows(const Rows &rows, int arity) { return build(rows.data(), rows.size() / arity, arity, nullptr); }

void solve(Engine &E) {
    for (auto &R : E.rel) {
        KeyVec k = from_rows(R.loaded, R.arity);
        Rows().swap(R.loaded);
        set_full(R, std::move(k));
        set_delta(R, KeyVec{R.arity, {}, 0});
    }
    E.rounds.clear();
    for (auto &C : E.comp) {
        if (!C.recursive) {
            for (auto &I : C.inst) {
                Relation &H = E.rel[I.head_rel];
                KeyVec got = from_rows(join(E, I), H.arity);
                set_full(H, merge(H.full, difference(got, H.full)));
            }
            E.rounds.push_back(1);
            continue;
        }
        for (int h : C.heads) set_delta(E.rel[h], E.rel[h].full);
        int rounds = 0;
        while (true) {
            ++rounds;
            std::map<int, Rows> staged;
            for (int h : C.heads) staged[h];
            for (auto &I : C.inst) {
                Rows got = join(E, I);
                Rows &dst = staged[I.head_rel];
                if (dst.empty())
                    dst.swap(got);
                else
                    dst.insert(dst.end(), got.begin(), got.end());
            }
            std::map<int, KeyVec> fresh;
            bool empty = true;
            for (int h : C.heads) {
                Relation &H = E.rel[h];
                KeyVec f = difference(from_rows(staged[h], H.arity), H.full);
                Rows().swap(staged[h]);
                empty = empty && f.n == 0;
                fresh[h] = std::move(f);
            }
            if (empty) break;
            for (int h : C.heads) add_fresh(E.rel[h], fresh[h]);
            for (int h : C.heads) set_delta(E.rel[h], std::move(fresh[h]));
        }
        for (int h : C.heads) set_delta(E.rel[h], KeyVec{E.rel[h].arity, {}, 0});
        E.rounds.push_back(rounds);
    }
}

Engine *decode(const int32_t *prog, size_t len) {
    Reader rd{prog, prog + len};
    auto *E = new Engine();
    const int nrel = rd.next();
    E->rel.resize(nrel);
    for (int r = 0; r < nrel; ++r) {
        E->rel[r].arity = rd.next();
        if (E->rel[r].arity < 1 || E->rel[r].arity > 8) throw std::runtime_error("arity outside [1, 8]");
    }
    const int ncomp = rd.next();
    E->comp.resize(ncomp);
    for (auto &C : E->comp) {
        C.recursive = rd.next() != 0;
        C.heads.resize(rd.next());
        for (int &h : C.heads) h = rd.next();
        C.inst.resize(rd.next());
        for (auto &I : C.inst) {
            I.head_rel = rd.next();
            I.head_arity = rd.next();
            for (int k = 0; k < I.head_arity; ++k) {
                const int kind = rd.next();
                const int32_t lo = rd.next(), hi = rd.next();
                I.head.emplace_back(kind, ((int64_t)(uint32_t)hi << 32) | (uint32_t)lo);
            }
            I.depth = rd.next();
            I.atoms.resize(rd.next());
            for (auto &A : I.atoms) {
                A.rel = rd.next();
                A.version = rd.next();
                A.negated = rd.next();
                A.arity = rd.next();
                A.perm.resize(A.arity);
                for (int &p : A.perm) p = rd.next();
                A.consts.resize(rd.next());
                for (auto &c : A.consts) {
                    const int32_t lo = rd.next(), hi = rd.next();
                    c = hi < 0 ? -1 : (((int64_t)(uint32_t)hi << 32) | (uint32_t)lo);
                }
                A.levels.resize(rd.next());
                for (int &l : A.levels) l = rd.next();
            }
        }
    }
    return E;
}

template <class F>
int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_error = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char *og_error() { return g_error.c_str(); }

void *og_new(const int32_t *prog, uint64_t len) {
    Engine *E = nullptr;
    if (guarded([&] { E = decode(prog, len); })) return nullptr;
    return E;
}

void og_free(void *h) { delete (Engine *)h; }

int og_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}

int og_load(void *h, int rel, const uint32_t *rows, uint64_t n) {
    return guarded([&] {
        Engine *E = (Engine *)h;
        Relation &R = E->rel.at(rel);
        R.loaded.insert(R.loaded.end(), rows, rows + n * (uint64_t)R.arity);
    });
}

int og_keep_level0(void *h, const uint32_t *keys, uint64_t n) {
    return guarded([&] {
        Engine *E = (Engine *)h;
        E->level0_keep.assign(keys, keys + n);
        std::sort(E->level0_keep.begin(), E->level0_keep.end());
    });
}

int og_solve(void *h) {
    return guarded([&] { solve(*(Engine *)h); });
}

uint64_t og_size(void *h, int rel) { return ((Engine *)h)->rel.at(rel).n(); }

int og_rows(void *h, int rel, uint32_t *out) {
    return guarded([&] {
        const Rows r = unpack_rows(((Engine *)h)->rel.at(rel).full);
        memcpy(out, r.data(), r.size() * sizeof(uint32_t));
    });
}

int og_ncomp(void *h) { return (int)((Engine *)h)->rounds.size(); }
int og_rounds(void *h, int comp) { return ((Engine *)h)->rounds.at(comp); }

}  // extern "C"
