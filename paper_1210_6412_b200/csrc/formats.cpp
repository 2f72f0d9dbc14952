// formats.cpp -- multithreaded readers for the reference's text formats.
//
// mcreach/formats.py reads matrices ("matrix <n> <m>" + "<row> <col> <value>" lines), vectors
// ("vector <n>" + one value per line) and chains ("dtmc", "states", "initial", "goal" lines in
// any order + "<src> <dst> <prob>" lines) one Python line at a time. These readers take the
// same files, split them into per-thread chunks at line boundaries, parse every chunk in
// parallel and assemble the reference's result: csr_from_triplets order (rows, then columns
// ascending; explicit zeros dropped) and, for chains, validate()'s checks (probabilities in
// (0, 1], row sums within ROW_SUM_TOL summed in column order like matvec, start state in range).
//
// Values are parsed with strtod, which is correctly rounded, exactly like Python's float(); the
// accepted token grammar is the plain decimal subset of Python's int()/float() (optional sign,
// digits, optional fraction and exponent). Anything outside the well-formed subset -- a
// malformed or out-of-range token, a duplicate, a missing header, a failed check, inf/nan,
// underscores, a lone carriage return, a non-ASCII byte -- makes the reader return
// MCR_UNSUPPORTED_INPUT with the reason, and the caller defers to the reference's own reader,
// which raises its exact error (ParseError with the line number, RowSumError, ...).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "mcr.h"

namespace {

constexpr double ROW_SUM_TOL = 1e-9;  // markov.py:41

struct Entry {
    int64_t row, col;
    double val;
};

struct Header {  // dtmc keyword lines (may appear anywhere after the first line)
    int64_t line;
    int kind;    // 0 states, 1 initial, 2 goal
    std::vector<int64_t> ints;
};

struct Chunk {
    const char* b = nullptr;
    const char* e = nullptr;
    int64_t first_line = 1;
    std::vector<Entry> entries;
    std::vector<double> values;   // vector files
    std::vector<Header> headers;
    int64_t first_sig_line = -1;  // first significant line of the chunk
    std::vector<std::string> first_tokens;
    std::string why;              // non-empty: not in the fast subset
};

// str.split() / str.strip() whitespace for ASCII text (str.isspace)
inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\v' || c == '\f' || c == '\r' || (c >= 0x1c && c <= 0x1f);
}

bool parse_int(const char* b, const char* e, int64_t* out) {
    const char* p = b;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p == e) return false;
    uint64_t v = 0;
    for (; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        if (v > (uint64_t)INT64_MAX / 10) return false;
        v = v * 10 + (uint64_t)(*p - '0');
        if (v > (uint64_t)INT64_MAX) return false;
    }
    *out = neg ? -(int64_t)v : (int64_t)v;
    return true;
}

// Plain decimal subset of Python float(): [+-]? (d+ (. d*)? | . d+) ([eE] [+-]? d+)?
bool parse_float(const char* b, const char* e, double* out) {
    const char* p = b;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* m0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    bool digits = p > m0;
    if (p < e && *p == '.') {
        ++p;
        const char* f0 = p;
        while (p < e && *p >= '0' && *p <= '9') ++p;
        digits = digits || p > f0;
    }
    if (!digits) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        ++p;
        if (p < e && (*p == '+' || *p == '-')) ++p;
        const char* x0 = p;
        while (p < e && *p >= '0' && *p <= '9') ++p;
        if (p == x0) return false;
    }
    if (p != e) return false;
    char buf[128];
    const size_t len = (size_t)(e - b);
    if (len >= sizeof(buf)) {
        std::string s(b, e);
        *out = std::strtod(s.c_str(), nullptr);
    } else {
        std::memcpy(buf, b, len);
        buf[len] = 0;
        *out = std::strtod(buf, nullptr);
    }
    return true;
}

struct Tok {
    const char* b;
    const char* e;
    bool is(const char* w) const {
        const size_t n = std::strlen(w);
        return (size_t)(e - b) == n && std::memcmp(b, w, n) == 0;
    }
};

// kind: 0 matrix, 1 vector, 2 dtmc. The first significant line of the FILE is handled by the
// caller (its chunk records it in first_tokens and skips it).
void parse_chunk(Chunk& c, int kind, bool first_chunk) {
    const char* p = c.b;
    int64_t line = c.first_line;
    std::vector<Tok> t;
    bool seen_first = !first_chunk;
    while (p < c.e) {
        const char* nl = (const char*)std::memchr(p, '\n', (size_t)(c.e - p));
        const char* le = nl ? nl : c.e;
        const char* ce = (const char*)std::memchr(p, '#', (size_t)(le - p));
        if (!ce) ce = le;
        t.clear();
        for (const char* q = p; q < ce;) {
            while (q < ce && is_space(*q)) ++q;
            if (q >= ce) break;
            const char* s0 = q;
            while (q < ce && !is_space(*q)) ++q;
            t.push_back(Tok{s0, q});
        }
        if (!t.empty()) {
            if (!seen_first) {
                seen_first = true;
                c.first_sig_line = line;
                for (auto& k : t) c.first_tokens.emplace_back(k.b, k.e);
            } else if (kind == 1) {
                double v;
                if (t.size() != 1 || !parse_float(t[0].b, t[0].e, &v)) {
                    c.why = "line " + std::to_string(line) + ": not a plain value";
                    return;
                }
                c.values.push_back(v);
            } else if (kind == 2 && (t[0].is("states") || t[0].is("initial") || t[0].is("goal"))) {
                Header h;
                h.line = line;
                h.kind = t[0].is("states") ? 0 : t[0].is("initial") ? 1 : 2;
                for (size_t k = 1; k < t.size(); ++k) {
                    int64_t v;
                    if (!parse_int(t[k].b, t[k].e, &v)) {
                        c.why = "line " + std::to_string(line) + ": not a plain integer";
                        return;
                    }
                    h.ints.push_back(v);
                }
                c.headers.push_back(std::move(h));
            } else {
                Entry en;
                if (t.size() != 3 || !parse_int(t[0].b, t[0].e, &en.row) ||
                    !parse_int(t[1].b, t[1].e, &en.col) || !parse_float(t[2].b, t[2].e, &en.val)) {
                    c.why = "line " + std::to_string(line) + ": not '<int> <int> <value>'";
                    return;
                }
                c.entries.push_back(en);
            }
        }
        ++line;
        if (!nl) break;
        p = nl + 1;
    }
}

struct Parsed {
    std::vector<Chunk> chunks;
    std::string why;
    int64_t first_line = -1;
    std::vector<std::string> first;
};

int run_parse(const char* path, int kind, int threads, Parsed* P) {
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        P->why = std::string("cannot open ") + path;
        return MCR_UNSUPPORTED_INPUT;
    }
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::vector<char>* buf = new std::vector<char>((size_t)std::max<long>(size, 0));
    std::unique_ptr<std::vector<char>> own(buf);
    if (size > 0 && std::fread(buf->data(), 1, (size_t)size, f) != (size_t)size) {
        std::fclose(f);
        P->why = "read error";
        return MCR_UNSUPPORTED_INPUT;
    }
    std::fclose(f);
    const char* b = buf->data();
    const char* e = b + buf->size();
    // ASCII only; "\r\n" is a newline, a lone '\r' would be one for Python's universal newlines
    for (const char* q = b; q < e; ++q) {
        const unsigned char ch = (unsigned char)*q;
        if (ch >= 0x80 || ch == 0) {
            P->why = "non-ASCII or NUL byte";
            return MCR_UNSUPPORTED_INPUT;
        }
        if (ch == '\r' && (q + 1 == e || q[1] != '\n')) {
            P->why = "lone carriage return";
            return MCR_UNSUPPORTED_INPUT;
        }
    }
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    T = std::max(1, std::min(T, 64));
    if (buf->size() < (size_t)1 << 20) T = 1;
    // chunk boundaries just after a newline
    std::vector<const char*> cut{b};
    for (int k = 1; k < T; ++k) {
        const char* q = b + buf->size() * (size_t)k / (size_t)T;
        if (q <= cut.back()) continue;
        const char* nl = (const char*)std::memchr(q, '\n', (size_t)(e - q));
        if (!nl) break;
        cut.push_back(nl + 1);
    }
    cut.push_back(e);
    const size_t nc = cut.size() - 1;
    P->chunks.resize(nc);
    std::vector<int64_t> lines(nc, 0);
    {
        std::vector<std::thread> th;
        for (size_t k = 0; k < nc; ++k)
            th.emplace_back([&, k] {
                int64_t cnt = 0;
                for (const char* q = cut[k]; q < cut[k + 1]; ++q) cnt += *q == '\n';
                lines[k] = cnt;
            });
        for (auto& x : th) x.join();
    }
    int64_t ln = 1;
    for (size_t k = 0; k < nc; ++k) {
        P->chunks[k].b = cut[k];
        P->chunks[k].e = cut[k + 1];
        P->chunks[k].first_line = ln;
        ln += lines[k];
    }
    // the file's first significant line may lie in a later chunk if the early ones are blank
    size_t firstc = 0;
    {
        std::vector<std::thread> th;
        for (size_t k = 0; k < nc; ++k)
            th.emplace_back([&, k] { parse_chunk(P->chunks[k], kind, k == 0); });
        for (auto& x : th) x.join();
    }
    Chunk& c0 = P->chunks[firstc];
    if (c0.first_sig_line < 0) {
        // chunk 0 had no significant line: re-parse sequentially (rare: leading blank MBs)
        P->chunks.clear();
        Chunk all;
        all.b = b;
        all.e = e;
        all.first_line = 1;
        parse_chunk(all, kind, true);
        P->chunks.push_back(std::move(all));
    }
    for (auto& c : P->chunks)
        if (!c.why.empty()) {
            P->why = c.why;
            return MCR_UNSUPPORTED_INPUT;
        }
    if (P->chunks[0].first_sig_line < 0) {
        P->why = "empty file";
        return MCR_UNSUPPORTED_INPUT;
    }
    P->first_line = P->chunks[0].first_sig_line;
    P->first = P->chunks[0].first_tokens;
    return MCR_OK;
}

}  // namespace

struct mcr_text {
    int kind = 0;
    int64_t n = 0, m = 0, initial = -1;
    std::vector<int64_t> rstart, col, goals;
    std::vector<double> val;
};

namespace {

// csr_from_triplets (sparse.py:145-172): rows then columns ascending, duplicates rejected,
// explicit zeros dropped. Duplicates / out-of-range positions leave the fast path.
int assemble(std::vector<Chunk>& chunks, int64_t n, mcr_text* out, std::string* why) {
    size_t total = 0;
    for (auto& c : chunks) total += c.entries.size();
    std::vector<int64_t> cnt((size_t)n + 1, 0);
    for (auto& c : chunks)
        for (auto& en : c.entries) {
            if (en.row < 0 || en.row >= n || en.col < 0 || en.col >= n) {
                *why = "entry outside the dimension";
                return MCR_UNSUPPORTED_INPUT;
            }
            ++cnt[(size_t)en.row + 1];
        }
    for (int64_t i = 0; i < n; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    std::vector<std::pair<int64_t, double>> cv(total);
    for (auto& c : chunks) {
        for (auto& en : c.entries) cv[(size_t)pos[(size_t)en.row]++] = {en.col, en.val};
        std::vector<Entry>().swap(c.entries);
    }
    // sort every row by column (in parallel over row ranges); check duplicates
    const int T = std::max(1, std::min(64, (int)std::thread::hardware_concurrency()));
    std::atomic<int> dup{0};
    std::vector<std::thread> th;
    for (int k = 0; k < T; ++k)
        th.emplace_back([&, k] {
            const int64_t r0 = n * k / T, r1 = n * (k + 1) / T;
            for (int64_t i = r0; i < r1; ++i) {
                auto b = cv.begin() + cnt[(size_t)i], e = cv.begin() + cnt[(size_t)i + 1];
                std::sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
                for (auto q = b; q + 1 < e; ++q)
                    if (q->first == (q + 1)->first) dup = 1;
            }
        });
    for (auto& x : th) x.join();
    if (dup) {
        *why = "duplicate entry";
        return MCR_UNSUPPORTED_INPUT;
    }
    out->n = n;
    out->rstart.assign((size_t)n + 1, 0);
    out->col.reserve(total);
    out->val.reserve(total);
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t k = cnt[(size_t)i]; k < cnt[(size_t)i + 1]; ++k)
            if (cv[(size_t)k].second != 0.0) {
                out->col.push_back(cv[(size_t)k].first);
                out->val.push_back(cv[(size_t)k].second);
            }
        out->rstart[(size_t)i + 1] = (int64_t)out->col.size();
    }
    out->m = (int64_t)out->col.size();
    return MCR_OK;
}

thread_local std::string t_why;

int finish(int rc, const std::string& why, mcr_text* t, mcr_text** out) {
    if (rc != MCR_OK) {
        t_why = why;
        delete t;
        return rc;
    }
    *out = t;
    return MCR_OK;
}

}  // namespace

extern "C" {

MCR_API const char* mcr_text_reason(void) { return t_why.c_str(); }

MCR_API int mcr_read_matrix(const char* path, int threads, mcr_text** out) {
    if (!path || !out) return MCR_INVALID_ARGUMENT;
    *out = nullptr;
    Parsed P;
    mcr_text* t = new mcr_text();
    t->kind = 0;
    int rc = run_parse(path, 0, threads, &P);
    if (rc != MCR_OK) return finish(rc, P.why, t, out);
    int64_t n, m;
    if (P.first.size() != 3 || P.first[0] != "matrix" ||
        !parse_int(P.first[1].data(), P.first[1].data() + P.first[1].size(), &n) ||
        !parse_int(P.first[2].data(), P.first[2].data() + P.first[2].size(), &m) || n < 0)
        return finish(MCR_UNSUPPORTED_INPUT, "bad header", t, out);
    size_t total = 0;
    for (auto& c : P.chunks) total += c.entries.size();
    if ((int64_t)total != m) return finish(MCR_UNSUPPORTED_INPUT, "entry count differs from header", t, out);
    std::string why;
    rc = assemble(P.chunks, n, t, &why);
    return finish(rc, why, t, out);
}

MCR_API int mcr_read_vector(const char* path, int threads, mcr_text** out) {
    if (!path || !out) return MCR_INVALID_ARGUMENT;
    *out = nullptr;
    Parsed P;
    mcr_text* t = new mcr_text();
    t->kind = 1;
    int rc = run_parse(path, 1, threads, &P);
    if (rc != MCR_OK) return finish(rc, P.why, t, out);
    int64_t n;
    if (P.first.size() != 2 || P.first[0] != "vector" ||
        !parse_int(P.first[1].data(), P.first[1].data() + P.first[1].size(), &n) || n < 0)
        return finish(MCR_UNSUPPORTED_INPUT, "bad header", t, out);
    for (auto& c : P.chunks) t->val.insert(t->val.end(), c.values.begin(), c.values.end());
    if ((int64_t)t->val.size() != n) return finish(MCR_UNSUPPORTED_INPUT, "value count differs from header", t, out);
    t->n = n;
    return finish(MCR_OK, "", t, out);
}

MCR_API int mcr_read_dtmc(const char* path, int threads, mcr_text** out) {
    if (!path || !out) return MCR_INVALID_ARGUMENT;
    *out = nullptr;
    Parsed P;
    mcr_text* t = new mcr_text();
    t->kind = 2;
    int rc = run_parse(path, 2, threads, &P);
    if (rc != MCR_OK) return finish(rc, P.why, t, out);
    if (P.first.size() != 1 || P.first[0] != "dtmc") return finish(MCR_UNSUPPORTED_INPUT, "bad header", t, out);
    int64_t n = -1, initial = -1;
    int have[3] = {0, 0, 0};
    std::vector<int64_t> goals;
    for (auto& c : P.chunks)
        for (auto& h : c.headers) {
            if (have[h.kind]++) return finish(MCR_UNSUPPORTED_INPUT, "duplicate keyword line", t, out);
            if (h.kind == 0 && h.ints.size() == 1) n = h.ints[0];
            else if (h.kind == 1 && h.ints.size() == 1) initial = h.ints[0];
            else if (h.kind == 2 && !h.ints.empty()) goals = h.ints;
            else return finish(MCR_UNSUPPORTED_INPUT, "malformed keyword line", t, out);
        }
    if (!have[0] || !have[1] || !have[2]) return finish(MCR_UNSUPPORTED_INPUT, "missing keyword line", t, out);
    if (n < 1 || initial < 0 || initial >= n) return finish(MCR_UNSUPPORTED_INPUT, "states / initial out of range", t, out);
    for (int64_t g : goals)
        if (g < 0 || g >= n) return finish(MCR_UNSUPPORTED_INPUT, "goal state out of range", t, out);
    std::string why;
    rc = assemble(P.chunks, n, t, &why);
    if (rc != MCR_OK) return finish(rc, why, t, out);
    // validate() (markov.py:117-142) on the assembled chain
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = t->rstart[(size_t)i]; k < t->rstart[(size_t)i + 1]; ++k) {
            const double v = t->val[(size_t)k];
            if (!(v > 0.0 && v <= 1.0)) return finish(MCR_UNSUPPORTED_INPUT, "probability outside (0, 1]", t, out);
            s += v * 1.0;  // matvec(p, ones): row sum in column order
        }
        if (std::fabs(s - 1.0) > ROW_SUM_TOL) return finish(MCR_UNSUPPORTED_INPUT, "row sum off 1", t, out);
    }
    std::sort(goals.begin(), goals.end());
    goals.erase(std::unique(goals.begin(), goals.end()), goals.end());
    t->goals = goals;
    t->initial = initial;
    return finish(MCR_OK, "", t, out);
}

MCR_API int mcr_text_info(const mcr_text* t, int64_t* n, int64_t* m, int64_t* initial,
                          int64_t* ngoals) {
    if (!t) return MCR_INVALID_ARGUMENT;
    if (n) *n = t->n;
    if (m) *m = t->m;
    if (initial) *initial = t->initial;
    if (ngoals) *ngoals = (int64_t)t->goals.size();
    return MCR_OK;
}

MCR_API int mcr_text_export(const mcr_text* t, int64_t* rstart, int64_t* col, double* values,
                            int64_t* goals) {
    if (!t) return MCR_INVALID_ARGUMENT;
    if (rstart && !t->rstart.empty()) std::memcpy(rstart, t->rstart.data(), sizeof(int64_t) * t->rstart.size());
    if (col && !t->col.empty()) std::memcpy(col, t->col.data(), sizeof(int64_t) * t->col.size());
    if (values && !t->val.empty()) std::memcpy(values, t->val.data(), sizeof(double) * t->val.size());
    if (goals && !t->goals.empty()) std::memcpy(goals, t->goals.data(), sizeof(int64_t) * t->goals.size());
    return MCR_OK;
}

MCR_API void mcr_text_destroy(mcr_text* t) { delete t; }

}  // extern "C"
