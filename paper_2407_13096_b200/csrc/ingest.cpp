// ingest.cpp — host feature ingestion: PTX text -> per-kernel category counts,
// DCGM CSV -> per-metric means (reference proj/src/ptx_features.cpp:238-309,
// proj/src/telemetry.cpp:63-101).  Host C++ (no device code): these produce the
// count arrays / CSR entries and DCGM rows the device feature stage consumes
// (dso_featurize, dso_pipeline, dso_pipeline_csr).  Thread-safe and re-entrant:
// callers parse many files in parallel (the Python helper uses a thread pool;
// ctypes releases the GIL).
//
// Semantics follow the reference parser:
//   * comments (// and /* */) are removed first; an unterminated block comment
//     is MalformedPtx with its opening line;
//   * each ".entry" token (token-bounded) starts a kernel; its name is the next
//     token; a declaration ending in ';' before any '{' is a kernel with zero
//     counts; otherwise the balanced-brace body is split on ';' at any depth
//     and an unterminated body is MalformedPtx with the line of its '{';
//   * in a statement, scope braces, whole-line directives (a '.' token up to
//     the end of its line), labels ("name:") and a predicate guard ("@p" /
//     "@!p") are skipped; a statement whose first remaining character is '.',
//     a brace, or not a letter/underscore counts nothing; otherwise the opcode
//     token's root (up to the first '.') is counted in its instruction slot
//     (or "other"), and every '.'-suffix that is a canonical data type or state
//     space (or one of the known out-of-list ones, counted as "other") is
//     counted in that category.
#include <cctype>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/dso_b200.h"

namespace {

constexpr int kInstr = DSO_INSTR_SLOTS, kDtype = DSO_DTYPE_SLOTS, kMem = DSO_MEMSPACE_SLOTS;
constexpr int kStatusMalformed = 1, kStatusEmpty = 2, kStatusOutOfRange = 3, kStatusSchema = 4,
              kStatusInvalid = 12;

// Category lists (ptx_features.cpp:18-49), canonical order; "other" is the last slot.
const char* const kOps[kInstr - 1] = {
    "add", "addc", "sub", "subc", "mul", "mad", "madc", "mul24", "mad24", "sad", "div", "rem",
    "abs", "neg", "min", "max", "popc", "clz", "bfind", "fns", "brev", "bfe", "bfi", "szext",
    "bmsk", "dp4a", "dp2a", "testp", "copysign", "rcp", "sqrt", "rsqrt", "sin", "cos", "lg2",
    "ex2", "tanh", "fma", "set", "setp", "selp", "slct", "and", "or", "xor", "not", "cnot",
    "lop3", "shf", "shl", "shr", "mov", "shfl", "prmt", "ld", "ldu", "st", "prefetch",
    "prefetchu", "isspacep", "cvta", "cvt", "cp", "tex", "tld4", "txq", "suld", "sust", "sured",
    "suq", "istypep", "bra", "brx", "call", "ret", "exit", "bar", "barrier", "membar", "fence",
    "atom", "red", "vote", "match", "activemask", "redux", "griddepcontrol", "elect", "wmma",
    "mma", "ldmatrix", "stmatrix", "movmatrix", "mbarrier", "trap", "brkpt", "nanosleep",
    "pmevent", "vadd", "vmad"};
const char* const kTypes[kDtype - 1] = {".s8",  ".s16", ".s32", ".s64",  ".u8",  ".u16",
                                        ".u32", ".u64", ".f16", ".f16x2", ".f32", ".f64",
                                        ".b8",  ".b16", ".b32", ".b64"};
const char* const kSpaces[kMem - 1] = {".reg", ".sreg", ".const", ".global",
                                       ".local", ".param", ".shared"};
// in the ISA but outside the canonical lists -> the category's "other"
const char* const kTypesOther[] = {".pred", ".bf16", ".tf32", ".e4m3", ".e5m2", ".b128", ".s16x2"};
const char* const kSpacesOther[] = {".tex"};

template <size_t N>
int find(const char* const (&list)[N], std::string_view s) {
    for (size_t i = 0; i < N; ++i)
        if (s == list[i]) return (int)i;
    return -1;
}

bool tok(char c) {
    return std::isalnum((unsigned char)c) || c == '_' || c == '.' || c == '$' || c == '%';
}
bool space(char c) { return std::isspace((unsigned char)c) != 0; }

struct Kernel {
    std::string name;
    uint64_t counts[DSO_COUNT_ROWS] = {};  // instr | dtype | memspace slots
    uint64_t total = 0;
};

struct Fail {
    int status;
    std::string msg;
};

// Comment removal keeping newlines (line numbers stay valid).
std::string uncomment(std::string_view t) {
    std::string out;
    out.reserve(t.size());
    size_t line = 1;
    for (size_t i = 0; i < t.size();) {
        if (t[i] == '/' && i + 1 < t.size() && t[i + 1] == '/') {
            while (i < t.size() && t[i] != '\n') ++i;
        } else if (t[i] == '/' && i + 1 < t.size() && t[i + 1] == '*') {
            const size_t open = line;
            size_t end = t.find("*/", i + 2);
            if (end == std::string_view::npos)
                throw Fail{kStatusMalformed, "unterminated block comment starting at line " +
                                                 std::to_string(open)};
            for (size_t j = i; j < end; ++j)
                if (t[j] == '\n') {
                    out.push_back('\n');
                    ++line;
                }
            i = end + 2;
        } else {
            if (t[i] == '\n') ++line;
            out.push_back(t[i++]);
        }
    }
    return out;
}

void count(std::string_view st, Kernel& k) {
    size_t i = 0;
    auto ws = [&] {
        while (i < st.size() && space(st[i])) ++i;
    };
    ws();
    bool more = true;
    while (more) {
        more = false;
        while (i < st.size() && (st[i] == '{' || st[i] == '}')) {
            ++i;
            ws();
            more = true;
        }
        if (i < st.size() && st[i] == '.') {
            const size_t nl = st.find('\n', i);
            if (nl == std::string_view::npos) return;  // the statement is a directive
            i = nl + 1;
            ws();
            more = true;
        }
        size_t j = i;
        while (j < st.size() && tok(st[j])) ++j;
        if (j > i && j < st.size() && st[j] == ':') {
            i = j + 1;
            ws();
            more = true;
        }
    }
    if (i < st.size() && st[i] == '@') {
        ++i;
        if (i < st.size() && st[i] == '!') ++i;
        while (i < st.size() && tok(st[i])) ++i;
        ws();
    }
    if (i >= st.size()) return;
    const char c0 = st[i];
    if (!(std::isalpha((unsigned char)c0) || c0 == '_')) return;
    size_t e = i;
    while (e < st.size() && tok(st[e])) ++e;
    const std::string_view op = st.substr(i, e - i);
    size_t dot = op.find('.');
    const int slot = find(kOps, op.substr(0, dot));
    k.counts[slot >= 0 ? slot : kInstr - 1] += 1;
    k.total += 1;
    while (dot != std::string_view::npos) {
        const size_t nx = op.find('.', dot + 1);
        const std::string_view sfx =
            op.substr(dot, nx == std::string_view::npos ? std::string_view::npos : nx - dot);
        int s;
        if ((s = find(kTypes, sfx)) >= 0)
            k.counts[kInstr + s] += 1;
        else if ((s = find(kSpaces, sfx)) >= 0)
            k.counts[kInstr + kDtype + s] += 1;
        else if (find(kTypesOther, sfx) >= 0)
            k.counts[kInstr + kDtype - 1] += 1;
        else if (find(kSpacesOther, sfx) >= 0)
            k.counts[DSO_COUNT_ROWS - 1] += 1;
        dot = nx;
    }
}

std::string_view trim(std::string_view s) {
    size_t b = 0, e = s.size();
    while (b < e && space(s[b])) ++b;
    while (e > b && space(s[e - 1])) --e;
    return s.substr(b, e - b);
}

std::vector<Kernel> parse(std::string_view text) {
    const std::string code = uncomment(text);
    std::vector<Kernel> out;
    size_t pos = 0;
    auto line_of = [&](size_t p) {
        size_t n = 1;
        for (size_t q = 0; q < p; ++q) n += code[q] == '\n';
        return n;
    };
    while (true) {
        const size_t at = code.find(".entry", pos);
        if (at == std::string::npos) break;
        const size_t after = at + 6;
        const bool bounded = (after >= code.size() || !tok(code[after])) &&
                             (at == 0 || !tok(code[at - 1]));
        if (!bounded) {
            pos = at + 1;
            continue;
        }
        size_t p = after;
        Kernel k;
        while (p < code.size() && space(code[p])) ++p;
        const size_t ns = p;
        while (p < code.size() && tok(code[p])) ++p;
        k.name = code.substr(ns, p - ns);
        while (p < code.size() && code[p] != '{' && code[p] != ';') ++p;
        if (p >= code.size() || code[p] == ';') {  // declaration: zero counts
            out.push_back(std::move(k));
            pos = p < code.size() ? p + 1 : p;
            continue;
        }
        const size_t open = p;
        int depth = 0;
        size_t st = p + 1;
        do {
            const char ch = code[p];
            if (ch == '{') {
                ++depth;
            } else if (ch == '}') {
                --depth;
            } else if (ch == ';') {
                count(trim(std::string_view(code).substr(st, p - st)), k);
                st = p + 1;
            }
            ++p;
        } while (p < code.size() && depth > 0);
        if (depth != 0)
            throw Fail{kStatusMalformed,
                       "unterminated kernel body opened at line " + std::to_string(line_of(open))};
        out.push_back(std::move(k));
        pos = p;
    }
    return out;
}

void put_msg(char* msg, int32_t len, const std::string& s) {
    if (!msg || len <= 0) return;
    const size_t n = std::min<size_t>((size_t)len - 1, s.size());
    std::memcpy(msg, s.data(), n);
    msg[n] = '\0';
}

}  // namespace

struct dso_ptx {
    std::vector<Kernel> kernels;
};

extern "C" {

int32_t dso_ptx_parse(const char* text, int64_t len, dso_ptx** out, char* msg, int32_t msg_len) {
    if (!out || (!text && len > 0) || len < 0) return kStatusInvalid;
    *out = nullptr;
    try {
        dso_ptx* r = new dso_ptx;
        r->kernels = parse(std::string_view(text ? text : "", (size_t)len));
        *out = r;
        put_msg(msg, msg_len, "");
        return 0;
    } catch (const Fail& f) {
        put_msg(msg, msg_len, f.msg);
        return f.status;
    }
}

void dso_ptx_free(dso_ptx* p) { delete p; }

int64_t dso_ptx_kernel_count(const dso_ptx* p) { return p ? (int64_t)p->kernels.size() : 0; }

const char* dso_ptx_kernel_name(const dso_ptx* p, int64_t k) {
    if (!p || k < 0 || k >= (int64_t)p->kernels.size()) return nullptr;
    return p->kernels[k].name.c_str();
}

int32_t dso_ptx_kernel_counts(const dso_ptx* p, int64_t k, uint64_t* counts126,
                              uint64_t* total_instructions) {
    if (!p || k < 0 || k >= (int64_t)p->kernels.size() || !counts126) return kStatusInvalid;
    std::memcpy(counts126, p->kernels[k].counts, sizeof(uint64_t) * DSO_COUNT_ROWS);
    if (total_instructions) *total_instructions = p->kernels[k].total;
    return 0;
}

int32_t dso_ptx_counts(const dso_ptx* p, uint32_t* counts, int64_t ld) {
    if (!p || !counts || ld < (int64_t)p->kernels.size()) return kStatusInvalid;
    const int64_t n = (int64_t)p->kernels.size();
    for (int64_t k = 0; k < n; ++k)
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const uint64_t c = p->kernels[k].counts[r];
            if (c > 0xFFFFFFFFull) return kStatusInvalid;
            counts[(int64_t)r * ld + k] = (uint32_t)c;
        }
    return 0;
}

int64_t dso_ptx_nnz(const dso_ptx* p) {
    if (!p) return 0;
    int64_t nnz = 0;
    for (const Kernel& k : p->kernels)
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) nnz += k.counts[r] != 0;
    return nnz;
}

int32_t dso_ptx_csr(const dso_ptx* p, uint64_t* row_ptr, uint32_t* entries) {
    if (!p || !row_ptr) return kStatusInvalid;
    uint64_t e = 0;
    row_ptr[0] = 0;
    for (size_t k = 0; k < p->kernels.size(); ++k) {
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const uint64_t c = p->kernels[k].counts[r];
            if (!c) continue;
            if (c >= (1ull << 25)) return kStatusInvalid;  // CSR entry limit (count << 7)
            if (entries) entries[e] = (uint32_t)(c << 7) | (uint32_t)r;
            ++e;
        }
        row_ptr[k + 1] = e;
    }
    return 0;
}

// Canonical category name of count row r (instruction_categories /
// data_type_categories / memory_space_categories, ptx_features.hpp:39-41): rows
// 0..100, 101..117, 118..125; the last of each list is "other".
const char* dso_category_name(int32_t row) {
    if (row < 0 || row >= kInstr + kDtype + kMem) return nullptr;
    if (row < kInstr) return row < kInstr - 1 ? kOps[row] : "other";
    row -= kInstr;
    if (row < kDtype) return row < kDtype - 1 ? kTypes[row] : "other";
    row -= kDtype;
    return row < kMem - 1 ? kSpaces[row] : "other";
}

// load_dcgm_samples (telemetry.cpp:63-101): header check, >= 1 data row, 9 fields
// per row, every metric in [0, 1], per-metric mean in double (row order).
int32_t dso_load_dcgm_csv(const char* text, int64_t len, double* mean8, char* msg,
                          int32_t msg_len) {
    static const std::string_view kHeader =
        "timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC";
    if (!mean8 || (!text && len > 0) || len < 0) return kStatusInvalid;
    const std::string_view t(text ? text : "", (size_t)len);
    std::vector<std::string_view> lines;
    for (size_t p = 0; p < t.size();) {
        size_t nl = t.find('\n', p);
        std::string_view l = t.substr(p, nl == std::string_view::npos ? std::string_view::npos : nl - p);
        if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
        if (!l.empty()) lines.push_back(l);
        if (nl == std::string_view::npos) break;
        p = nl + 1;
    }
    auto strip = [](std::string_view s) {
        while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
        while (!s.empty() && (s.back() == ' ' || s.back() == '\t')) s.remove_suffix(1);
        return s;
    };
    if (lines.empty() || strip(lines[0]) != kHeader) {
        put_msg(msg, msg_len, "expected header '" + std::string(kHeader) + "'");
        return kStatusSchema;
    }
    if (lines.size() < 2) {
        put_msg(msg, msg_len, "no data rows");
        return kStatusEmpty;
    }
    double sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t r = 1; r < lines.size(); ++r) {
        std::vector<std::string_view> f;
        for (size_t p = 0;;) {
            const size_t c = lines[r].find(',', p);
            f.push_back(lines[r].substr(p, c == std::string_view::npos ? std::string_view::npos : c - p));
            if (c == std::string_view::npos) break;
            p = c + 1;
        }
        if (f.size() != 9) {
            put_msg(msg, msg_len, "row " + std::to_string(r) + ": expected 9 fields, got " +
                                      std::to_string(f.size()));
            return kStatusSchema;
        }
        for (int m = 0; m < 8; ++m) {
            const std::string_view s = strip(f[m + 1]);
            std::string buf(s);
            char* end = nullptr;
            const double v = buf.empty() ? 0.0 : std::strtod(buf.c_str(), &end);
            // from_chars semantics: the whole field must be a number (no leading '+', no hex)
            if (buf.empty() || end != buf.c_str() + buf.size() || buf[0] == '+' ||
                buf.find_first_of("xXpP") != std::string::npos || std::isspace((unsigned char)buf[0])) {
                put_msg(msg, msg_len, "row " + std::to_string(r) + ": not a number: '" + buf + "'");
                return kStatusSchema;
            }
            if (v < 0.0 || v > 1.0) {
                put_msg(msg, msg_len, "row " + std::to_string(r) + ": metric value " +
                                          std::to_string(v) + " outside [0, 1]");
                return kStatusOutOfRange;
            }
            sum[m] += v;
        }
    }
    for (int m = 0; m < 8; ++m) mean8[m] = sum[m] / (double)(lines.size() - 1);
    put_msg(msg, msg_len, "");
    return 0;
}

}  // extern "C"
