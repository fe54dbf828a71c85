// moesim_gpu — the reference CLI's trace / profiling / placement / simulation
// commands (moesim, cli.cpp:446-567) as a C++ host program over the B200
// C-ABI (include/occult.h): same options, output files, stdout lines and exit
// codes (2 usage, 3 data, 4 placement / capacity, 1 other).
//
//   moesim_gpu gen-trace  --experts E --topk K --tokens N --seed S --out F [--dist uniform|zipf|blocks ...]
//   moesim_gpu profile    --trace F --out-prefix P
//   moesim_gpu reschedule --graph F --devices D --out F
//   moesim_gpu simulate   --seed S --out F [--trace F] [--placement F] [--prune none|router|similarity] ...
//   moesim_gpu sweep-prune --seed S --mode router|similarity --out-prefix P ...
//
// Text formats follow io.cpp:55-204 with std::to_chars / std::from_chars, as
// the reference does, so files round-trip byte for byte.  Placement is host
// code in libocc; the co-activation histogram, fp64 router, top-k, pruning and
// the expert-parallel forward are CUDA kernels behind the C-ABI.  Trace
// generation, the RNG streams and the component-growth statistic are
// test-input tooling outside the layer (moesim_tools.hpp).  Pinned to the
// reference in tests/test_cli.py / tests/test_gpu_cli.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "moesim_tools.hpp"
#include "occult.h"

namespace {

// ------------------------------------------------------------------ errors --
struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PlacementError : std::runtime_error { using std::runtime_error::runtime_error; };

void occ_ok(occ_status s, const char* what) {
    if (s == OCC_OK) return;
    const std::string msg = std::string(what) + ": " + occ_last_error();
    if (s == OCC_ERR_CONFIG) throw UsageError(occ_last_error());
    if (s == OCC_ERR_PLACEMENT) throw PlacementError(occ_last_error());
    if (s == OCC_ERR_CAPACITY) throw CapacityError(occ_last_error());
    throw std::runtime_error(msg);
}
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct Dev {  // owning device buffer
    T* p = nullptr;
    explicit Dev(size_t n) { cuda_ok(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    void put(const T* h, size_t n) { cuda_ok(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
    void get(T* h, size_t n) const { cuda_ok(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }
};

uint16_t to_bf16(double v) {  // round to nearest even through float
    const float f = static_cast<float>(v);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
double from_bf16(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// ----------------------------------------------------------------- formats --
std::string fmt(double v) {  // format_double (io.cpp:55-60)
    if (!std::isfinite(v)) throw DataError("refusing to serialize non-finite value");
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

std::vector<std::string> split_ws(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream ss(line);
    std::string t;
    while (ss >> t) out.push_back(t);
    return out;
}

[[noreturn]] void bad(int line_no, const std::string& what) {
    throw DataError("line " + std::to_string(line_no) + ": " + what);
}

long long parse_int(const std::string& s, int line_no) {
    long long v = 0;
    const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) bad(line_no, "expected integer, got '" + s + "'");
    return v;
}
double parse_double(const std::string& s, int line_no) {
    double v = 0.0;
    const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) bad(line_no, "expected number, got '" + s + "'");
    return v;
}

std::string expect_header(std::istream& is, const char* header, int& line_no) {
    std::string line;
    if (!std::getline(is, line)) throw DataError("line 1: empty input");
    ++line_no;
    if (line != header) bad(line_no, std::string("expected header '") + header + "'");
    if (!std::getline(is, line)) bad(line_no + 1, "missing header fields");
    ++line_no;
    return line;
}

struct Trace {
    int ne = 0, k = 0, n = 0;
    std::string tag;
    std::vector<int32_t> ids;
    std::vector<double> w;
};

std::string write_trace(const Trace& t) {
    std::ostringstream os;
    os << "#moesim-trace v1\n" << "experts=" << t.ne << " topk=" << t.k << " tokens=" << t.n;
    if (!t.tag.empty()) os << " tag=" << t.tag;
    os << "\n";
    for (int i = 0; i < t.n; ++i) {
        for (int j = 0; j < t.k; ++j) os << (j ? " " : "") << t.ids[(size_t)i * t.k + j];
        for (int j = 0; j < t.k; ++j) os << ' ' << fmt(t.w[(size_t)i * t.k + j]);
        os << "\n";
    }
    return os.str();
}

Trace read_trace(const std::string& text) {
    std::istringstream is(text);
    int line_no = 0;
    const std::string fields = expect_header(is, "#moesim-trace v1", line_no);
    Trace t;
    int tokens = -1;
    for (const auto& f : split_ws(fields)) {
        const auto eq = f.find('=');
        if (eq == std::string::npos) bad(line_no, "malformed header field '" + f + "'");
        const std::string key = f.substr(0, eq), val = f.substr(eq + 1);
        if (key == "experts") t.ne = static_cast<int>(parse_int(val, line_no));
        else if (key == "topk") t.k = static_cast<int>(parse_int(val, line_no));
        else if (key == "tokens") tokens = static_cast<int>(parse_int(val, line_no));
        else if (key == "tag") t.tag = val;
        else bad(line_no, "unknown header field '" + key + "'");
    }
    if (t.ne < 1 || t.k < 1 || tokens < 0) bad(line_no, "incomplete trace header");
    std::string line;
    int seen = 0;
    while (std::getline(is, line)) {
        ++line_no;
        if (line.empty()) continue;
        const auto parts = split_ws(line);
        if ((int)parts.size() != 2 * t.k)
            bad(line_no, "record needs " + std::to_string(2 * t.k) + " fields, got " + std::to_string(parts.size()));
        for (int j = 0; j < t.k; ++j) {
            const long long id = parse_int(parts[j], line_no);
            if (id < 0 || id >= t.ne) bad(line_no, "expert id out of range");
            t.ids.push_back(static_cast<int32_t>(id));
        }
        for (int j = 0; j < t.k; ++j) t.w.push_back(parse_double(parts[t.k + j], line_no));
        ++seen;
    }
    if (seen != tokens)
        throw DataError("trace declares " + std::to_string(tokens) + " tokens but has " + std::to_string(seen) +
                        " records");
    t.n = tokens;
    for (int i = 0; i < t.n; ++i)  // RoutingOutcome::validate (routing.cpp:11-31)
        for (int j = 0; j < t.k; ++j) {
            const int32_t e = t.ids[(size_t)i * t.k + j];
            if (t.w[(size_t)i * t.k + j] <= 0.0)
                throw DataError("trace file: routing: non-positive weight at token " + std::to_string(i));
            for (int l = 0; l < j; ++l)
                if (t.ids[(size_t)i * t.k + l] == e)
                    throw DataError("trace file: routing: duplicate expert id at token " + std::to_string(i));
        }
    return t;
}

struct Mat {
    int rows = 0, cols = 0;
    std::vector<double> v;
};
std::string write_matrix(const Mat& m) {
    std::ostringstream os;
    os << "#moesim-matrix v1\n" << m.rows << ' ' << m.cols << "\n";
    for (int i = 0; i < m.rows; ++i) {
        for (int j = 0; j < m.cols; ++j) os << (j ? " " : "") << fmt(m.v[(size_t)i * m.cols + j]);
        os << "\n";
    }
    return os.str();
}
Mat read_matrix(const std::string& text) {
    std::istringstream is(text);
    int line_no = 0;
    const auto shape = split_ws(expect_header(is, "#moesim-matrix v1", line_no));
    if (shape.size() != 2) bad(line_no, "expected 'rows cols'");
    Mat m;
    m.rows = static_cast<int>(parse_int(shape[0], line_no));
    m.cols = static_cast<int>(parse_int(shape[1], line_no));
    if (m.rows < 0 || m.cols < 0) bad(line_no, "negative matrix shape");
    m.v.assign((size_t)m.rows * m.cols, 0.0);
    std::string line;
    for (int i = 0; i < m.rows; ++i) {
        if (!std::getline(is, line)) bad(line_no + 1, "missing matrix row");
        ++line_no;
        const auto parts = split_ws(line);
        if ((int)parts.size() != m.cols) bad(line_no, "wrong column count");
        for (int j = 0; j < m.cols; ++j) m.v[(size_t)i * m.cols + j] = parse_double(parts[j], line_no);
    }
    return m;
}

using Devices = std::vector<std::vector<int>>;
void validate_placement(const Devices& d, int expected) {  // placement.cpp:17-45
    if (d.empty()) throw PlacementError("placement: no devices");
    int n = 0;
    for (const auto& x : d) n += (int)x.size();
    if (expected >= 0 && n != expected)
        throw PlacementError("placement: covers " + std::to_string(n) + " experts, expected " +
                             std::to_string(expected));
    if (n % (int)d.size()) throw PlacementError("placement: uneven device lists");
    for (const auto& x : d)
        if ((int)x.size() != n / (int)d.size()) throw PlacementError("placement: uneven device lists");
    std::vector<char> seen(n, 0);
    for (const auto& x : d)
        for (int e : x) {
            if (e < 0 || e >= n || seen[e])
                throw PlacementError("placement: device lists are not a partition of [0, " + std::to_string(n) + ")");
            seen[e] = 1;
        }
}
std::string write_placement(const Devices& d) {
    std::ostringstream os;
    os << "#moesim-placement v1\n" << "devices=" << d.size() << "\n";
    for (const auto& x : d) {
        for (size_t i = 0; i < x.size(); ++i) os << (i ? " " : "") << x[i];
        os << "\n";
    }
    return os.str();
}
Devices read_placement(const std::string& text) {
    std::istringstream is(text);
    int line_no = 0;
    const auto parts = split_ws(expect_header(is, "#moesim-placement v1", line_no));
    if (parts.size() != 1 || parts[0].rfind("devices=", 0) != 0) bad(line_no, "expected 'devices=N'");
    const int nd = static_cast<int>(parse_int(parts[0].substr(8), line_no));
    Devices d;
    std::string line;
    for (int i = 0; i < nd; ++i) {
        if (!std::getline(is, line)) bad(line_no + 1, "missing device list");
        ++line_no;
        std::vector<int> ex;
        for (const auto& tok : split_ws(line)) ex.push_back(static_cast<int>(parse_int(tok, line_no)));
        d.push_back(std::move(ex));
    }
    try {
        validate_placement(d, -1);
    } catch (const PlacementError& e) {
        throw DataError(std::string("placement file: ") + e.what());
    }
    return d;
}

std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw DataError("cannot open '" + path + "'");
    std::ostringstream ss;
    ss << f.rdbuf();
    return ss.str();
}
void write_file(const std::string& path, const std::string& s) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw DataError("cannot write '" + path + "'");
    f << s;
}

struct Report {  // ReportWriter (io.cpp:206-213)
    std::ostringstream os;
    Report() { os << "#moesim-report v1\n"; }
    void kv(const std::string& k, const std::string& v) { os << k << '=' << v << "\n"; }
    void kv(const std::string& k, double v) { kv(k, fmt(v)); }
    void kv(const std::string& k, long long v) { kv(k, std::to_string(v)); }
    void kv(const std::string& k, int v) { kv(k, std::to_string(v)); }
};

// ------------------------------------------------------------ arguments ----
struct Args {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;
    std::string get(const std::string& k, const std::string& dflt) const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : it->second;
    }
    std::string need(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end()) throw UsageError(k + " is required");
        return it->second;
    }
    long long num(const std::string& k, long long dflt) const {
        auto it = kv.find(k);
        if (it == kv.end()) return dflt;
        long long v = 0;
        const auto& s = it->second;
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw UsageError(k + ": expected an integer");
        return v;
    }
    double real(const std::string& k, double dflt) const {
        auto it = kv.find(k);
        if (it == kv.end()) return dflt;
        double v = 0;
        const auto& s = it->second;
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw UsageError(k + ": expected a number");
        return v;
    }
};

Args parse_args(const std::vector<std::string>& a, const std::vector<std::string>& options,
                const std::vector<std::string>& flag_names) {
    Args out;
    for (size_t i = 0; i < a.size(); ++i) {
        std::string key = a[i], val;
        const auto eq = key.find('=');
        if (eq != std::string::npos) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        }
        if (std::find(flag_names.begin(), flag_names.end(), key) != flag_names.end()) {
            out.flags[key] = true;
            continue;
        }
        if (std::find(options.begin(), options.end(), key) == options.end())
            throw UsageError("unknown option '" + key + "'");
        if (eq == std::string::npos) {
            if (i + 1 >= a.size()) throw UsageError(key + " needs a value");
            val = a[++i];
        }
        out.kv[key] = val;
    }
    return out;
}

// ------------------------------------------------------------- commands ----
int cmd_gen_trace(const std::vector<std::string>& a) {  // cli.cpp:92-110
    const Args o = parse_args(a, {"--dist", "--experts", "--topk", "--tokens", "--alpha", "--blocks", "--p-in",
                                  "--tag", "--seed", "--out"}, {});
    const std::string dist = o.get("--dist", "uniform");
    tools::TraceSpec spec{};
    if (dist == "uniform") spec.dist = tools::kUniform;
    else if (dist == "zipf") spec.dist = tools::kZipf;
    else if (dist == "blocks") spec.dist = tools::kBlocks;
    else throw UsageError("unknown distribution '" + dist + "'");
    spec.num_experts = (int)std::stoll(o.need("--experts"));
    spec.top_k = (int)std::stoll(o.need("--topk"));
    spec.num_tokens = (int)std::stoll(o.need("--tokens"));
    spec.alpha = o.real("--alpha", 1.0);
    spec.num_blocks = (int)o.num("--blocks", 1);
    spec.p_in = o.real("--p-in", 0.9);
    const uint64_t seed = std::stoull(o.need("--seed"));
    const std::string out = o.need("--out");
    Trace t;
    t.ne = spec.num_experts, t.k = spec.top_k, t.n = spec.num_tokens, t.tag = o.get("--tag", "");
    const size_t nk = (size_t)std::max(t.n, 0) * std::max(t.k, 0);
    t.ids.resize(nk);
    t.w.resize(nk);
    const std::string bad = tools::gen_trace(&spec, seed, t.ids.data(), t.w.data());
    if (!bad.empty()) throw UsageError(bad);
    write_file(out, write_trace(t));
    return 0;
}

int cmd_profile(const std::vector<std::string>& a, std::ostream& out) {  // cli.cpp:112-171
    const Args o = parse_args(a, {"--trace", "--out-prefix"}, {});
    const Trace t = read_trace(slurp(o.need("--trace")));
    const std::string prefix = o.need("--out-prefix");
    const int ne = t.ne, n = t.n, batch = 256;
    Dev<int32_t> ids((size_t)n * t.k);
    ids.put(t.ids.data(), (size_t)n * t.k);
    Dev<int64_t> counts((size_t)ne * ne);
    cuda_ok(cudaMemset(counts.p, 0, sizeof(int64_t) * ne * ne), "memset");
    occ_ok(occ_coactivation_histogram(ids.p, n, t.k, ne, counts.p, nullptr), "histogram");
    std::vector<int64_t> hc((size_t)ne * ne);
    counts.get(hc.data(), hc.size());
    // ComponentTracker (collab.cpp:120-169) over 256-token batches: host statistic
    const std::vector<int32_t> hf = tools::first_batch_of(t.ids.data(), n, t.k, ne, batch);
    const int nb = (n + batch - 1) / batch;
    std::vector<int32_t> largest(std::max(nb, 1));
    tools::component_growth(hf.data(), ne, nb, largest.data());
    Mat cm{ne, ne, std::vector<double>(hc.begin(), hc.end())};
    Mat nm{ne, ne, std::vector<double>((size_t)ne * ne)};
    occ_ok(occ_normalize_graph(hc.data(), ne, nm.v.data()), "normalize_graph");
    write_file(prefix + ".collab.mat", write_matrix(cm));
    write_file(prefix + ".norm.mat", write_matrix(nm));
    long long edges = 0, coact = 0;
    for (int i = 0; i < ne; ++i)
        for (int j = i + 1; j < ne; ++j) {
            edges += hc[(size_t)i * ne + j] > 0;
            coact += hc[(size_t)i * ne + j];
        }
    const int maxc = nb ? largest[nb - 1] : 0;
    Report r;
    r.kv("command", std::string("profile"));
    r.kv("trace.experts", ne);
    r.kv("trace.topk", t.k);
    r.kv("trace.tokens", n);
    if (!t.tag.empty()) r.kv("trace.tag", t.tag);
    r.kv("graph.edges", edges);
    r.kv("graph.coactivations", coact);
    r.kv("graph.max_component", (long long)maxc);
    r.kv("growth.0", 0);
    for (int b = 0; b < nb; ++b) r.kv("growth." + std::to_string(std::min(n, (b + 1) * batch)), largest[b]);
    write_file(prefix + ".profile.txt", r.os.str());
    out << "profile: " << n << " tokens, " << edges << " edges, max component " << maxc << "\n";
    return 0;
}

int cmd_reschedule(const std::vector<std::string>& a) {  // cli.cpp:173-188
    const Args o = parse_args(a, {"--graph", "--devices", "--out"}, {});
    const Mat m = read_matrix(slurp(o.need("--graph")));
    const int nd = (int)std::stoll(o.need("--devices"));
    const std::string out = o.need("--out");
    if (nd < 1 || m.rows % std::max(nd, 1) != 0)
        throw UsageError("reschedule: expert count " + std::to_string(m.rows) + " is not divisible by --devices " +
                         std::to_string(nd));
    // norm_graph_from_matrix (cli.cpp:62-80)
    if (m.rows != m.cols) throw DataError("graph: matrix must be square");
    double mx = 0.0;
    for (int i = 0; i < m.rows; ++i)
        for (int j = 0; j < m.cols; ++j) {
            const double v = m.v[(size_t)i * m.cols + j];
            if (v < 0.0) throw DataError("graph: negative edge value");
            if (v != m.v[(size_t)j * m.cols + i]) throw DataError("graph: matrix must be symmetric");
            if (i == j && v != 0.0) throw DataError("graph: diagonal must be zero");
            mx = std::max(mx, v);
        }
    std::vector<double> p(m.v.size(), 0.0);
    if (mx != 0.0)
        for (size_t i = 0; i < p.size(); ++i) p[i] = m.v[i] / mx;
    std::vector<int32_t> flat(m.rows);
    occ_ok(occ_reschedule_placement(p.data(), m.rows, nd, flat.data()), "reschedule_placement");
    const int per = m.rows / nd;
    Devices d(nd);
    for (int i = 0; i < nd; ++i) d[i].assign(flat.begin() + i * per, flat.begin() + (i + 1) * per);
    write_file(out, write_placement(d));
    return 0;
}

struct SimOpts {
    uint64_t seed = 0;
    int devices = 1, experts = 8, topk = 2, tokens = 64, dim = 32, hidden = 64, budget = 1, bps = 4;
    int tile_m = 32, tile_k = 32, tile_n = 32;
    std::string trace, placement, prune = "none", table, dump_table, weight_policy = "inherit", precision = "single";
    std::string activation = "identity", source_mode = "roundrobin", out;
    bool renormalize = true, check_oracle = false;
};

SimOpts sim_opts(const Args& o) {
    SimOpts s;
    s.seed = std::stoull(o.need("--seed"));
    s.devices = (int)o.num("--devices", 1);
    s.experts = (int)o.num("--experts", 8);
    s.topk = (int)o.num("--topk", 2);
    s.tokens = (int)o.num("--tokens", 64);
    s.dim = (int)o.num("--dim", 32);
    s.hidden = (int)o.num("--hidden", 64);
    s.trace = o.get("--trace", "");
    s.placement = o.get("--placement", "");
    s.prune = o.get("--prune", "none");
    s.budget = (int)o.num("--budget", 1);
    s.table = o.get("--table", "");
    s.dump_table = o.get("--dump-table", "");
    s.weight_policy = o.get("--weight-policy", "inherit");
    s.check_oracle = o.flags.count("--check-oracle") > 0;
    s.bps = (int)o.num("--bytes-per-scalar", 4);
    s.precision = o.get("--precision", "single");
    if (o.flags.count("--no-renormalize")) s.renormalize = false;
    s.activation = o.get("--activation", "identity");
    s.source_mode = o.get("--source-mode", "roundrobin");
    s.tile_m = (int)o.num("--tile-m", 32);
    s.tile_k = (int)o.num("--tile-k", 32);
    s.tile_n = (int)o.num("--tile-n", 32);
    s.out = o.get("--out", "");
    return s;
}

const std::vector<std::string> kSimOptions = {
    "--seed", "--devices", "--experts", "--topk", "--tokens", "--dim", "--hidden", "--trace", "--placement",
    "--prune", "--budget", "--table", "--dump-table", "--weight-policy", "--bytes-per-scalar", "--precision",
    "--activation", "--source-mode", "--tile-m", "--tile-k", "--tile-n", "--out", "--mode", "--out-prefix"};
const std::vector<std::string> kSimFlags = {"--check-oracle", "--renormalize", "--no-renormalize"};

struct SimResult {
    int ne = 0, k = 0, n = 0;
    Devices devices;
    occ_comm_report rep{};
    std::vector<int64_t> counts;
    double oracle_err = -1.0;
};

SimResult run_simulate(const SimOpts& o) {  // cli.cpp:201-320
    if (o.precision != "single" && o.precision != "double") throw UsageError("unknown precision '" + o.precision + "'");
    int act;
    if (o.activation == "identity") act = OCC_ACT_IDENTITY;
    else if (o.activation == "silu") act = OCC_ACT_SILU;
    else if (o.activation == "relu") act = OCC_ACT_RELU;
    else throw UsageError("unknown activation '" + o.activation + "'");
    int pmode;
    if (o.prune == "none") pmode = OCC_PRUNE_NONE;
    else if (o.prune == "router") pmode = OCC_PRUNE_ROUTER;
    else if (o.prune == "similarity") pmode = OCC_PRUNE_SIMILARITY;
    else throw UsageError("unknown prune mode '" + o.prune + "'");
    if (o.weight_policy != "inherit" && o.weight_policy != "own")
        throw UsageError("unknown weight policy '" + o.weight_policy + "'");
    Trace tr;
    const bool trace_mode = !o.trace.empty();
    int ne = o.experts, k = o.topk;
    if (trace_mode) {
        if (pmode != OCC_PRUNE_NONE) throw UsageError("pruning needs gate scores; drop --trace to simulate from a seed");
        tr = read_trace(slurp(o.trace));
        ne = tr.ne, k = tr.k;
    }
    const int nd = o.devices;
    if (ne < 1) throw UsageError("config: num_experts must be >= 1");
    if (nd < 1) throw UsageError("config: num_devices must be >= 1");
    if (k < 1 || k > ne)
        throw UsageError("config: top_k must satisfy 1 <= k <= num_experts (k=" + std::to_string(k) +
                         ", experts=" + std::to_string(ne) + ")");
    if (ne % nd)
        throw UsageError("config: num_experts (" + std::to_string(ne) + ") must be divisible by num_devices (" +
                         std::to_string(nd) + ")");
    if (o.dim < 1 || o.hidden < 1) throw UsageError("config: dims must be >= 1");
    if (o.tile_m < 1 || o.tile_k < 1 || o.tile_n < 1) throw UsageError("config: tile sizes must be >= 1");
    SimResult R;
    R.ne = ne, R.k = k;
    if (!o.placement.empty()) {
        R.devices = read_placement(slurp(o.placement));
        validate_placement(R.devices, ne);
    } else {
        R.devices.assign(nd, {});
        for (int d = 0; d < nd; ++d)
            for (int i = 0; i < ne / nd; ++i) R.devices[d].push_back(d * (ne / nd) + i);
    }
    if ((int)R.devices.size() != nd) throw PlacementError("placement: device count differs from --devices");
    const int single = o.precision == "single";
    tools::Rng master(o.seed);  // cli.cpp:248-251: token, gate, expert streams in that order
    tools::Rng trng(master.g()), grng(master.g()), erng(master.g());
    const int n = trace_mode ? tr.n : o.tokens, D = o.dim, F = o.hidden;
    R.n = n;
    std::vector<double> x((size_t)n * D), w1((size_t)ne * D * F), w2((size_t)ne * F * D), g((size_t)ne * D);
    tools::rng_matrix(&trng, n, D, single, x.data());
    for (int e = 0; e < ne; ++e) {  // ExpertWeights::random (core.cpp:40-52)
        tools::rng_matrix(&erng, D, F, single, w1.data() + (size_t)e * D * F);
        tools::rng_matrix(&erng, F, D, single, w2.data() + (size_t)e * F * D);
    }
    if (o.source_mode != "single" && o.source_mode != "roundrobin")
        throw UsageError("unknown source mode '" + o.source_mode + "'");
    // the layer on the device
    occ_config cfg{ne, k, nd, D, F, o.renormalize ? 1 : 0, act, 1};
    std::vector<int32_t> flat;
    for (const auto& dv : R.devices) flat.insert(flat.end(), dv.begin(), dv.end());
    occ_handle* h = nullptr;
    occ_ok(occ_create(&cfg, flat.data(), 1, 0, &h), "create");
    struct Free {
        occ_handle* h;
        ~Free() { occ_destroy(h); }
    } guard{h};
    std::vector<uint16_t> b1(w1.size()), b2(w2.size()), bx(x.size());
    for (size_t i = 0; i < w1.size(); ++i) b1[i] = to_bf16(w1[i]);
    for (size_t i = 0; i < w2.size(); ++i) b2[i] = to_bf16(w2[i]);
    for (size_t i = 0; i < x.size(); ++i) bx[i] = to_bf16(x[i]);
    Dev<uint16_t> d1(b1.size()), d2(b2.size()), dxb(bx.size()), dout(bx.size());
    d1.put(b1.data(), b1.size());
    d2.put(b2.data(), b2.size());
    dxb.put(bx.data(), bx.size());
    occ_ok(occ_load_experts(h, d1.p, nullptr, d2.p, nullptr), "load_experts");
    Dev<int32_t> ids((size_t)n * k);
    std::vector<double> wh((size_t)n * k);
    double cap = -1.0;
    if (trace_mode) {
        ids.put(tr.ids.data(), tr.ids.size());
        wh = tr.w;
    } else {
        tools::rng_matrix(&grng, ne, D, single, g.data());
        Dev<double> dx(x.size()), dg(g.size()), sc((size_t)n * ne), dw((size_t)n * k);
        dx.put(x.data(), x.size());
        dg.put(g.data(), g.size());
        occ_ok(occ_gate_scores_f64(dx.p, n, D, dg.p, ne, sc.p, nullptr), "gate_scores");
        occ_ok(occ_topk_route_f64(sc.p, n, ne, k, o.renormalize ? 1 : 0, ids.p, dw.p, nullptr), "topk_route");
        std::vector<double> table;
        if (pmode == OCC_PRUNE_SIMILARITY) {
            if (!o.table.empty()) {
                const Mat tm = read_matrix(slurp(o.table));
                if (tm.rows != ne || tm.cols != ne) throw DataError("similarity table shape mismatch");
                table = tm.v;
            } else {  // profile the batch's own router logits (cli.cpp:296-299)
                Dev<double> lg((size_t)n * ne), inner((size_t)ne * ne);
                occ_ok(occ_gate_logits_f64(dx.p, n, D, dg.p, ne, lg.p, nullptr), "gate_logits");
                cuda_ok(cudaMemset(inner.p, 0, sizeof(double) * ne * ne), "memset");
                occ_ok(occ_similarity_accumulate(lg.p, 1, n, ne, inner.p, nullptr), "similarity_accumulate");
                std::vector<double> hi((size_t)ne * ne);
                inner.get(hi.data(), hi.size());
                table.resize(hi.size());
                occ_ok(occ_similarity_finalize(hi.data(), n, ne, table.data()), "similarity_finalize");
            }
            if (!o.dump_table.empty()) write_file(o.dump_table, write_matrix(Mat{ne, ne, table}));
        }
        if (pmode != OCC_PRUNE_NONE) {
            if (o.budget < 1 || o.budget > nd) throw UsageError("prune: device budget must be in [1, num_devices]");
            if (pmode == OCC_PRUNE_SIMILARITY) occ_ok(occ_set_similarity(h, table.data()), "set_similarity");
            occ_prune pr{pmode, o.budget, o.weight_policy == "own" ? 1 : 0};
            Dev<int32_t> ids2((size_t)n * k);
            Dev<double> w2d((size_t)n * k);
            occ_ok(occ_prune_routing_f64(h, sc.p, ids.p, dw.p, n, &pr, ids2.p, w2d.p, nullptr), "prune_routing");
            cuda_ok(cudaMemcpy(ids.p, ids2.p, sizeof(int32_t) * n * k, cudaMemcpyDeviceToDevice), "copy");
            w2d.get(wh.data(), wh.size());
            cap = std::min({(double)k, (double)nd, (double)o.budget});
        } else {
            dw.get(wh.data(), wh.size());
        }
    }
    std::vector<float> wf(wh.begin(), wh.end());
    Dev<float> dwf(wf.size());
    dwf.put(wf.data(), wf.size());
    std::vector<int32_t> src;
    Dev<int32_t> dsrc(std::max(n, 1));
    if (o.source_mode == "single") {
        src.assign(n, 0);
        dsrc.put(src.data(), src.size());
    }
    occ_ok(occ_forward(h, dxb.p, ids.p, dwf.p, o.source_mode == "single" ? dsrc.p : nullptr, n, dout.p, nullptr),
           "forward");
    occ_ok(occ_comm_report_get(h, o.bps, &R.rep, nullptr), "comm_report");
    if (cap >= 0.0) R.rep.cap_replicas = cap;
    Dev<int64_t> counts((size_t)ne * ne);
    cuda_ok(cudaMemset(counts.p, 0, sizeof(int64_t) * ne * ne), "memset");
    occ_ok(occ_coactivation_histogram(ids.p, n, k, ne, counts.p, nullptr), "histogram");
    R.counts.resize((size_t)ne * ne);
    counts.get(R.counts.data(), R.counts.size());
    if (o.check_oracle) {  // max_rel_error (matrix.cpp:52-62) against a dense fp64 evaluation of the routing
        std::vector<uint16_t> ob(bx.size());
        dout.get(ob.data(), ob.size());
        std::vector<int32_t> hid((size_t)n * k);
        ids.get(hid.data(), hid.size());
        double diff = 0.0, ref = 0.0;
        std::vector<double> hrow(F), yrow(D);
        for (int t = 0; t < n; ++t) {
            std::fill(yrow.begin(), yrow.end(), 0.0);
            for (int j = 0; j < k; ++j) {
                const int e = hid[(size_t)t * k + j];
                for (int f = 0; f < F; ++f) {
                    double s = 0.0;
                    for (int c = 0; c < D; ++c) s += x[(size_t)t * D + c] * w1[((size_t)e * D + c) * F + f];
                    hrow[f] = act == OCC_ACT_SILU ? s / (1.0 + std::exp(-s)) : act == OCC_ACT_RELU ? std::max(s, 0.0) : s;
                }
                for (int c = 0; c < D; ++c) {
                    double s = 0.0;
                    for (int f = 0; f < F; ++f) s += hrow[f] * w2[((size_t)e * F + f) * D + c];
                    yrow[c] += wh[(size_t)t * k + j] * s;
                }
            }
            for (int c = 0; c < D; ++c) {
                diff = std::max(diff, std::fabs(from_bf16(ob[(size_t)t * D + c]) - yrow[c]));
                ref = std::max(ref, std::fabs(yrow[c]));
            }
        }
        R.oracle_err = ref > 0.0 ? diff / ref : diff;
    }
    return R;
}

void write_simulate_report(const SimOpts& o, const SimResult& R) {  // cli.cpp:326-378
    const int nd = (int)R.devices.size(), ne = R.ne, k = R.k;
    Report r;
    r.kv("command", std::string("simulate"));
    r.kv("config.devices", nd);
    r.kv("config.experts", ne);
    r.kv("config.topk", k);
    r.kv("config.tokens", R.n);
    r.kv("config.dim", o.dim);
    r.kv("config.hidden", o.hidden);
    r.kv("config.seed", (long long)o.seed);
    r.kv("config.precision", o.precision);
    r.kv("config.activation", o.activation);
    r.kv("config.renormalize", o.renormalize ? 1 : 0);
    r.kv("config.prune.mode", o.prune);
    if (o.prune != "none") r.kv("config.prune.budget", o.budget);
    r.kv("config.trace", o.trace.empty() ? std::string("-") : o.trace);
    r.kv("config.placement", o.placement.empty() ? std::string("trivial") : o.placement);
    r.kv("replicas.mean", R.rep.mean_replicas);
    r.kv("replicas.cap", R.rep.cap_replicas);
    r.kv("replicas.lower_bound", (double)((k * nd + ne - 1) / ne));  // collab.cpp:63-74
    r.kv("replicas.upper_bound", (double)std::min(k, nd));
    r.kv("replicas.baseline_k", R.n ? (double)k : 0.0);  // simnet.cpp:26-34
    r.kv("shares.intra", R.rep.intra_share);
    r.kv("shares.inter", R.rep.inter_share);
    r.kv("bytes.cross_device", R.rep.cross_device_bytes);
    r.kv("bytes.per_scalar", o.bps);
    long long total = 0;
    for (int d = 0; d < nd; ++d) {
        r.kv("device." + std::to_string(d) + ".received", R.rep.per_device_rows[d]);
        total += R.rep.per_device_rows[d];
    }
    r.kv("tokens.sfd_total", total);
    std::vector<double> p((size_t)ne * ne);
    occ_ok(occ_normalize_graph(R.counts.data(), ne, p.data()), "normalize_graph");
    for (int d = 0; d < nd; ++d) {  // collab.cpp:76-103, same summation order
        const auto& ex = R.devices[d];
        const int m = (int)ex.size();
        double s = 0.0;
        if (m >= 2)
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b)
                    if (a != b) s += p[(size_t)ex[a] * ne + ex[b]];
        r.kv("collab.intra." + std::to_string(d), m >= 2 ? s / (double)(m * (m - 1)) : 0.0);
    }
    for (int d1 = 0; d1 < nd; ++d1)
        for (int d2 = d1 + 1; d2 < nd; ++d2) {
            double s = 0.0;
            for (int i : R.devices[d1])
                for (int j : R.devices[d2]) s += p[(size_t)i * ne + j];
            r.kv("collab.inter." + std::to_string(d1) + "." + std::to_string(d2),
                 s / (double)(R.devices[d1].size() * R.devices[d2].size()));
        }
    if (R.oracle_err >= 0.0) r.kv("oracle.max_rel_error", R.oracle_err);
    write_file(o.out, r.os.str());
}

int cmd_simulate(const std::vector<std::string>& a, std::ostream& out) {  // cli.cpp:380-391
    SimOpts o = sim_opts(parse_args(a, kSimOptions, kSimFlags));
    if (o.out.empty()) throw UsageError("--out is required");
    const SimResult R = run_simulate(o);
    write_simulate_report(o, R);
    out << "simulate: mean replicas " << fmt(R.rep.mean_replicas) << " (cap " << fmt(R.rep.cap_replicas)
        << "), cross-device bytes " << R.rep.cross_device_bytes << "\n";
    if (R.oracle_err >= 0.0) out << "oracle max relative error: " << fmt(R.oracle_err) << "\n";
    return 0;
}

int cmd_sweep_prune(const std::vector<std::string>& a, std::ostream& out) {  // cli.cpp:422-441
    const Args args = parse_args(a, kSimOptions, kSimFlags);
    SimOpts o = sim_opts(args);
    o.prune = args.need("--mode");
    const std::string prefix = args.need("--out-prefix");
    if (o.prune == "none") throw UsageError("sweep-prune: --mode must be router or similarity");
    o.trace.clear();
    const int per = o.experts / std::max(o.devices, 1);
    const int d_min = per ? std::max(1, (o.topk + per - 1) / per) : 1;
    for (int d = 1; d < d_min; ++d)
        out << "budget " << d << ": skipped (" << d << " device(s) host fewer than k=" << o.topk << " experts)\n";
    for (int d = d_min; d <= o.devices; ++d) {
        o.budget = d;
        o.out = prefix + ".d" + std::to_string(d) + ".txt";
        const SimResult R = run_simulate(o);
        write_simulate_report(o, R);
        out << "budget " << d << ": mean replicas " << fmt(R.rep.mean_replicas) << " -> " << o.out << "\n";
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> a(argv + 1, argv + argc);
    if (a.empty()) {
        std::cerr << "usage: moesim_gpu gen-trace|profile|reschedule|simulate|sweep-prune [options]\n";
        return 2;
    }
    const std::string cmd = a[0];
    a.erase(a.begin());
    try {
        if (cmd == "gen-trace") return cmd_gen_trace(a);
        if (cmd == "profile") return cmd_profile(a, std::cout);
        if (cmd == "reschedule") return cmd_reschedule(a);
        if (cmd == "simulate") return cmd_simulate(a, std::cout);
        if (cmd == "sweep-prune") return cmd_sweep_prune(a, std::cout);
        std::cerr << "usage error: unknown command '" << cmd << "'\n";
        return 2;
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 2;
    } catch (const DataError& e) {
        std::cerr << "data error: " << e.what() << "\n";
        return 3;
    } catch (const CapacityError& e) {
        std::cerr << "capacity error: " << e.what() << "\n";
        return 4;
    } catch (const PlacementError& e) {
        std::cerr << "placement error: " << e.what() << "\n";
        return 4;
    } catch (const std::invalid_argument& e) {
        std::cerr << "usage error: expected a number\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
