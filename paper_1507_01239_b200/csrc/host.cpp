#include "host.h"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <stdexcept>
#include <thread>

namespace pnb {
namespace host {

std::string fmt_num(double v) {
    std::ostringstream os;
    if (std::isnan(v)) os << (std::signbit(v) ? "-nan" : "nan");  // as glibc prints it
    else os << v;
    return os.str();
}

namespace {
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

inline uint64_t splitmix_next(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }
}  // namespace

Rng::Rng(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s_[i] = splitmix_next(x);
}

uint64_t Rng::next_u64() {
    const uint64_t out = rotl(s_[1] * 5, 7) * 9;
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

uint64_t Rng::uniform_index(uint64_t bound) {
    if (bound == 0) fail("uniform_index: bound must be positive");
    const uint64_t reject_below = (0ull - bound) % bound;
    uint64_t r;
    do {
        r = next_u64();
    } while (r < reject_below);
    return r % bound;
}

double Rng::gaussian(double mean, double stddev) {
    if (stddev < 0.0) fail("gaussian: stddev must be >= 0, got " + std::to_string(stddev));
    if (stddev == 0.0) return mean;  // no draw consumed
    if (has_spare_) {
        has_spare_ = false;
        return mean + stddev * spare_;
    }
    double u, v, s;
    for (;;) {
        u = uniform(-1.0, 1.0);
        v = uniform(-1.0, 1.0);
        s = u * u + v * v;
        if (s < 1.0 && s != 0.0) break;
    }
    const double k = std::sqrt(-2.0 * std::log(s) / s);
    spare_ = v * k;
    has_spare_ = true;
    return mean + stddev * (u * k);
}

namespace {
void advance(uint64_t s[4]) {  // state update of next_u64 without the output
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
}

void apply(const Jump& m, const uint64_t x[4], uint64_t out[4]) {
    uint64_t r[4] = {0, 0, 0, 0};
    for (int k = 0; k < 256; ++k)
        if ((x[k >> 6] >> (k & 63)) & 1)
            for (int w = 0; w < 4; ++w) r[w] ^= m.col[k][w];
    for (int w = 0; w < 4; ++w) out[w] = r[w];
}

void compose(const Jump& a, const Jump& b, Jump& out) {  // out = a o b
    Jump t;
    for (int j = 0; j < 256; ++j) apply(a, b.col[j], t.col[j]);
    out = t;
}
}  // namespace

Jump make_jump(uint64_t n) {
    Jump step, acc;
    for (int j = 0; j < 256; ++j) {
        uint64_t e[4] = {0, 0, 0, 0};
        e[j >> 6] = 1ull << (j & 63);
        for (int w = 0; w < 4; ++w) acc.col[j][w] = e[w];
        advance(e);
        for (int w = 0; w < 4; ++w) step.col[j][w] = e[w];
    }
    while (n) {
        if (n & 1) compose(step, acc, acc);
        n >>= 1;
        if (n) compose(step, step, step);
    }
    return acc;
}

Jump jump_square(const Jump& j) {
    Jump out;
    compose(j, j, out);
    return out;
}

void Rng::jump(const Jump& j) {
    uint64_t out[4];
    apply(j, s_, out);
    for (int w = 0; w < 4; ++w) s_[w] = out[w];
}

std::vector<uint64_t> shuffled_indices(uint64_t n, uint64_t seed) {
    std::vector<uint64_t> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = i;
    Rng(seed).shuffle(v);
    return v;
}

std::vector<uint64_t> partition_rows(uint64_t n, uint64_t m, uint64_t seed) {
    if (m == 0) fail("partition_data: m must be >= 1");
    if (m > n) fail("partition_data: m = " + std::to_string(m) + " exceeds dataset size " + std::to_string(n));
    std::vector<uint64_t> idx = shuffled_indices(n, seed);
    idx.resize((n / m) * m);
    return idx;
}

std::vector<uint64_t> minibatch_rows(uint64_t n, uint64_t b, uint64_t seed) {
    if (b == 0) fail("minibatches: batch size must be >= 1");
    if (b > n) fail("minibatches: batch size " + std::to_string(b) + " exceeds dataset size " + std::to_string(n));
    std::vector<uint64_t> idx = shuffled_indices(n, seed);
    idx.resize((n / b) * b);
    return idx;
}

HostData generate_synthetic(uint64_t classes, uint64_t dim, uint64_t per_class, double sep, uint64_t seed) {
    if (classes == 0 || dim == 0 || per_class == 0)
        fail("generate_synthetic: classes, dim and per_class must be >= 1");
    if (sep < 0.0) fail("generate_synthetic: separation must be >= 0, got " + fmt_num(sep));
    Rng rng(seed);
    std::vector<double> mu(classes * dim);
    for (uint64_t k = 0; k < classes; ++k) {
        double* row = mu.data() + k * dim;
        double nrm;
        do {
            for (uint64_t j = 0; j < dim; ++j) row[j] = rng.gaussian(0.0, 1.0);
            double acc = 0.0;
            for (uint64_t j = 0; j < dim; ++j) acc += row[j] * row[j];
            nrm = std::sqrt(acc);
        } while (nrm == 0.0);
        const double scale = sep / nrm;
        for (uint64_t j = 0; j < dim; ++j) row[j] *= scale;
    }
    HostData d;
    d.n = classes * per_class;
    d.d = dim;
    d.x.resize(d.n * dim);
    d.y.resize(d.n);
    uint64_t r = 0;
    for (uint64_t k = 0; k < classes; ++k)
        for (uint64_t i = 0; i < per_class; ++i, ++r) {
            for (uint64_t j = 0; j < dim; ++j) d.x[r * dim + j] = mu[k * dim + j] + rng.gaussian(0.0, 1.0);
            d.y[r] = static_cast<int32_t>(k);
        }
    return d;
}

void split_cv(const HostData& all, double f, uint64_t seed, HostData& train, HostData& cv) {
    if (f <= 0.0 || f >= 1.0) fail("split_cv: cv_fraction must be in (0,1), got " + fmt_num(f));
    if (all.n < 10) fail("split_cv: need at least 10 examples, got " + std::to_string(all.n));
    const std::vector<uint64_t> idx = shuffled_indices(all.n, seed);
    const uint64_t c = static_cast<uint64_t>(std::ceil(f * static_cast<double>(all.n)));
    auto take = [&](HostData& out, uint64_t lo, uint64_t hi) {
        out.n = hi - lo;
        out.d = all.d;
        out.x.resize(out.n * all.d);
        out.y.resize(out.n);
        for (uint64_t i = lo; i < hi; ++i) {
            std::memcpy(out.x.data() + (i - lo) * all.d, all.x.data() + idx[i] * all.d, all.d * sizeof(double));
            out.y[i - lo] = all.y[idx[i]];
        }
    };
    take(cv, 0, c);
    take(train, c, all.n);
}

void feature_stats(const HostData& d, std::vector<double>& mean, std::vector<double>& sd) {
    if (d.n == 0) fail("feature_stats: empty dataset");
    mean.assign(d.d, 0.0);
    sd.assign(d.d, 0.0);
    for (uint64_t i = 0; i < d.n; ++i)
        for (uint64_t j = 0; j < d.d; ++j) mean[j] += d.x[i * d.d + j];
    for (double& m : mean) m /= static_cast<double>(d.n);
    for (uint64_t i = 0; i < d.n; ++i)
        for (uint64_t j = 0; j < d.d; ++j) {
            const double c = d.x[i * d.d + j] - mean[j];
            sd[j] += c * c;
        }
    for (double& s : sd) {
        s = std::sqrt(s / static_cast<double>(d.n));
        if (s < 1e-12) s = 1.0;  // data.cpp:226 replaces (not floors) tiny spreads
    }
}

void standardize(HostData& d, const std::vector<double>& mean, const std::vector<double>& sd) {
    if (mean.size() != d.d) fail("standardize: stats dim does not match data dim");
    for (uint64_t i = 0; i < d.n; ++i)
        for (uint64_t j = 0; j < d.d; ++j) d.x[i * d.d + j] = (d.x[i * d.d + j] - mean[j]) / sd[j];
}

// ---- load_csv / save_csv (data.cpp:29-122) --------------------------------
namespace {

std::string csv_trim(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r");
    if (a == std::string::npos) return "";
    const size_t b = s.find_last_not_of(" \t\r");
    return s.substr(a, b - a + 1);
}

// std::stod semantics (data.cpp:29-41): strtod over the whole field, range errors
// (errno ERANGE) and non-finite values rejected
bool csv_number(const std::string& f, double& v) {
    if (f.empty()) return false;
    errno = 0;
    char* end = nullptr;
    v = std::strtod(f.c_str(), &end);
    if (end == f.c_str() || errno == ERANGE) return false;
    return static_cast<size_t>(end - f.c_str()) == f.size() && std::isfinite(v);
}

struct CsvChunk {
    std::vector<double> x;
    std::vector<int32_t> y;
    uint64_t dim = 0;          // features of this chunk's first data row
    uint64_t first_line = 0;   // its line number (0: no data rows)
    uint64_t err_line = 0;     // first failing line of the chunk (0: none)
    std::string err;
    int max_label = -1;
};

// lines [l0, l1) of the file, numbered from line_base + 1
void csv_parse_chunk(const char* text, const std::vector<size_t>& starts, size_t l0, size_t l1, size_t len,
                     CsvChunk& c) {
    for (size_t li = l0; li < l1; ++li) {
        const size_t a = starts[li];
        size_t b = li + 1 < starts.size() ? starts[li + 1] - 1 : len;  // drop the '\n'
        if (li + 1 == starts.size() && b > a && text[b - 1] == '\n') --b;  // the file's final newline
        const std::string stripped = csv_trim(std::string(text + a, text + b));
        const uint64_t line_no = li + 1;
        if (stripped.empty() || stripped[0] == '#') continue;
        std::vector<std::string> fields;
        size_t st = 0;
        for (;;) {
            const size_t comma = stripped.find(',', st);
            if (comma == std::string::npos) {
                fields.push_back(stripped.substr(st));
                break;
            }
            fields.push_back(stripped.substr(st, comma - st));
            st = comma + 1;
        }
        auto error = [&](const std::string& m) {
            c.err_line = line_no;
            c.err = m;
        };
        if (fields.size() < 2) return error("load_csv: expected 'label,f1,...' at line " + std::to_string(line_no));
        double lv = 0.0;
        const std::string lf = csv_trim(fields[0]);
        if (!csv_number(lf, lv))
            return error("load_csv: non-numeric label '" + lf + "' at line " + std::to_string(line_no));
        if (lv < 0 || lv != std::floor(lv))
            return error("load_csv: label must be a non-negative integer, got '" + fields[0] + "' at line " +
                         std::to_string(line_no));
        const uint64_t row_dim = fields.size() - 1;
        if (c.first_line == 0) {
            c.first_line = line_no;
            c.dim = row_dim;
        } else if (row_dim != c.dim) {
            return error("load_csv: ragged row with " + std::to_string(row_dim) + " features (expected " +
                         std::to_string(c.dim) + ") at line " + std::to_string(line_no));
        }
        for (size_t j = 1; j < fields.size(); ++j) {
            double v = 0.0;
            const std::string ff = csv_trim(fields[j]);
            if (!csv_number(ff, v))
                return error("load_csv: non-numeric feature '" + ff + "' at line " + std::to_string(line_no));
            c.x.push_back(v);
        }
        c.y.push_back(static_cast<int32_t>(lv));
        c.max_label = std::max(c.max_label, c.y.back());
    }
}

}  // namespace

HostData load_csv(const std::string& path, uint64_t* classes) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail("load_csv: cannot open '" + path + "'");
    const std::string text((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    // line starts (std::getline semantics: a final line without '\n' still counts)
    std::vector<size_t> starts;
    if (!text.empty()) starts.push_back(0);
    for (size_t i = 0; i < text.size(); ++i)
        if (text[i] == '\n' && i + 1 < text.size()) starts.push_back(i + 1);
    const size_t nl = starts.size();
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nch = std::max<size_t>(1, std::min<size_t>(hw, nl / 4096 + 1));
    std::vector<CsvChunk> ch(nch);
    std::vector<std::thread> th;
    for (size_t k = 0; k < nch; ++k)
        th.emplace_back([&, k] { csv_parse_chunk(text.data(), starts, nl * k / nch, nl * (k + 1) / nch, text.size(), ch[k]); });
    for (auto& t : th) t.join();
    // the reference stops at the first failing line in file order; a chunk's first
    // data row is checked against the file's first data row (global dim) first
    uint64_t dim = 0;
    for (const CsvChunk& c : ch) {
        if (c.first_line && dim == 0) dim = c.dim;
        if (c.first_line && c.dim != dim)
            fail("load_csv: ragged row with " + std::to_string(c.dim) + " features (expected " + std::to_string(dim) +
                 ") at line " + std::to_string(c.first_line));
        if (c.err_line) fail(c.err);
    }
    HostData d;
    d.d = dim;
    int max_label = -1;
    for (const CsvChunk& c : ch) {
        d.x.insert(d.x.end(), c.x.begin(), c.x.end());
        d.y.insert(d.y.end(), c.y.begin(), c.y.end());
        max_label = std::max(max_label, c.max_label);
    }
    d.n = d.y.size();
    if (d.n == 0) fail("load_csv: no data rows in '" + path + "'");
    if (classes) *classes = static_cast<uint64_t>(max_label) + 1;
    return d;
}

void save_csv(const std::string& path, const HostData& d) {
    std::ofstream os(path, std::ios::trunc);
    if (!os) fail("save_csv: cannot open '" + path + "' for writing");
    char buf[32];
    for (uint64_t i = 0; i < d.n; ++i) {
        os << d.y[i];
        for (uint64_t j = 0; j < d.d; ++j) {
            std::snprintf(buf, sizeof(buf), "%.17g", d.x[i * d.d + j]);
            os << ',' << buf;
        }
        os << '\n';
    }
    if (!os) fail("save_csv: write failed for '" + path + "'");
}

uint64_t param_count(const std::vector<uint64_t>& dims) {
    uint64_t t = 0;
    for (size_t l = 0; l + 1 < dims.size(); ++l) t += dims[l + 1] * dims[l] + dims[l + 1];
    return t;
}

std::vector<double> init_random(const std::vector<uint64_t>& dims, Rng& rng) {
    if (dims.size() < 2) fail("init_random: need at least 2 dims, got " + std::to_string(dims.size()));
    for (uint64_t d : dims)
        if (d == 0) fail("init_random: zero layer dimension");
    std::vector<double> p;
    p.reserve(param_count(dims));
    for (size_t l = 0; l + 1 < dims.size(); ++l) {
        const double r = std::sqrt(6.0 / static_cast<double>(dims[l] + dims[l + 1]));
        for (uint64_t i = 0; i < dims[l] * dims[l + 1]; ++i) p.push_back(rng.uniform(-r, r));
        for (uint64_t i = 0; i < dims[l + 1]; ++i) p.push_back(0.0);
    }
    return p;
}

Schedule make_schedule(bool newbob, double lr_init, uint64_t epochs) {
    if (lr_init <= 0.0) fail("make_schedule: lr_init must be positive, got " + fmt_num(lr_init));
    if (epochs == 0) fail("make_schedule: planned_epochs must be positive");
    Schedule s;
    s.newbob = newbob;
    s.lr_init = lr_init;
    s.newbob_lr = lr_init;
    s.planned_epochs = epochs;
    return s;
}

double exponential_lr(const Schedule& s, double progress) {
    if (progress < 0.0 || progress > 1.0)
        fail("exponential_lr: progress must be in [0,1], got " + fmt_num(progress));
    return s.lr_init * std::pow(s.final_ratio, progress);
}

bool newbob_next(Schedule& s, double prev, double acc, double* lr_out) {
    if (prev < 0.0 || prev > 1.0 || acc < 0.0 || acc > 1.0)
        fail("newbob_next: accuracies must be in [0,1], got " + fmt_num(prev) + " and " + fmt_num(acc));
    const double gain = acc - prev;
    bool stop = false;
    if (s.halving) {
        stop = gain < s.stop_threshold;
        s.newbob_lr *= 0.5;
    } else if (gain < s.halve_threshold) {
        s.halving = true;
        s.newbob_lr *= 0.5;
    }
    if (lr_out) *lr_out = s.newbob_lr;
    return stop;
}

double scale_lr_for_workers(double lr_init, uint64_t workers) {
    if (workers == 0) fail("scale_lr_for_workers: workers must be >= 1");
    return lr_init * static_cast<double>(workers);
}

namespace {
void put_le(std::string& buf, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) buf.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}
uint64_t get_le(const unsigned char* p, int bytes) {
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    return v;
}
}  // namespace

void save_model(const std::string& path, const std::vector<uint64_t>& dims, int act, const std::vector<double>& p) {
    if (p.size() != param_count(dims)) fail("save_model: parameter count does not match dims");
    std::string buf("PARNNET1");
    put_le(buf, 1, 4);
    put_le(buf, act == 0 ? 0 : 1, 4);
    put_le(buf, dims.size(), 4);
    for (uint64_t d : dims) put_le(buf, d, 8);
    for (double v : p) {
        uint64_t bits;
        std::memcpy(&bits, &v, 8);
        put_le(buf, bits, 8);
    }
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) fail("save_model: cannot open '" + path + "' for writing");
    os.write(buf.data(), static_cast<std::streamsize>(buf.size()));
    if (!os) fail("save_model: write failed for '" + path + "'");
}

void load_model(const std::string& path, std::vector<uint64_t>& dims, int& act, std::vector<double>& p) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail("load_model: cannot open '" + path + "'");
    std::string buf((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    const auto* u = reinterpret_cast<const unsigned char*>(buf.data());
    if (buf.size() < 8 || buf.compare(0, 8, "PARNNET1") != 0) fail("load_model: bad magic in '" + path + "'");
    auto need = [&](size_t end) {
        if (buf.size() < end) fail("load_model: truncated file " + path);
    };
    need(20);
    const uint64_t ver = get_le(u + 8, 4), a = get_le(u + 12, 4), nd = get_le(u + 16, 4);
    if (ver != 1) fail("load_model: unsupported version " + std::to_string(ver));
    if (a > 1) fail("load_model: bad activation code " + std::to_string(a));
    if (nd < 2) fail("load_model: bad dim count " + std::to_string(nd));
    need(20 + 8 * nd);
    dims.resize(nd);
    for (uint64_t i = 0; i < nd; ++i) dims[i] = get_le(u + 20 + 8 * i, 8);
    const uint64_t P = param_count(dims);
    const size_t off = 20 + 8 * nd;
    need(off + 8 * P);
    p.resize(P);
    for (uint64_t i = 0; i < P; ++i) {
        const uint64_t bits = get_le(u + off + 8 * i, 8);
        std::memcpy(&p[i], &bits, 8);
    }
    act = static_cast<int>(a);
}

namespace {
void tree_into(const std::vector<const double*>& c, size_t lo, size_t hi, uint64_t len, double* out) {
    if (hi - lo == 1) {
        std::memcpy(out, c[lo], len * sizeof(double));
        return;
    }
    const size_t mid = lo + (hi - lo) / 2;
    tree_into(c, lo, mid, len, out);
    std::vector<double> right(len);
    tree_into(c, mid, hi, len, right.data());
    for (uint64_t i = 0; i < len; ++i) out[i] += right[i];
}
}  // namespace

std::vector<double> allreduce_average(const std::vector<const double*>& contrib, uint64_t len) {
    const size_t m = contrib.size();
    if (m == 0) fail("allreduce_average: m must be >= 1");
    std::vector<double> out(len);
    tree_into(contrib, 0, m, len, out.data());
    const double inv = 1.0 / static_cast<double>(m);
    for (double& v : out) v *= inv;
    return out;
}

std::vector<double> lowrank_basis(uint64_t dim, uint64_t rank, uint64_t seed) {
    if (rank == 0 || rank >= dim) fail("lowrank_basis: need 0 < rank < dim, got rank " + std::to_string(rank) +
                                       ", dim " + std::to_string(dim));
    Rng rng(seed);
    std::vector<double> m(rank * dim);
    for (uint64_t i = 0; i < rank * dim; ++i) m[i] = rng.gaussian(0.0, 1.0);
    for (uint64_t i = 0; i < rank; ++i) {
        double* v = &m[i * dim];
        for (uint64_t k = 0; k < i; ++k) {
            const double* u = &m[k * dim];
            double dot = 0.0;
            for (uint64_t j = 0; j < dim; ++j) dot += u[j] * v[j];
            for (uint64_t j = 0; j < dim; ++j) v[j] -= dot * u[j];
        }
        double nn = 0.0;
        for (uint64_t j = 0; j < dim; ++j) nn += v[j] * v[j];
        const double inv = 1.0 / std::sqrt(nn);
        for (uint64_t j = 0; j < dim; ++j) v[j] *= inv;
    }
    return m;
}

uint64_t lowrank_seed(int layer, int side) { return 0x4C524E470000ULL + 2ULL * layer + side; }

}  // namespace host
}  // namespace pnb
