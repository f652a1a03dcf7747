// csd_host.cpp — the reference's C++ csd:: operator API (include/csd/*.hpp) implemented on
// top of the C ABI (include/csd_b200.h).  A caller of the reference library relinks against
// libcsd_host.so and its voxel / top-k / attention / MLP calls run on the B200 in
// CSD_MODE_CHECK (bit-exact with the reference's CPU arithmetic); the caches keep the
// reference's public host layouts so existing callers and tests read them unchanged.
//
// Validation order and exception types follow the reference functions cited per routine;
// the ABI's csd_status codes are rethrown as the matching csd:: exception.
#include <algorithm>
#include <cctype>
#include <iterator>
#include <memory>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>


#include "csd/attention.hpp"
#include "csd/metrics.hpp"
#include "csd/mlp.hpp"
#include "csd/model.hpp"
#include "csd/rng.hpp"
#include "csd/voxel.hpp"
#include "csd_b200.h"

namespace csd {
namespace {

[[noreturn]] void rethrow(csd_status s) {
    const std::string msg = csd_last_error();
    switch (s) {
        case CSD_ERR_SHAPE: throw ShapeError(msg);
        case CSD_ERR_INDEX: throw IndexError(msg);
        case CSD_ERR_NUMERIC: throw NumericError(msg);
        case CSD_ERR_STATE: throw StateError(msg);
        case CSD_ERR_VALUE: throw ValueError(msg);
        case CSD_ERR_CONFIG: throw ConfigError(msg);
        default: throw Error(std::string(csd_status_name(s)) + ": " + msg);
    }
}
void ok(csd_status s) {
    if (s != CSD_OK) rethrow(s);
}

csd_ctx* ctx() {  // one context per process, on device 0 (fails loudly without a GPU)
    static csd_ctx* c = [] {
        csd_ctx* h = nullptr;
        ok(csd_ctx_create(0, &h));
        return h;
    }();
    return c;
}

// RAII device buffer
class Dev {
public:
    explicit Dev(size_t bytes) : bytes_(bytes) { ok(csd_device_alloc(bytes, &p_)); }
    template <class T>
    explicit Dev(const std::vector<T>& host) : Dev(host.size() * sizeof(T)) {
        ok(csd_copy_to_device(p_, host.data(), bytes_));
    }
    explicit Dev(const Tensor& t) : Dev(sizeof(float) * static_cast<size_t>(t.numel())) {
        ok(csd_copy_to_device(p_, t.data(), bytes_));
    }
    ~Dev() { csd_device_free(p_); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    float* f() const { return static_cast<float*>(p_); }
    int32_t* i() const { return static_cast<int32_t*>(p_); }
    void* v() const { return p_; }
    void to(Tensor& t) const { ok(csd_copy_to_host(t.data(), p_, sizeof(float) * t.numel())); }
    template <class T>
    void to(std::vector<T>& h) const { ok(csd_copy_to_host(h.data(), p_, sizeof(T) * h.size())); }

private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

void sync() { ok(csd_ctx_sync(ctx(), nullptr)); }

}  // namespace

// ====================================================================== Tensor (host)
Tensor::Tensor() : dims_(), vals_(1, 0.0f) {}
Tensor::Tensor(std::vector<int64_t> shape) : dims_(std::move(shape)) {
    for (int64_t d : dims_)
        if (d < 1) throw ShapeError("invalid tensor shape " + shape_str(dims_) + ": dims must be >= 1");
    vals_.assign(static_cast<size_t>(shape_numel(dims_)), 0.0f);
}
Tensor::Tensor(std::vector<int64_t> shape, std::vector<float> data)
    : dims_(std::move(shape)), vals_(std::move(data)) {
    for (int64_t d : dims_)
        if (d < 1) throw ShapeError("invalid tensor shape " + shape_str(dims_) + ": dims must be >= 1");
    if (shape_numel(dims_) != static_cast<int64_t>(vals_.size()))
        throw ShapeError("tensor data length " + std::to_string(vals_.size()) +
                         " does not match shape " + shape_str(dims_));
}
Tensor Tensor::full(std::vector<int64_t> shape, float value) {
    Tensor t(std::move(shape));
    std::fill(t.vals_.begin(), t.vals_.end(), value);
    return t;
}
int64_t Tensor::dim(int64_t axis) const {
    if (axis < 0 || axis >= rank())
        throw ShapeError("dimension index " + std::to_string(axis) + " out of range for shape " +
                         shape_str(dims_));
    return dims_[static_cast<size_t>(axis)];
}
std::string shape_str(const std::vector<int64_t>& shape) {
    std::string s = "[";
    for (size_t i = 0; i < shape.size(); ++i) s += (i ? "x" : "") + std::to_string(shape[i]);
    return s + "]";
}
int64_t shape_numel(const std::vector<int64_t>& shape) {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
}

// Host tensor utilities with the reference's arithmetic (tensor.cpp:66-225): sequential
// fp32 accumulation (this file is compiled with -ffp-contract=off).
Tensor gemm(const Tensor& a, const Tensor& b, bool transpose_b) {
    if (a.rank() != 2 || b.rank() != 2)
        throw ShapeError("gemm expects rank-2 operands, got " + shape_str(a.shape()) + " and " +
                         shape_str(b.shape()));
    const int64_t m = a.dim(0), kk = a.dim(1);
    const int64_t inner = transpose_b ? b.dim(1) : b.dim(0), n = transpose_b ? b.dim(0) : b.dim(1);
    if (kk != inner)
        throw ShapeError("gemm inner dimensions disagree: " + shape_str(a.shape()) + " @ " +
                         shape_str(b.shape()));
    Tensor c({m, n});
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (int64_t k = 0; k < kk; ++k)
                acc += a[i * kk + k] * (transpose_b ? b[j * kk + k] : b[k * n + j]);
            c[i * n + j] = acc;
        }
    return c;
}
SoftmaxResult softmax_rows(const Tensor& logits) {
    if (logits.rank() < 1) throw ShapeError("softmax_rows expects rank >= 1, got scalar");
    const int64_t len = logits.dim(logits.rank() - 1), rows = logits.numel() / len;
    std::vector<int64_t> st(logits.shape().begin(), logits.shape().end() - 1);
    SoftmaxResult r{Tensor(logits.shape()), {Tensor(st), Tensor(st)}};
    for (int64_t i = 0; i < rows; ++i) {
        const float* row = logits.data() + i * len;
        float m = row[0];
        for (int64_t j = 0; j < len; ++j) {
            if (!std::isfinite(row[j]))
                throw NumericError("softmax_rows: non-finite logit at row " + std::to_string(i) +
                                   ", position " + std::to_string(j));
            m = std::max(m, row[j]);
        }
        float l = 0.0f;
        float* o = r.probs.data() + i * len;
        for (int64_t j = 0; j < len; ++j) l += (o[j] = std::exp(row[j] - m));
        for (int64_t j = 0; j < len; ++j) o[j] /= l;
        r.stats.row_max[i] = m;
        r.stats.exp_sum[i] = l;
    }
    return r;
}
Tensor gelu(const Tensor& x) {
    const float k = std::sqrt(2.0f / static_cast<float>(M_PI));
    Tensor y(x.shape());
    for (int64_t i = 0; i < x.numel(); ++i) {
        const float v = x[i];
        y[i] = 0.5f * v * (1.0f + std::tanh(k * (v + 0.044715f * v * v * v)));
    }
    return y;
}
Tensor gather_rows(const Tensor& t, const std::vector<int64_t>& indices) {
    if (t.rank() < 2) throw ShapeError("gather_rows expects rank >= 2, got " + shape_str(t.shape()));
    const int64_t cols = t.dim(t.rank() - 1), rows = t.dim(t.rank() - 2);
    for (int64_t id : indices)
        if (id < 0 || id >= rows)
            throw IndexError("gather_rows: index " + std::to_string(id) + " out of range [0, " +
                             std::to_string(rows) + ")");
    if (indices.empty()) throw ShapeError("gather_rows: empty index list");
    std::vector<int64_t> os = t.shape();
    os[os.size() - 2] = static_cast<int64_t>(indices.size());
    Tensor out(os);
    const int64_t slices = t.numel() / (rows * cols), orow = static_cast<int64_t>(indices.size());
    for (int64_t s = 0; s < slices; ++s)
        for (int64_t j = 0; j < orow; ++j)
            std::memcpy(out.data() + (s * orow + j) * cols,
                        t.data() + (s * rows + indices[static_cast<size_t>(j)]) * cols,
                        sizeof(float) * cols);
    return out;
}
Tensor chunk_reduce(const Tensor& t, int64_t chunk, ReduceMode mode) {
    if (t.rank() < 2) throw ShapeError("chunk_reduce expects rank >= 2, got " + shape_str(t.shape()));
    if (chunk < 1) throw ValueError("chunk_reduce: chunk must be >= 1, got " + std::to_string(chunk));
    const int64_t cols = t.dim(t.rank() - 1), rows = t.dim(t.rank() - 2);
    if (rows % chunk)
        throw ShapeError("chunk_reduce: row count " + std::to_string(rows) +
                         " not divisible by chunk " + std::to_string(chunk));
    std::vector<int64_t> os = t.shape();
    os[os.size() - 2] = rows / chunk;
    Tensor out(os);
    const int64_t slices = t.numel() / (rows * cols);
    const float inv = 1.0f / static_cast<float>(chunk);
    for (int64_t s = 0; s < slices; ++s)
        for (int64_t i = 0; i < rows / chunk; ++i) {
            float* w = out.data() + (s * (rows / chunk) + i) * cols;
            for (int64_t r = i * chunk; r < (i + 1) * chunk; ++r)
                for (int64_t c = 0; c < cols; ++c) w[c] += t[(s * rows + r) * cols + c];
            if (mode == ReduceMode::Mean)
                for (int64_t c = 0; c < cols; ++c) w[c] *= inv;
        }
    return out;
}
double r_squared(const Tensor& exact, const Tensor& approx) {
    if (exact.shape() != approx.shape())
        throw ShapeError("r_squared shapes disagree: " + shape_str(exact.shape()) + " vs " +
                         shape_str(approx.shape()));
    const int64_t n = exact.numel();
    double mean = 0.0;
    for (int64_t i = 0; i < n; ++i) mean += exact[i];
    mean /= static_cast<double>(n);
    double res = 0.0, tot = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double e = exact[i], a = approx[i];
        res += (e - a) * (e - a);
        tot += (e - mean) * (e - mean);
    }
    if (tot == 0.0) throw NumericError("r_squared undefined: true delta has zero variance");
    return 1.0 - res / tot;
}

// ====================================================================== voxel (device)
void VoxelLayout::validate() const {  // voxel.cpp:7-16
    if (t < 1 || h < 1 || w < 1 || vt < 1 || vh < 1 || vw < 1)
        throw ConfigError("voxel layout dimensions must be >= 1");
    if (t % vt || h % vh || w % vw)
        throw ConfigError("voxel (" + std::to_string(vt) + "," + std::to_string(vh) + "," +
                          std::to_string(vw) + ") does not tile grid (" + std::to_string(t) + "," +
                          std::to_string(h) + "," + std::to_string(w) + ")");
}
std::vector<int64_t> voxel_permutation(const VoxelLayout& L) {
    L.validate();
    std::vector<int64_t> perm(static_cast<size_t>(L.tokens()));
    ok(csd_voxel_permutation(L.t, L.h, L.w, L.vt, L.vh, L.vw, perm.data()));
    return perm;
}
VoxelOrderResult voxel_order(const Tensor& x, const VoxelLayout& L) {  // voxel.cpp:44-73
    L.validate();
    if (x.rank() != 5) throw ShapeError("voxel_order expects [B x T x H x W x D], got " + shape_str(x.shape()));
    if (x.dim(1) != L.t || x.dim(2) != L.h || x.dim(3) != L.w)
        throw ShapeError("voxel_order: tensor grid " + shape_str(x.shape()) + " does not match layout");
    VoxelOrderResult r{Tensor({x.dim(0), L.tokens(), x.dim(4)}), voxel_permutation(L)};
    Dev src(x), dst(sizeof(float) * x.numel());
    ok(csd_voxel_reorder(ctx(), src.v(), dst.v(), x.dim(0), L.t, L.h, L.w, L.vt, L.vh, L.vw,
                         sizeof(float) * x.dim(4), 0, nullptr));
    dst.to(r.reordered);
    return r;
}
Tensor reverse_voxel_order(const Tensor& x, const VoxelLayout& L) {  // voxel.cpp:75-102
    L.validate();
    if (x.rank() != 3) throw ShapeError("reverse_voxel_order expects [B x N x D], got " + shape_str(x.shape()));
    if (x.dim(1) != L.tokens())
        throw ShapeError("reverse_voxel_order: sequence length " + std::to_string(x.dim(1)) +
                         " does not match layout token count " + std::to_string(L.tokens()));
    Tensor out({x.dim(0), L.t, L.h, L.w, x.dim(2)});
    Dev src(x), dst(sizeof(float) * x.numel());
    ok(csd_voxel_reorder(ctx(), src.v(), dst.v(), x.dim(0), L.t, L.h, L.w, L.vt, L.vh, L.vw,
                         sizeof(float) * x.dim(2), 1, nullptr));
    dst.to(out);
    return out;
}

// ====================================================================== index sets
SparseIndexSet SparseIndexSet::empty(int64_t batch, int64_t heads, int64_t chunks,
                                     int64_t chunk_size, int64_t k_max, int64_t domain) {
    SparseIndexSet s;
    s.batch = batch; s.heads = heads; s.chunks = chunks; s.chunk_size = chunk_size;
    s.k_max = k_max; s.domain = domain;
    s.indices.assign(static_cast<size_t>(batch * heads * chunks * k_max), 0);
    s.counts.assign(static_cast<size_t>(batch * heads * chunks), 0);
    return s;
}
void SparseIndexSet::validate() const {  // sparse_index.cpp:27-62, range/dup checks on device
    if (batch < 1 || heads < 1 || chunks < 1 || chunk_size < 1 || domain < 1)
        throw ValueError("sparse index set has empty dimensions");
    if (k_max < 0 || k_max > domain)
        throw ValueError("sparse index set k_max " + std::to_string(k_max) + " outside [0, domain=" +
                         std::to_string(domain) + "]");
    if (static_cast<int64_t>(indices.size()) != batch * heads * chunks * k_max ||
        static_cast<int64_t>(counts.size()) != batch * heads * chunks)
        throw ValueError("sparse index set storage does not match its dimensions");
    Dev di(indices.empty() ? std::vector<int32_t>{0} : indices), dc(counts);
    ok(csd_validate_index_set(ctx(), di.i(), dc.i(), batch * heads * chunks, k_max, domain, nullptr));
    sync();
}
SparseIndexSet select_top_k(const Tensor& scores, int64_t k, int64_t chunk_size) {
    if (scores.rank() != 4)
        throw ShapeError("select_top_k expects [B x H x C x M] scores, got " + shape_str(scores.shape()));
    const int64_t b = scores.dim(0), h = scores.dim(1), c = scores.dim(2), m = scores.dim(3);
    if (k < 1 || k > m)
        throw ValueError("select_top_k: k=" + std::to_string(k) + " outside [1, " + std::to_string(m) + "]");
    SparseIndexSet s = SparseIndexSet::empty(b, h, c, chunk_size, k, m);
    Dev ds(scores), di(sizeof(int32_t) * s.indices.size()), dc(sizeof(int32_t) * s.counts.size());
    ok(csd_select_top_k(ctx(), ds.f(), b * h * c, m, k, di.i(), dc.i(), nullptr));
    di.to(s.indices);
    dc.to(s.counts);
    return s;
}
// ---- static sparsity patterns from JSON (sparse_index.hpp:36-39).  Host-side IO outside
// the hot path; a small schema-specific reader (no JSON library): the document is an object
// {"chunk_size": int, "k_max": int, "entries": [[b, h, chunk, [ids...]], ...]} (other keys
// are skipped).  Error classes follow the reference contract: malformed text / schema ->
// IoError, k_max outside [1, domain] or an entry longer than k_max -> ValueError, entry
// coordinates or ids out of range -> IndexError; the assembled set is then validated
// (duplicates -> IndexError).
namespace {
class PatternReader {
  public:
    explicit PatternReader(const std::string& t) : t_(t) {}

    [[noreturn]] void fail(const std::string& what) const {
        throw IoError("sparsity pattern JSON: " + what + " at offset " + std::to_string(p_));
    }
    void ws() {
        while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    bool peek(char c) {
        ws();
        return p_ < t_.size() && t_[p_] == c;
    }
    void expect(char c) {
        if (!peek(c)) fail(std::string("expected '") + c + "'");
        ++p_;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (p_ < t_.size() && t_[p_] != '"') {
            if (t_[p_] == '\\') {
                if (++p_ >= t_.size()) break;
            }
            out.push_back(t_[p_++]);
        }
        if (p_ >= t_.size()) fail("unterminated string");
        ++p_;
        return out;
    }
    int64_t integer() {
        ws();
        const size_t s0 = p_;
        if (p_ < t_.size() && (t_[p_] == '-' || t_[p_] == '+')) ++p_;
        while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
        if (p_ == s0 || (p_ == s0 + 1 && !std::isdigit(static_cast<unsigned char>(t_[s0]))))
            fail("expected an integer");
        if (p_ < t_.size() && (t_[p_] == '.' || t_[p_] == 'e' || t_[p_] == 'E'))
            fail("expected an integer, got a fraction");
        return std::stoll(t_.substr(s0, p_ - s0));
    }
    // skip any JSON value (for keys the schema does not use)
    void skip() {
        ws();
        if (p_ >= t_.size()) fail("unexpected end of text");
        const char c = t_[p_];
        if (c == '"') {
            str();
        } else if (c == '{' || c == '[') {
            const char close = c == '{' ? '}' : ']';
            ++p_;
            if (peek(close)) {
                ++p_;
                return;
            }
            for (;;) {
                if (c == '{') {
                    str();
                    expect(':');
                }
                skip();
                if (peek(',')) {
                    ++p_;
                    continue;
                }
                expect(close);
                return;
            }
        } else {
            while (p_ < t_.size() && !std::strchr(",]} \t\r\n", t_[p_])) ++p_;
        }
    }
    // comma-separated list in brackets; `item` parses one element
    template <typename F>
    void list(F&& item) {
        expect('[');
        if (peek(']')) {
            ++p_;
            return;
        }
        for (;;) {
            item();
            if (peek(',')) {
                ++p_;
                continue;
            }
            expect(']');
            return;
        }
    }
    void end() {
        ws();
        if (p_ != t_.size()) fail("trailing characters");
    }

  private:
    const std::string& t_;
    size_t p_ = 0;
};

struct PatternEntry {
    int64_t b, h, c;
    std::vector<int64_t> ids;
};
}  // namespace

SparseIndexSet load_index_set_json(const std::string& text, int64_t batch, int64_t heads,
                                   int64_t chunks, int64_t domain) {
    PatternReader rd(text);
    bool have_chunk = false, have_k = false, have_entries = false;
    int64_t chunk_size = 0, k_max = 0;
    std::vector<PatternEntry> entries;
    rd.expect('{');
    if (!rd.peek('}')) {
        for (;;) {
            const std::string key = rd.str();
            rd.expect(':');
            if (key == "chunk_size") {
                chunk_size = rd.integer();
                have_chunk = true;
            } else if (key == "k_max") {
                k_max = rd.integer();
                have_k = true;
            } else if (key == "entries") {
                have_entries = true;
                entries.clear();
                rd.list([&] {
                    PatternEntry e{};
                    int field = 0;
                    rd.list([&] {
                        switch (field++) {
                            case 0: e.b = rd.integer(); break;
                            case 1: e.h = rd.integer(); break;
                            case 2: e.c = rd.integer(); break;
                            case 3: rd.list([&] { e.ids.push_back(rd.integer()); }); break;
                            default: rd.fail("an entry has more than 4 fields");
                        }
                    });
                    if (field != 4) rd.fail("an entry must be [b, h, chunk, [ids...]]");
                    entries.push_back(std::move(e));
                });
            } else {
                rd.skip();
            }
            if (rd.peek(',')) {
                rd.expect(',');
                continue;
            }
            break;
        }
    }
    rd.expect('}');
    rd.end();
    if (!(have_chunk && have_k && have_entries))
        throw IoError("sparsity pattern JSON needs the keys chunk_size, k_max and entries");
    if (k_max < 1 || k_max > domain)
        throw ValueError("sparsity pattern: k_max = " + std::to_string(k_max) +
                         " is not in [1, domain = " + std::to_string(domain) + "]");
    SparseIndexSet set = SparseIndexSet::empty(batch, heads, chunks, chunk_size, k_max, domain);
    for (const PatternEntry& e : entries) {
        const bool inside = e.b >= 0 && e.b < batch && e.h >= 0 && e.h < heads && e.c >= 0 &&
                            e.c < chunks;
        if (!inside)
            throw IndexError("sparsity pattern: entry (b=" + std::to_string(e.b) + ", h=" +
                             std::to_string(e.h) + ", chunk=" + std::to_string(e.c) +
                             ") is outside [" + std::to_string(batch) + ", " +
                             std::to_string(heads) + ", " + std::to_string(chunks) + ")");
        if ((int64_t)e.ids.size() > k_max)
            throw ValueError("sparsity pattern: an entry lists " + std::to_string(e.ids.size()) +
                             " ids, more than k_max = " + std::to_string(k_max));
        int32_t* row = set.chunk_indices(e.b, e.h, e.c);
        for (size_t i = 0; i < e.ids.size(); ++i) {
            if (e.ids[i] < 0 || e.ids[i] >= domain)
                throw IndexError("sparsity pattern: id " + std::to_string(e.ids[i]) +
                                 " is not in [0, " + std::to_string(domain) + ")");
            row[i] = static_cast<int32_t>(e.ids[i]);
        }
        set.counts[static_cast<size_t>((e.b * heads + e.h) * chunks + e.c)] =
            static_cast<int32_t>(e.ids.size());
    }
    set.validate();
    return set;
}

SparseIndexSet load_index_set_json_file(const std::string& path, int64_t batch, int64_t heads,
                                        int64_t chunks, int64_t domain) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("sparsity pattern file " + path + " cannot be opened");
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return load_index_set_json(text, batch, heads, chunks, domain);
}

// ====================================================================== attention (device)
namespace {
void check_qkv(const Tensor& q, const Tensor& k, const Tensor& v) {  // attention.cpp:11-21
    if (q.rank() != 4 || k.rank() != 4 || v.rank() != 4)
        throw ShapeError("attention expects [B x H x N x E] tensors, got q=" + shape_str(q.shape()) +
                         " k=" + shape_str(k.shape()) + " v=" + shape_str(v.shape()));
    if (q.shape() != k.shape() || q.shape() != v.shape())
        throw ShapeError("attention q/k/v shapes disagree: q=" + shape_str(q.shape()) + " k=" +
                         shape_str(k.shape()) + " v=" + shape_str(v.shape()));
}
void check_index_set(const SparseIndexSet& idx, const Tensor& q) {  // attention.cpp:46-55
    if (idx.batch != q.dim(0) || idx.heads != q.dim(1))
        throw ShapeError("sparse index set dims do not match q " + shape_str(q.shape()));
    if (idx.domain != q.dim(2) || idx.chunks * idx.chunk_size != q.dim(2))
        throw ShapeError("sparse index set chunking does not cover the sequence length " +
                         std::to_string(q.dim(2)));
}
}  // namespace

Tensor dense_attention(const Tensor& q, const Tensor& k, const Tensor& v) {
    check_qkv(q, k, v);
    Tensor out(q.shape());
    Dev dq(q), dk(k), dv(v), dout(sizeof(float) * q.numel());
    ok(csd_dense_attention(ctx(), CSD_MODE_CHECK, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(), q.dim(0),
                           q.dim(1), q.dim(2), q.dim(3), dout.v(), nullptr));
    dout.to(out);
    return out;
}
ColumnSumAttentionResult column_sum_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                                              const SoftmaxStats* prev, int64_t chunk) {
    check_qkv(q, k, v);
    const int64_t b = q.dim(0), h = q.dim(1), n = q.dim(2), e = q.dim(3);
    if (chunk < 1 || n % chunk)
        throw ShapeError("column_sum_attention: sequence length " + std::to_string(n) +
                         " not divisible by chunk " + std::to_string(chunk));
    if (prev && (prev->row_max.shape() != std::vector<int64_t>{b, h, n} ||
                 prev->exp_sum.shape() != std::vector<int64_t>{b, h, n}))
        throw ShapeError("column_sum_attention: previous stats shape " +
                         shape_str(prev->row_max.shape()) + " does not match");
    ColumnSumAttentionResult r{Tensor(q.shape()), Tensor({b, h, n / chunk, n}),
                               {Tensor({b, h, n}), Tensor({b, h, n})}};
    Dev dq(q), dk(k), dv(v), dout(sizeof(float) * q.numel()), dm(sizeof(float) * b * h * n),
        dl(sizeof(float) * b * h * n), dcs(sizeof(float) * r.column_sums.numel());
    Dev pm(prev ? prev->row_max : Tensor({1})), pl(prev ? prev->exp_sum : Tensor({1}));
    ok(csd_column_sum_attention(ctx(), CSD_MODE_CHECK, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(),
                                prev ? pm.f() : nullptr, prev ? pl.f() : nullptr, b, h, n, e, chunk,
                                dout.v(), dm.f(), dl.f(), dcs.f(), nullptr));
    dout.to(r.output);
    dcs.to(r.column_sums);
    dm.to(r.stats.row_max);
    dl.to(r.stats.exp_sum);
    return r;
}
Tensor sparse_delta_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                              const SparseIndexSet& idx, const Tensor& base, float scale) {
    check_qkv(q, k, v);
    if (base.shape() != q.shape())
        throw ShapeError("sparse_delta_attention: base shape " + shape_str(base.shape()) +
                         " does not match q " + shape_str(q.shape()));
    check_index_set(idx, q);
    Tensor out(q.shape());
    Dev dq(q), dk(k), dv(v), db(base), dout(sizeof(float) * q.numel());
    Dev di(idx.indices.empty() ? std::vector<int32_t>{0} : idx.indices), dc(idx.counts);
    ok(csd_sparse_delta_attention(ctx(), CSD_MODE_CHECK, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(),
                                  di.i(), dc.i(), idx.k_max, idx.chunk_size, db.v(), scale,
                                  q.dim(0), q.dim(1), q.dim(2), q.dim(3), dout.v(), nullptr));
    dout.to(out);
    return out;
}
Tensor attention_step(const Tensor& q, const Tensor& k, const Tensor& v, AttentionCache& cache,
                      bool dense_step, int64_t top_k, int64_t chunk,
                      const SparseIndexSet* static_indices) {  // attention.cpp:196-219
    if (!dense_step && !cache.initialized)
        throw StateError("sparse attention step requested before any dense step");
    if (dense_step) {
        auto res = column_sum_attention(q, k, v, cache.initialized ? &cache.stats : nullptr, chunk);
        SparseIndexSet idx = static_indices ? *static_indices : select_top_k(res.column_sums, top_k, chunk);
        check_index_set(idx, q);
        idx.validate();
        cache.residual_output = sparse_delta_attention(q, k, v, idx, res.output, -1.0f);
        cache.stats = std::move(res.stats);
        cache.indices = std::move(idx);
        cache.age = 0;
        cache.initialized = true;
        return res.output;
    }
    cache.age += 1;
    return sparse_delta_attention(q, k, v, cache.indices, cache.residual_output, 1.0f);
}

// ====================================================================== MLP (device)
void MlpWeights::validate() const {  // mlp.cpp:38-47
    if (w1.rank() != 2 || w2.rank() != 2 || b1.rank() != 1 || b2.rank() != 1)
        throw ShapeError("mlp weights must be w1 [F x D], b1 [F], w2 [F x D], b2 [D]");
    if (w2.shape() != w1.shape() || b1.dim(0) != w1.dim(0) || b2.dim(0) != w1.dim(1))
        throw ShapeError("mlp weight shapes disagree: w1=" + shape_str(w1.shape()) + " w2=" +
                         shape_str(w2.shape()));
}
namespace {
void check_x(const Tensor& x, const MlpWeights& w) {  // mlp.cpp:26-34
    if (x.rank() != 3) throw ShapeError("mlp expects [B x N x D] input, got " + shape_str(x.shape()));
    if (x.dim(2) != w.model_dim())
        throw ShapeError("mlp input dim " + std::to_string(x.dim(2)) +
                         " does not match weights' model dim " + std::to_string(w.model_dim()));
}
}  // namespace

MlpDenseResult dense_mlp(const Tensor& x, const MlpWeights& w) {
    w.validate();
    check_x(x, w);
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w.hidden();
    MlpDenseResult r{Tensor({b, n, d}), Tensor({b, n, f}), Tensor({b, n, f})};
    Dev dx(x), d1(w.w1), db1(w.b1), d2(w.w2), db2(w.b2), dout(sizeof(float) * b * n * d),
        dact(sizeof(float) * b * n * f), dpre(sizeof(float) * b * n * f);
    ok(csd_dense_mlp(ctx(), CSD_MODE_CHECK, dx.v(), d1.v(), db1.f(), d2.v(), db2.f(), b, n, d, f, n,
                     dout.f(), dact.v(), nullptr));
    ok(csd_mlp_preact(ctx(), CSD_MODE_CHECK, dx.v(), d1.v(), db1.f(), b, n, d, f, dpre.f(), nullptr));
    dout.to(r.output);
    dact.to(r.act);
    dpre.to(r.preact);
    return r;
}
Tensor mlp_tile_means(const Tensor& x, const Tensor& w1, int64_t chunk) {
    if (x.rank() != 3) throw ShapeError("mlp_tile_means expects [B x N x D] input, got " + shape_str(x.shape()));
    if (w1.rank() != 2 || w1.dim(1) != x.dim(2))
        throw ShapeError("gemm inner dimensions disagree: " + shape_str(x.shape()) + " @ " +
                         shape_str(w1.shape()) + " (b transposed)");
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w1.dim(0);
    if (chunk < 1 || n % chunk)
        throw ShapeError("chunk_reduce: row count " + std::to_string(n) + " not divisible by chunk " +
                         std::to_string(chunk));
    Tensor out({b, n / chunk, f});
    Dev dx(x), d1(w1), dout(sizeof(float) * out.numel());
    ok(csd_mlp_tile_means(ctx(), CSD_MODE_CHECK, dx.v(), d1.v(), b, n, d, f, chunk, dout.f(), nullptr));
    dout.to(out);
    return out;
}
SparseIndexSet mlp_change_indices(const Tensor& x, const Tensor& w1, const Tensor& tile_means,
                                  int64_t k, int64_t chunk) {  // mlp.cpp:98-118
    if (x.rank() != 3) throw ShapeError("mlp_tile_means expects [B x N x D] input, got " + shape_str(x.shape()));
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w1.dim(0);
    if (chunk < 1 || n % chunk)
        throw ShapeError("chunk_reduce: row count " + std::to_string(n) + " not divisible by chunk " +
                         std::to_string(chunk));
    if (tile_means.shape() != std::vector<int64_t>{b, n / chunk, f})
        throw ShapeError("mlp_change_indices: cached tile means " + shape_str(tile_means.shape()) +
                         " do not match fresh");
    if (k < 1 || k > f)
        throw ValueError("mlp_change_indices: k=" + std::to_string(k) + " outside [1, " + std::to_string(f) + "]");
    SparseIndexSet s = SparseIndexSet::empty(b, 1, n / chunk, chunk, k, f);
    Dev dx(x), d1(w1), dtm(tile_means), di(sizeof(int32_t) * s.indices.size()),
        dc(sizeof(int32_t) * s.counts.size());
    ok(csd_mlp_change_indices(ctx(), CSD_MODE_CHECK, dx.v(), d1.v(), dtm.f(), b, n, d, f, k, chunk,
                              di.i(), dc.i(), nullptr));
    di.to(s.indices);
    dc.to(s.counts);
    return s;
}
Tensor sparse_delta_mlp(const Tensor& x, const MlpWeights& w, const SparseIndexSet& idx,
                        MlpCache& cache) {  // mlp.cpp:120-182
    w.validate();
    check_x(x, w);
    if (!cache.initialized) throw StateError("sparse MLP step requested before any dense step");
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w.hidden();
    if (idx.batch != b || idx.heads != 1 || idx.domain != f || idx.chunks * idx.chunk_size != n)
        throw ShapeError("mlp sparse index set does not match (B=" + std::to_string(b) + ", N=" +
                         std::to_string(n) + ", F=" + std::to_string(f) + ")");
    Dev dx(x), d1(w.w1), db1(w.b1), d2(w.w2), dact(cache.activations), dout(cache.outputs);
    Dev di(idx.indices.empty() ? std::vector<int32_t>{0} : idx.indices), dc(idx.counts);
    ok(csd_sparse_delta_mlp(ctx(), CSD_MODE_CHECK, dx.v(), d1.v(), db1.f(), d2.v(), di.i(), dc.i(),
                            idx.k_max, idx.chunk_size, b, n, d, f, dact.v(), dout.f(), nullptr));
    dact.to(cache.activations);
    dout.to(cache.outputs);
    return cache.outputs;
}
Tensor mlp_step(const Tensor& x, const MlpWeights& w, MlpCache& cache, bool dense_step,
                int64_t top_k, int64_t chunk) {  // mlp.cpp:184-211
    if (!dense_step && !cache.initialized) throw StateError("sparse MLP step requested before any dense step");
    if (x.rank() != 3) throw ShapeError("mlp_step expects [B x N x D] input, got " + shape_str(x.shape()));
    if (chunk < 1 || x.dim(1) % chunk)
        throw ShapeError("mlp_step: sequence length " + std::to_string(x.dim(1)) +
                         " not divisible by chunk " + std::to_string(chunk));
    if (dense_step) {
        auto res = dense_mlp(x, w);
        cache.tile_means = mlp_tile_means(x, w.w1, chunk);
        cache.activations = std::move(res.act);
        cache.outputs = res.output;
        cache.indices = SparseIndexSet{};
        cache.age = 0;
        cache.initialized = true;
        return res.output;
    }
    SparseIndexSet idx = mlp_change_indices(x, w.w1, cache.tile_means, top_k, chunk);
    cache.age += 1;
    Tensor out = sparse_delta_mlp(x, w, idx, cache);
    cache.indices = std::move(idx);
    return out;
}


// ====================================================================== block stack
// model.cpp:10-216.  Projections run on the device (csd_project, CHECK mode: the
// reference's sequential-k fp32 gemm); attention_step / mlp_step are the device-backed
// routines above; head split/merge and the residual add are host data movement / fp32 adds.
// ModelConfig (model.hpp:16-41) consistency, the model.cpp:10-28 contract: every ConfigError
// case of the reference, checked as a list of (holds, message) rules in order.
void ModelConfig::validate() const {
    const int64_t dims[] = {batch, grid_t, grid_h, grid_w, model_dim, head_dim, heads, mlp_hidden,
                            chunk};
    const bool positive = std::all_of(std::begin(dims), std::end(dims), [](int64_t v) { return v > 0; });
    const int64_t vol = voxel_t * voxel_h * voxel_w;
    const struct {
        bool ok;
        std::string msg;
    } rules[] = {
        {positive && layers >= 0,
         "model config: batch, grid, dims, heads, hidden and chunk must be >= 1 (layers >= 0)"},
        {model_dim == heads * head_dim,
         "model config: model_dim = " + std::to_string(model_dim) + " but heads x head_dim = " +
             std::to_string(heads * head_dim)},
        {positive && seq_len() % chunk == 0,
         "model config: chunk " + std::to_string(chunk) + " does not divide the sequence length " +
             std::to_string(seq_len())},
        {vol == chunk, "model config: voxel volume " + std::to_string(vol) +
                           " differs from the chunk size " + std::to_string(chunk)},
    };
    for (const auto& r : rules)
        if (!r.ok) throw ConfigError(r.msg);
    voxel_layout().validate();
}

namespace {
Tensor draw(GaussianRng& rng, std::vector<int64_t> shape, float stddev) {
    Tensor t(std::move(shape));
    for (int64_t i = 0; i < t.numel(); ++i) t[i] = rng.next(0.0f, stddev);
    return t;
}
Tensor residual_add(const Tensor& a, const Tensor& b) {  // model.cpp:47-57
    if (a.shape() != b.shape())
        throw ShapeError("residual add shapes disagree: " + shape_str(a.shape()) + " vs " +
                         shape_str(b.shape()));
    Tensor out = a;
    for (int64_t i = 0; i < out.numel(); ++i) out[i] += b[i];
    return out;
}
struct Qkv {
    Tensor q, k, v;
};
Qkv project_qkv(const LayerWeights& lw, const Tensor& x, int64_t heads, int64_t head_dim) {
    return {split_heads(project(x, lw.wq), heads, head_dim),
            split_heads(project(x, lw.wk), heads, head_dim),
            split_heads(project(x, lw.wv), heads, head_dim)};
}
}  // namespace

ToyModel build_toy_model(const ModelConfig& cfg) {  // model.cpp:79-99 (draw order, 0.5 gain)
    cfg.validate();
    ToyModel m;
    m.cfg = cfg;
    GaussianRng rng(cfg.seed);
    const float s = 1.0f / std::sqrt(static_cast<float>(cfg.model_dim)), so = 0.5f * s;
    const int64_t d = cfg.model_dim, f = cfg.mlp_hidden;
    for (int64_t l = 0; l < cfg.layers; ++l) {
        LayerWeights lw;
        lw.wq = draw(rng, {d, d}, s);
        lw.wk = draw(rng, {d, d}, s);
        lw.wv = draw(rng, {d, d}, s);
        lw.wo = draw(rng, {d, d}, so);
        lw.mlp.w1 = draw(rng, {f, d}, s);
        lw.mlp.b1 = draw(rng, {f}, s);
        lw.mlp.w2 = draw(rng, {f, d}, so);
        lw.mlp.b2 = draw(rng, {d}, so);
        m.layers.push_back(std::move(lw));
    }
    return m;
}

ModelState make_state(const ToyModel& model) {
    ModelState st;
    st.layers.resize(model.layers.size());
    return st;
}

Tensor project(const Tensor& x, const Tensor& w) {  // model.cpp:107-120
    if (x.rank() != 3) throw ShapeError("project expects [B x N x D] input, got " + shape_str(x.shape()));
    if (w.rank() != 2 || w.dim(0) != x.dim(2))
        throw ShapeError("gemm inner dimensions disagree: " + shape_str({x.dim(1), x.dim(2)}) +
                         " @ " + shape_str(w.shape()));
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), dout = w.dim(1);
    Tensor out({b, n, dout});
    Dev dx(x), dw(w), dout_(sizeof(float) * out.numel());
    ok(csd_project(ctx(), CSD_MODE_CHECK, dx.v(), dw.v(), b, n, d, dout, dout_.v(), nullptr));
    dout_.to(out);
    return out;
}

Tensor split_heads(const Tensor& x, int64_t heads, int64_t head_dim) {  // model.cpp:122-143
    if (x.rank() != 3 || x.dim(2) != heads * head_dim)
        throw ShapeError("split_heads: input " + shape_str(x.shape()) + " does not factor into " +
                         std::to_string(heads) + " heads of dim " + std::to_string(head_dim));
    const int64_t b = x.dim(0), n = x.dim(1);
    Tensor out({b, heads, n, head_dim});
    for (int64_t bb = 0; bb < b; ++bb)
        for (int64_t h = 0; h < heads; ++h)
            for (int64_t t = 0; t < n; ++t)
                std::memcpy(out.data() + ((bb * heads + h) * n + t) * head_dim,
                            x.data() + ((bb * n + t) * heads + h) * head_dim, sizeof(float) * head_dim);
    return out;
}

Tensor merge_heads(const Tensor& x) {  // model.cpp:145-165
    if (x.rank() != 4) throw ShapeError("merge_heads expects [B x H x N x E], got " + shape_str(x.shape()));
    const int64_t b = x.dim(0), heads = x.dim(1), n = x.dim(2), e = x.dim(3);
    Tensor out({b, n, heads * e});
    for (int64_t bb = 0; bb < b; ++bb)
        for (int64_t h = 0; h < heads; ++h)
            for (int64_t t = 0; t < n; ++t)
                std::memcpy(out.data() + ((bb * n + t) * heads + h) * e,
                            x.data() + ((bb * heads + h) * n + t) * e, sizeof(float) * e);
    return out;
}

Tensor model_forward_dense(const ToyModel& model, const Tensor& x) {  // model.cpp:167-176
    Tensor cur = x;
    for (const auto& lw : model.layers) {
        const Qkv p = project_qkv(lw, cur, model.cfg.heads, model.cfg.head_dim);
        cur = residual_add(cur, project(merge_heads(dense_attention(p.q, p.k, p.v)), lw.wo));
        cur = residual_add(cur, dense_mlp(cur, lw.mlp).output);
    }
    return cur;
}

Tensor model_forward_step(const ToyModel& model, ModelState& state, const Tensor& x,
                          bool dense_step, const SparsityConfig& sparsity, LayerProbe* probe,
                          const SparseIndexSet* static_attn) {  // model.cpp:178-216
    if (state.layers.size() != model.layers.size())
        throw StateError("model state layer count does not match the model");
    Tensor cur = x;
    for (size_t l = 0; l < model.layers.size(); ++l) {
        const auto& lw = model.layers[l];
        LayerState& ls = state.layers[l];
        const Qkv p = project_qkv(lw, cur, model.cfg.heads, model.cfg.head_dim);
        const Tensor a = attention_step(p.q, p.k, p.v, ls.attn, dense_step, sparsity.attn_k,
                                        model.cfg.chunk, static_attn);
        if (probe)
            probe->attention_sample(static_cast<int64_t>(l), dense_step,
                                    dense_step ? a : dense_attention(p.q, p.k, p.v), a);
        cur = residual_add(cur, project(merge_heads(a), lw.wo));
        const Tensor mlp_in = cur;
        const Tensor m = mlp_step(mlp_in, lw.mlp, ls.mlp, dense_step, sparsity.mlp_k, model.cfg.chunk);
        if (probe)
            probe->mlp_sample(static_cast<int64_t>(l), dense_step,
                              dense_step ? m : dense_mlp(mlp_in, lw.mlp).output, m);
        cur = residual_add(cur, m);
    }
    return cur;
}

}  // namespace csd

// ====================================================================== production route
// include/csd/device.hpp: the same operations on the PROD (bf16 / tcgen05) kernels.
#include "csd/device.hpp"

namespace csd {
namespace dev {
namespace {

// a bf16 device copy of a host fp32 tensor (round to nearest even on the device)
class Bf16 {
public:
    explicit Bf16(const Tensor& t) : d_(2 * static_cast<size_t>(t.numel())) {
        Dev f(t);
        ok(csd_cast(ctx(), f.v(), d_.v(), t.numel(), 1, nullptr));
    }
    explicit Bf16(int64_t numel) : d_(2 * static_cast<size_t>(numel)) {}
    void* v() const { return d_.v(); }

private:
    Dev d_;
};

Tensor from_bf16(const void* dev_bf16, std::vector<int64_t> shape) {
    Tensor out(std::move(shape));
    Dev f(sizeof(float) * static_cast<size_t>(out.numel()));
    ok(csd_cast(ctx(), dev_bf16, f.v(), out.numel(), 0, nullptr));
    f.to(out);
    return out;
}

}  // namespace

Tensor dense_attention(const Tensor& q, const Tensor& k, const Tensor& v) {  // attention.cpp:59-74
    check_qkv(q, k, v);
    Bf16 dq(q), dk(k), dv(v), out(q.numel());
    ok(csd_dense_attention(ctx(), CSD_MODE_PROD, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(), q.dim(0),
                           q.dim(1), q.dim(2), q.dim(3), out.v(), nullptr));
    sync();
    return from_bf16(out.v(), q.shape());
}

ColumnSumAttentionResult column_sum_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                                              const SoftmaxStats* prev, int64_t chunk) {  // :76-145
    check_qkv(q, k, v);
    const int64_t b = q.dim(0), h = q.dim(1), n = q.dim(2), e = q.dim(3);
    if (chunk < 1 || n % chunk)
        throw ShapeError("column_sum_attention: sequence length " + std::to_string(n) +
                         " not divisible by chunk " + std::to_string(chunk));
    if (prev && (prev->row_max.shape() != std::vector<int64_t>{b, h, n} ||
                 prev->exp_sum.shape() != std::vector<int64_t>{b, h, n}))
        throw ShapeError("column_sum_attention: previous stats shape does not match");
    Bf16 dq(q), dk(k), dv(v), out(q.numel());
    ColumnSumAttentionResult r;
    r.stats.row_max = Tensor({b, h, n});
    r.stats.exp_sum = Tensor({b, h, n});
    r.column_sums = Tensor({b, h, n / chunk, n});
    Dev m(sizeof(float) * b * h * n), l(sizeof(float) * b * h * n), cs(sizeof(float) * r.column_sums.numel());
    std::unique_ptr<Dev> pm, pl;
    if (prev) {
        pm = std::make_unique<Dev>(prev->row_max);
        pl = std::make_unique<Dev>(prev->exp_sum);
    }
    ok(csd_column_sum_attention(ctx(), CSD_MODE_PROD, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(),
                                pm ? pm->f() : nullptr, pl ? pl->f() : nullptr, b, h, n, e, chunk,
                                out.v(), m.f(), l.f(), cs.f(), nullptr));
    sync();
    r.output = from_bf16(out.v(), q.shape());
    m.to(r.stats.row_max);
    l.to(r.stats.exp_sum);
    cs.to(r.column_sums);
    return r;
}

Tensor sparse_delta_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                              const SparseIndexSet& idx, const Tensor& base, float scale) {  // :147-194
    check_qkv(q, k, v);
    check_index_set(idx, q);
    if (base.shape() != q.shape())
        throw ShapeError("sparse_delta_attention: base " + shape_str(base.shape()) +
                         " does not match q " + shape_str(q.shape()));
    Bf16 dq(q), dk(k), dv(v), db(base), out(q.numel());
    Dev di(idx.indices), dc(idx.counts);
    ok(csd_sparse_delta_attention(ctx(), CSD_MODE_PROD, CSD_LAYOUT_BHNE, dq.v(), dk.v(), dv.v(),
                                  di.i(), dc.i(), idx.k_max, idx.chunk_size, db.v(), scale, q.dim(0),
                                  q.dim(1), q.dim(2), q.dim(3), out.v(), nullptr));
    sync();  // surfaces the on-device index validation as IndexError / ValueError
    return from_bf16(out.v(), q.shape());
}

MlpDenseResult dense_mlp(const Tensor& x, const MlpWeights& w, int64_t chunk) {  // mlp.cpp:49-81
    check_x(x, w);
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w.w1.dim(0);
    if (chunk < 1 || n % chunk)
        throw ShapeError("dense_mlp: sequence length " + std::to_string(n) + " not divisible by chunk " +
                         std::to_string(chunk));
    Bf16 dx(x), dw1(w.w1), dw2(w.w2), act(b * n * f);
    Dev db1(w.b1), db2(w.b2), out(sizeof(float) * b * n * d), aref(sizeof(float) * b * n * f);
    ok(csd_dense_mlp(ctx(), CSD_MODE_PROD, dx.v(), dw1.v(), db1.f(), dw2.v(), db2.f(), b, n, d, f,
                     chunk, out.f(), act.v(), nullptr));
    ok(csd_mlp_act_cache_to_ref(ctx(), CSD_MODE_PROD, act.v(), b, n, f, chunk, aref.f(), nullptr));
    sync();
    MlpDenseResult r;
    r.output = Tensor({b, n, d});
    r.act = Tensor({b, n, f});
    out.to(r.output);
    aref.to(r.act);
    return r;  // preact stays empty: the fused GEMM never materialises x W1^T + b1
}

Tensor mlp_tile_means(const Tensor& x, const Tensor& w1, int64_t chunk) {  // mlp.cpp:83-96
    if (x.rank() != 3 || w1.rank() != 2 || w1.dim(1) != x.dim(2))
        throw ShapeError("mlp_tile_means: x " + shape_str(x.shape()) + " and w1 " + shape_str(w1.shape()) +
                         " disagree");
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w1.dim(0);
    if (chunk < 1 || n % chunk)
        throw ShapeError("mlp_tile_means: sequence length not divisible by chunk");
    Bf16 dx(x), dw1(w1);
    Tensor out({b, n / chunk, f});
    Dev dout(sizeof(float) * out.numel());
    ok(csd_mlp_tile_means(ctx(), CSD_MODE_PROD, dx.v(), dw1.v(), b, n, d, f, chunk, dout.f(), nullptr));
    sync();
    dout.to(out);
    return out;
}

SparseIndexSet mlp_change_indices(const Tensor& x, const Tensor& w1, const Tensor& tile_means,
                                  int64_t k, int64_t chunk) {  // mlp.cpp:98-118
    if (x.rank() != 3 || w1.rank() != 2 || w1.dim(1) != x.dim(2))
        throw ShapeError("mlp_change_indices: x " + shape_str(x.shape()) + " and w1 " +
                         shape_str(w1.shape()) + " disagree");
    const int64_t b = x.dim(0), n = x.dim(1), d = x.dim(2), f = w1.dim(0);
    if (chunk < 1 || n % chunk) throw ShapeError("mlp_change_indices: sequence length not divisible by chunk");
    if (tile_means.shape() != std::vector<int64_t>{b, n / chunk, f})
        throw ShapeError("mlp_change_indices: tile means " + shape_str(tile_means.shape()) +
                         " do not match the input");
    if (k < 0 || k > f) throw ValueError("mlp_change_indices: k " + std::to_string(k) + " outside [0, F]");
    Bf16 dx(x), dw1(w1);
    Dev dtm(tile_means);
    SparseIndexSet s = SparseIndexSet::empty(b, 1, n / chunk, chunk, k, f);
    Dev di(sizeof(int32_t) * s.indices.size()), dc(sizeof(int32_t) * s.counts.size());
    ok(csd_mlp_change_indices(ctx(), CSD_MODE_PROD, dx.v(), dw1.v(), dtm.f(), b, n, d, f, k, chunk,
                              di.i(), dc.i(), nullptr));
    sync();
    di.to(s.indices);
    dc.to(s.counts);
    return s;
}

// ---------------------------------------------------------------- DeviceModel
DeviceModel::DeviceModel(const ToyModel& model, const SparsityConfig& sparsity)
    : cfg_(model.cfg), sparsity_(sparsity) {
    cfg_.validate();
    csd_block_config c{};
    c.batch = cfg_.batch;
    c.seq = cfg_.seq_len();
    c.dim = cfg_.model_dim;
    c.heads = cfg_.heads;
    c.head_dim = cfg_.head_dim;
    c.hidden = cfg_.mlp_hidden;
    c.chunk = cfg_.chunk;
    c.attn_k = sparsity.attn_k;
    c.mlp_k = sparsity.mlp_k;
    for (const auto& lw : model.layers) {
        csd_block* blk = nullptr;
        const csd_status s =
            csd_block_create(ctx(), CSD_MODE_PROD, &c, lw.wq.data(), lw.wk.data(), lw.wv.data(),
                             lw.wo.data(), lw.mlp.w1.data(), lw.mlp.b1.data(), lw.mlp.w2.data(),
                             lw.mlp.b2.data(), &blk);
        if (s != CSD_OK) {
            for (void* b : blocks_) csd_block_destroy(static_cast<csd_block*>(b));
            blocks_.clear();
            rethrow(s);
        }
        blocks_.push_back(blk);
    }
    const size_t elems = static_cast<size_t>(c.batch * c.seq * c.dim);
    ok(csd_device_alloc(2 * elems, &buf_[0]));
    ok(csd_device_alloc(2 * elems, &buf_[1]));
    ok(csd_device_alloc(4 * elems, &io_));
}

DeviceModel::~DeviceModel() {
    for (void* b : blocks_) csd_block_destroy(static_cast<csd_block*>(b));
    csd_device_free(buf_[0]);
    csd_device_free(buf_[1]);
    csd_device_free(io_);
}

void DeviceModel::reset() {
    for (void* b : blocks_) ok(csd_block_reset(static_cast<csd_block*>(b)));
}

void DeviceModel::forward_step_device(const void* x_bf16, void* y_bf16, bool dense_step, void* stream) {
    // layer l reads the previous layer's output; the last one writes y
    const void* in = x_bf16;
    for (size_t l = 0; l < blocks_.size(); ++l) {
        void* out = l + 1 == blocks_.size() ? y_bf16 : buf_[l & 1];
        ok(csd_block_step(static_cast<csd_block*>(blocks_[l]), in, out, dense_step ? 1 : 0, nullptr,
                          nullptr, 0, stream));
        in = out;
    }
    if (blocks_.empty()) {  // a zero-layer model is the identity (model.cpp:184-186)
        const size_t bytes = 2 * static_cast<size_t>(cfg_.batch * cfg_.seq_len() * cfg_.model_dim);
        std::vector<char> tmp(bytes);
        ok(csd_copy_to_host(tmp.data(), x_bf16, bytes));
        ok(csd_copy_to_device(y_bf16, tmp.data(), bytes));
    }
}

Tensor DeviceModel::forward_step(const Tensor& x, bool dense_step, const SparseIndexSet* static_attn) {
    const int64_t b = cfg_.batch, n = cfg_.seq_len(), d = cfg_.model_dim;
    if (x.shape() != std::vector<int64_t>{b, n, d})
        throw ShapeError("model_forward_step: input " + shape_str(x.shape()) + " does not match the model");
    ok(csd_copy_to_device(io_, x.data(), sizeof(float) * x.numel()));
    ok(csd_cast(ctx(), io_, buf_[0], x.numel(), 1, nullptr));
    std::unique_ptr<Dev> si, sc;
    if (static_attn) {
        si = std::make_unique<Dev>(static_attn->indices);
        sc = std::make_unique<Dev>(static_attn->counts);
    }
    // ping-pong through the two bf16 buffers (buf_[0] holds x)
    int cur = 0;
    for (void* bp : blocks_) {
        ok(csd_block_step(static_cast<csd_block*>(bp), buf_[cur], buf_[1 - cur], dense_step ? 1 : 0,
                          si ? si->i() : nullptr, sc ? sc->i() : nullptr,
                          static_attn ? static_attn->k_max : 0, nullptr));
        cur = 1 - cur;
    }
    sync();
    return from_bf16(buf_[cur], x.shape());
}

}  // namespace dev
}  // namespace csd
