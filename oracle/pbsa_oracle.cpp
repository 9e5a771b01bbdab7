// pbsa_oracle.cpp -- CPU ORACLE (test infrastructure only; see pbsa_oracle.h header comment).
//
// A restatement of the reference's algorithm for the PBSA hot path:
//   * numeric primitives restated from /root/reference/proj/src/tensor.cpp and blockify.cpp and
//     /root/reference/proj/include/pbsa/rng.hpp (checked bit-exactly against the compiled
//     reference sources by tests/test_oracle_vs_ref.py);
//   * SPEC-only ops restated from /root/reference/SPEC.md (the reference ships no code for them).
// Never linked into the product library.

#include "pbsa_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

int fail(const std::string& msg) {
    g_err = msg;
    return 1;
}

constexpr float kNegInf = -std::numeric_limits<float>::infinity();

// rng.hpp:11-57 -- splitmix64 core, 53-bit uniforms, Box-Muller with a cached spare.
struct Rng {
    uint64_t state;
    bool have_spare = false;
    float spare = 0.0f;
    explicit Rng(uint64_t s) : state(s) {}
    uint64_t next_u64() {  // rng.hpp:15-20
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }  // rng.hpp:23
    float normal() {  // rng.hpp:32-45: returns the cos branch, caches the sin branch
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.14159265358979323846 * u2;
        spare = static_cast<float>(r * std::sin(theta));
        have_spare = true;
        return static_cast<float>(r * std::cos(theta));
    }
};

// ascending-k fp64 dot of two fp32 rows (tensor.cpp:45-52).  The products of two floats are
// exact in double, so FMA contraction cannot change the result.
inline double dot64(const float* a, const float* b, int64_t n) {
    double acc = 0.0;
    for (int64_t k = 0; k < n; ++k) acc += static_cast<double>(a[k]) * static_cast<double>(b[k]);
    return acc;
}

// masked_softmax_rows for one row (tensor.cpp:82-106): fp32 max over visible entries, fp64
// exp(s - max) and ascending-j fp64 denominator, fp32 output; fully masked row -> zeros.
void softmax_row(const float* srow, const float* mrow, int64_t m, float* orow,
                 std::vector<double>& e) {
    float row_max = kNegInf;
    for (int64_t j = 0; j < m; ++j) {
        const float s = (mrow != nullptr && mrow[j] == kNegInf) ? kNegInf : srow[j];
        if (s > row_max) row_max = s;
    }
    if (row_max == kNegInf) {
        for (int64_t j = 0; j < m; ++j) orow[j] = 0.0f;
        return;
    }
    e.assign(static_cast<size_t>(m), 0.0);
    double denom = 0.0;
    for (int64_t j = 0; j < m; ++j) {
        if (mrow != nullptr && mrow[j] == kNegInf) {
            e[j] = 0.0;
        } else {
            e[j] = std::exp(static_cast<double>(srow[j]) - static_cast<double>(row_max));
            denom += e[j];
        }
    }
    for (int64_t j = 0; j < m; ++j) orow[j] = static_cast<float>(e[j] / denom);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_rng_normal(uint64_t seed, int64_t n, float* out) {
    if (n < 0 || (n > 0 && out == nullptr)) return fail("orc_rng_normal: bad arguments");
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
    return 0;
}

int orc_rng_uniform(uint64_t seed, int64_t n, double* out) {
    if (n < 0 || (n > 0 && out == nullptr)) return fail("orc_rng_uniform: bad arguments");
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
    return 0;
}

uint64_t orc_rng_derive(uint64_t seed, uint64_t stream) {  // rng.hpp:48-51
    Rng r(seed ^ (0xd1b54a32d192ed03ULL * (stream + 1)));
    return r.next_u64();
}

int orc_matmul_nt(const float* a, int64_t ar, int64_t ac, const float* b, int64_t br, float* out) {
    if (ar < 0 || ac < 0 || br < 0) return fail("matmul_nt: negative dims");
#pragma omp parallel for schedule(static) if (ar > 8)
    for (int64_t i = 0; i < ar; ++i) {
        const float* arow = a + i * ac;
        float* crow = out + i * br;
        for (int64_t j = 0; j < br; ++j) crow[j] = static_cast<float>(dot64(arow, b + j * ac, ac));
    }
    return 0;
}

int orc_matmul(const float* a, int64_t ar, int64_t ac, const float* b, int64_t bc, float* out) {
    if (ar < 0 || ac < 0 || bc < 0) return fail("matmul: negative dims");
#pragma omp parallel for schedule(static) if (ar > 8)
    for (int64_t i = 0; i < ar; ++i) {
        std::vector<double> acc(static_cast<size_t>(bc), 0.0);
        const float* arow = a + i * ac;
        for (int64_t k = 0; k < ac; ++k) {
            const double av = arow[k];
            const float* brow = b + k * bc;
            for (int64_t j = 0; j < bc; ++j) acc[j] += av * static_cast<double>(brow[j]);
        }
        float* crow = out + i * bc;
        for (int64_t j = 0; j < bc; ++j) crow[j] = static_cast<float>(acc[j]);
    }
    return 0;
}

int orc_masked_softmax_rows(const float* scores, int64_t rows, int64_t cols, const float* mask,
                            float* out) {
    const int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i)
        if (std::isnan(scores[i])) return fail("masked_softmax_rows: NaN in scores");
    if (mask != nullptr)
        for (int64_t i = 0; i < n; ++i)
            if (!(mask[i] == 0.0f || mask[i] == kNegInf))
                return fail("masked_softmax_rows: mask entries must be 0 or -inf");
#pragma omp parallel for schedule(static) if (rows > 8)
    for (int64_t i = 0; i < rows; ++i) {
        std::vector<double> e;
        softmax_row(scores + i * cols, mask ? mask + i * cols : nullptr, cols, out + i * cols, e);
    }
    return 0;
}

static int check_layout(int64_t t, int64_t h, int64_t w, int64_t bt, int64_t bh, int64_t bw) {
    if (bt <= 0 || bh <= 0 || bw <= 0) return fail("block shape extents must be >= 1");
    if (t % bt) return fail("axis t (" + std::to_string(t) + ") not divisible by b_t (" + std::to_string(bt) + ")");
    if (h % bh) return fail("axis h (" + std::to_string(h) + ") not divisible by b_h (" + std::to_string(bh) + ")");
    if (w % bw) return fail("axis w (" + std::to_string(w) + ") not divisible by b_w (" + std::to_string(bw) + ")");
    return 0;
}

// blockify.cpp:38-65 restated as a gather over destination tokens.
static int permute_blocks(const float* src, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                          int64_t bh, int64_t bw, float* dst, bool forward) {
    if (check_layout(t, h, w, bt, bh, bw)) return 1;
    const int64_t nh = h / bh, nw = w / bw, b = bt * bh * bw;
    const int64_t nb = (t / bt) * nh * nw;
#pragma omp parallel for schedule(static) if (nb > 4)
    for (int64_t bid = 0; bid < nb; ++bid) {
        const int64_t it = bid / (nh * nw), ih = (bid / nw) % nh, iw = bid % nw;
        for (int64_t off = 0; off < b; ++off) {
            const int64_t dt = off / (bh * bw), dh = (off / bw) % bh, dw = off % bw;
            const int64_t src_tok = ((it * bt + dt) * h + (ih * bh + dh)) * w + (iw * bw + dw);
            const int64_t blk_tok = bid * b + off;
            if (forward)
                std::memcpy(dst + blk_tok * d, src + src_tok * d, sizeof(float) * d);
            else
                std::memcpy(dst + src_tok * d, src + blk_tok * d, sizeof(float) * d);
        }
    }
    return 0;
}

int orc_blockify(const float* x, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                 int64_t bh, int64_t bw, float* out) {
    return permute_blocks(x, t, h, w, d, bt, bh, bw, out, true);
}

int orc_unblockify(const float* xb, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                   int64_t bh, int64_t bw, float* out) {
    return permute_blocks(xb, t, h, w, d, bt, bh, bw, out, false);
}

int orc_block_index_map(int64_t t, int64_t h, int64_t w, int64_t bt, int64_t bh, int64_t bw,
                        int64_t flat, int64_t* block_id, int64_t* in_block) {
    if (check_layout(t, h, w, bt, bh, bw)) return 1;
    if (flat < 0 || flat >= t * h * w)
        return fail("flat source index " + std::to_string(flat) + " out of range");
    const int64_t ti = flat / (h * w), hi = (flat / w) % h, wi = flat % w;
    *block_id = ((ti / bt) * (h / bh) + hi / bh) * (w / bw) + wi / bw;
    *in_block = ((ti % bt) * bh + hi % bh) * bw + wi % bw;
    return 0;
}

int orc_compress_blocks(const float* x, int64_t n_blocks, int64_t b, int64_t d, float* reps) {
    if (n_blocks < 0 || b <= 0 || d <= 0) return fail("compress_blocks: bad geometry");
#pragma omp parallel for schedule(static) if (n_blocks > 8)
    for (int64_t j = 0; j < n_blocks; ++j) {
        const float* blk = x + j * b * d;
        for (int64_t c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int64_t t = 0; t < b; ++t) acc += static_cast<double>(blk[t * d + c]);
            reps[j * d + c] = static_cast<float>(acc / static_cast<double>(b));
        }
    }
    return 0;
}

float orc_attention_scale(int64_t d) {
    return static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
}

int orc_coarse_logits(const float* qc, int64_t nq, const float* kc, int64_t nk, int64_t d,
                      float scale, float* logits) {
    if (orc_matmul_nt(qc, nq, d, kc, nk, logits)) return 1;
    const int64_t n = nq * nk;
    for (int64_t i = 0; i < n; ++i) logits[i] = logits[i] * scale;
    return 0;
}

int orc_coarse_attention(const float* qc, int64_t nq, const float* kc, int64_t nk, int64_t d,
                         float scale, float* probs) {
    if (nk <= 0) return fail("coarse_attention: no key blocks");
    std::vector<float> logits(static_cast<size_t>(nq * nk));
    if (orc_coarse_logits(qc, nq, kc, nk, d, scale, logits.data())) return 1;
    return orc_masked_softmax_rows(logits.data(), nq, nk, nullptr, probs);
}

int orc_aggregate_scores(const float* a, int64_t rows, int64_t cols, float* s) {
    if (rows <= 0) return fail("aggregate_scores: no rows");
    for (int64_t j = 0; j < cols; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < rows; ++i) acc += static_cast<double>(a[i * cols + j]);
        s[j] = static_cast<float>(acc / static_cast<double>(rows));
    }
    return 0;
}

int orc_topk_count(int64_t n_local, double ratio, int64_t* k) {
    if (n_local < 1) return fail("select_topk: empty local region");
    if (!(ratio > 0.0 && ratio <= 1.0)) return fail("select_topk: topk_ratio must be in (0,1]");
    int64_t kk = static_cast<int64_t>(std::ceil(static_cast<double>(n_local) * ratio));
    *k = std::min<int64_t>(n_local, std::max<int64_t>(1, kk));
    return 0;
}

int orc_select_topk(const float* a, int64_t rows, int64_t cols, int64_t k, int32_t* sel) {
    if (cols < 1) return fail("select_topk: empty local region");
    if (k < 1 || k > cols) return fail("select_topk: k out of range");
#pragma omp parallel for schedule(static) if (rows > 8)
    for (int64_t i = 0; i < rows; ++i) {
        const float* row = a + i * cols;
        std::vector<int32_t> idx(static_cast<size_t>(cols));
        for (int64_t j = 0; j < cols; ++j) idx[j] = static_cast<int32_t>(j);
        // (value desc, index asc): a strict total order, so the top-k set is unique
        std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), [row](int32_t x, int32_t y) {
            if (row[x] != row[y]) return row[x] > row[y];
            return x < y;
        });
        std::sort(idx.begin(), idx.begin() + k);
        std::memcpy(sel + i * k, idx.data(), sizeof(int32_t) * k);
    }
    return 0;
}

int orc_build_mask(int64_t nqb, int64_t b, int64_t n_p_tok, int64_t n_local, const int32_t* sel,
                   int64_t k, float* mask) {
    const int64_t cols = n_p_tok + n_local * b;
    for (int64_t i = 0; i < nqb; ++i) {
        std::vector<char> vis(static_cast<size_t>(n_local), 0);
        for (int64_t j = 0; j < k; ++j) {
            const int32_t l = sel[i * k + j];
            if (l < 0 || l >= n_local) return fail("build_mask: selected index out of range");
            vis[l] = 1;
        }
        for (int64_t r = 0; r < b; ++r) {
            float* row = mask + (i * b + r) * cols;
            for (int64_t c = 0; c < n_p_tok; ++c) row[c] = 0.0f;
            for (int64_t l = 0; l < n_local; ++l)
                for (int64_t c = 0; c < b; ++c) row[n_p_tok + l * b + c] = vis[l] ? 0.0f : kNegInf;
        }
    }
    return 0;
}

int orc_attention_reference(const float* q, int64_t nq, const float* k, const float* v,
                            int64_t nkv, int64_t d, const float* mask, float scale, float* out) {
    if (nkv <= 0 || d <= 0) return fail("attention_reference: bad shape");
    std::vector<float> s(static_cast<size_t>(nq * nkv));
    if (orc_matmul_nt(q, nq, d, k, nkv, s.data())) return 1;
    for (auto& x : s) x = x * scale;
    std::vector<float> p(s.size());
    if (orc_masked_softmax_rows(s.data(), nq, nkv, mask, p.data())) return 1;
    return orc_matmul(p.data(), nq, nkv, v, d, out);
}

int orc_attention_sparse(const float* q, int64_t nqb, int64_t bq, const float* k, const float* v,
                         int64_t bkv, const int32_t* vis, int64_t n_vis, int64_t d, float scale,
                         const uint8_t* qmask, float* out, float* lse) {
    if (nqb < 0 || bq <= 0 || bkv <= 0 || d <= 0 || n_vis < 0)
        return fail("attention_sparse: bad geometry");
    const int64_t rows = nqb * bq;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t qb = r / bq;
        if (qmask != nullptr && qmask[qb] == 0) continue;
        const float* qrow = q + r * d;
        std::vector<double> acc(static_cast<size_t>(d), 0.0);
        std::vector<float> z(static_cast<size_t>(bkv));
        float m = kNegInf;
        double l = 0.0;
        for (int64_t j = 0; j < n_vis; ++j) {
            const int64_t g = vis[qb * n_vis + j];
            const float* kb = k + g * bkv * d;
            const float* vb = v + g * bkv * d;
            float bm = kNegInf;
            for (int64_t t = 0; t < bkv; ++t) {
                z[t] = static_cast<float>(dot64(qrow, kb + t * d, d)) * scale;
                bm = std::max(bm, z[t]);
            }
            if (bm > m) {  // streaming rescale
                const double corr = (m == kNegInf) ? 0.0 : std::exp(double(m) - double(bm));
                l *= corr;
                for (int64_t c = 0; c < d; ++c) acc[c] *= corr;
                m = bm;
            }
            for (int64_t t = 0; t < bkv; ++t) {
                const double e = std::exp(double(z[t]) - double(m));
                l += e;
                const float* vr = vb + t * d;
                for (int64_t c = 0; c < d; ++c) acc[c] += e * static_cast<double>(vr[c]);
            }
        }
        float* orow = out + r * d;
        for (int64_t c = 0; c < d; ++c) orow[c] = l > 0.0 ? static_cast<float>(acc[c] / l) : 0.0f;
        if (lse != nullptr) lse[r] = l > 0.0 ? static_cast<float>(double(m) + std::log(l)) : kNegInf;
    }
    return 0;
}

int orc_attention_sparse_backward(const float* q, int64_t nqb, int64_t bq, const float* k, const float* v,
                                  int64_t bkv, const int32_t* vis, int64_t n_vis, int64_t d, float scale,
                                  const float* d_out, float* dq, float* dk, float* dv, int64_t n_store) {
    if (nqb < 0 || bq <= 0 || bkv <= 0 || d <= 0 || n_vis < 0 || n_store < 0)
        return fail("attention_sparse_backward: bad geometry");
    std::vector<double> dk64(static_cast<size_t>(n_store * bkv * d), 0.0), dv64(dk64.size(), 0.0);
    const int64_t nt = n_vis * bkv;
    std::vector<double> s(static_cast<size_t>(nt)), p(s.size()), dp(s.size());
    for (int64_t r = 0; r < nqb * bq; ++r) {  // sequential: dk / dv accumulate in row order
        const int64_t qb = r / bq;
        const float* qrow = q + r * d;
        const float* grow = d_out + r * d;
        double m = -std::numeric_limits<double>::infinity();
        for (int64_t j = 0; j < n_vis; ++j)
            for (int64_t t = 0; t < bkv; ++t) {
                const int64_t g = vis[qb * n_vis + j];
                const int64_t i = j * bkv + t;
                s[i] = dot64(qrow, k + (g * bkv + t) * d, d) * static_cast<double>(scale);
                dp[i] = dot64(grow, v + (g * bkv + t) * d, d);
                m = std::max(m, s[i]);
            }
        double l = 0.0;
        for (int64_t i = 0; i < nt; ++i) l += (p[i] = std::exp(s[i] - m));
        double D = 0.0;
        for (int64_t i = 0; i < nt; ++i) D += (p[i] /= l) * dp[i];
        double* dqr = nullptr;
        std::vector<double> dq64(static_cast<size_t>(d), 0.0);
        dqr = dq64.data();
        for (int64_t j = 0; j < n_vis; ++j) {
            const int64_t g = vis[qb * n_vis + j];
            for (int64_t t = 0; t < bkv; ++t) {
                const int64_t i = j * bkv + t;
                const double ds = p[i] * (dp[i] - D);
                const float* kr = k + (g * bkv + t) * d;
                double* dkr = dk64.data() + (g * bkv + t) * d;
                double* dvr = dv64.data() + (g * bkv + t) * d;
                for (int64_t c = 0; c < d; ++c) {
                    dqr[c] += ds * kr[c];
                    dkr[c] += ds * static_cast<double>(scale) * qrow[c];
                    dvr[c] += p[i] * grow[c];
                }
            }
        }
        for (int64_t c = 0; c < d; ++c) dq[r * d + c] = static_cast<float>(dqr[c] * static_cast<double>(scale));
    }
    for (size_t i = 0; i < dk64.size(); ++i) {
        dk[i] = static_cast<float>(dk64[i]);
        dv[i] = static_cast<float>(dv64[i]);
    }
    return 0;
}

int orc_flop_count(int64_t nq, int64_t np, int64_t nl, int64_t b, int64_t k_sel, int64_t d,
                   double* dense, double* sparse, double* ratio) {
    if (nq <= 0 || b <= 0 || d <= 0 || np < 0 || nl < 0 || k_sel < 0)
        return fail("flop_count: non-positive geometry");
    const double dn = 4.0 * double(nq) * double(np + nl) * double(d);
    const double coarse = 4.0 * (double(nq) / double(b)) * (double(np + nl) / double(b)) * double(d);
    const double sp = 4.0 * double(nq) * double(np + k_sel * b) * double(d) + coarse;
    *dense = dn;
    *sparse = sp;
    *ratio = dn / sp;
    return 0;
}

static bool integral(double x, int64_t* out) {
    const double r = std::round(x);
    if (std::fabs(x - r) > 1e-9 * std::max(1.0, std::fabs(x))) return false;
    *out = static_cast<int64_t>(r);
    return true;
}

int orc_kv_length(int64_t n_c, double local_ratio, double persist_ratio, int64_t* n_kv) {
    if (n_c <= 0 || local_ratio < 0 || persist_ratio < 0) return fail("kv_length: bad geometry");
    int64_t n_l = 0, n_p = 0;
    if (!integral(double(n_c) * local_ratio, &n_l)) return fail("kv_length: N_L not integral");
    if (!integral(double(n_l) * persist_ratio, &n_p)) return fail("kv_length: N_P not integral");
    *n_kv = n_l + n_p;
    return 0;
}

int orc_kv_bytes(int64_t tokens, int64_t layers, int64_t kv_heads, int64_t head_dim, int64_t bpe,
                 int64_t* bytes) {
    if (tokens < 0 || layers < 0 || kv_heads < 0 || head_dim < 0 || bpe < 0)
        return fail("kv_bytes: negative argument");
    *bytes = 2 * layers * tokens * kv_heads * head_dim * bpe;
    return 0;
}

// ---------------------------------------------------------------------------------------------
// memory
// ---------------------------------------------------------------------------------------------
struct orc_mem {
    int64_t capacity_c = 0;
    int64_t window_chunks = 0;
    std::vector<int64_t> sinks;                       // id asc
    std::vector<std::pair<int64_t, float>> dynamic;   // (id, score), (score desc, id asc)
    std::vector<std::vector<int64_t>> window;         // FIFO of chunks
    int64_t max_id = -1;
    bool have_sink_chunk = false;
    int64_t sink_lo = 0, sink_hi = -1;                // id range of the first (sink) chunk
};

static bool rank_before(int64_t ida, float sa, int64_t idb, float sb) {
    if (sa != sb) return sa > sb;
    return ida < idb;
}

orc_mem* orc_mem_create(int64_t capacity_c, int64_t window_chunks) {
    if (capacity_c < 0 || window_chunks < 1) {
        fail("mem_create: capacity must be >= 0 and window >= 1 chunk");
        return nullptr;
    }
    auto* m = new orc_mem;
    m->capacity_c = capacity_c;
    m->window_chunks = window_chunks;
    return m;
}

void orc_mem_destroy(orc_mem* m) { delete m; }

int orc_mem_push_chunk(orc_mem* m, const int64_t* ids, int64_t n, int64_t* evicted,
                       int64_t max_evicted, int64_t* n_evicted) {
    if (m == nullptr || n <= 0) return fail("push_chunk: empty chunk");
    int64_t prev = m->max_id;
    for (int64_t i = 0; i < n; ++i) {
        if (ids[i] <= prev) return fail("push_chunk: id ordering violation");
        prev = ids[i];
    }
    m->max_id = prev;
    if (!m->have_sink_chunk) {  // sinks = blocks of the first generated chunk
        m->have_sink_chunk = true;
        m->sink_lo = ids[0];
        m->sink_hi = ids[n - 1];
    }
    m->window.emplace_back(ids, ids + n);
    *n_evicted = 0;
    if (static_cast<int64_t>(m->window.size()) > m->window_chunks) {
        const auto& old = m->window.front();
        if (static_cast<int64_t>(old.size()) > max_evicted) return fail("push_chunk: evicted buffer too small");
        std::copy(old.begin(), old.end(), evicted);
        *n_evicted = static_cast<int64_t>(old.size());
        m->window.erase(m->window.begin());
    }
    return 0;
}

int orc_mem_update_persistent(orc_mem* m, const int64_t* evicted, int64_t n_evicted,
                              const int64_t* score_ids, const float* scores, int64_t n_scores) {
    if (m == nullptr) return fail("update_persistent: null memory");
    auto lookup = [&](int64_t id, float* out) {
        for (int64_t i = 0; i < n_scores; ++i)
            if (score_ids[i] == id) {
                *out = scores[i];
                return true;
            }
        return false;
    };
    std::vector<std::pair<int64_t, float>> cand;
    std::vector<int64_t> new_sinks = m->sinks;
    for (const auto& e : m->dynamic) {  // scores refreshed from the current s_t
        float s;
        if (!lookup(e.first, &s)) return fail("update_persistent: missing score for id " + std::to_string(e.first));
        cand.emplace_back(e.first, s);
    }
    for (int64_t i = 0; i < n_evicted; ++i) {
        const int64_t id = evicted[i];
        if (m->have_sink_chunk && id >= m->sink_lo && id <= m->sink_hi) {
            new_sinks.push_back(id);  // sinks are always retained (paper footnote, Eq. 9)
            continue;
        }
        float s;
        if (!lookup(id, &s)) return fail("update_persistent: missing score for id " + std::to_string(id));
        cand.emplace_back(id, s);
    }
    std::sort(new_sinks.begin(), new_sinks.end());
    std::sort(cand.begin(), cand.end(), [](const auto& a, const auto& b) {
        return rank_before(a.first, a.second, b.first, b.second);
    });
    const int64_t dyn_cap = std::max<int64_t>(0, m->capacity_c - static_cast<int64_t>(new_sinks.size()));
    if (static_cast<int64_t>(cand.size()) > dyn_cap) cand.resize(static_cast<size_t>(dyn_cap));
    m->sinks = std::move(new_sinks);
    m->dynamic = std::move(cand);
    return 0;
}

int orc_mem_assemble(const orc_mem* m, int64_t* ids, int32_t* region, int64_t cap, int64_t* n_p,
                     int64_t* n_l) {
    if (m == nullptr) return fail("assemble_kv: null memory");
    std::vector<int64_t> dyn;
    for (const auto& e : m->dynamic) dyn.push_back(e.first);
    std::sort(dyn.begin(), dyn.end());
    int64_t n = 0;
    auto put = [&](int64_t id, int32_t reg) {
        if (n < cap) {
            ids[n] = id;
            if (region) region[n] = reg;
        }
        ++n;
    };
    for (int64_t id : m->sinks) put(id, 0);
    for (int64_t id : dyn) put(id, 0);
    *n_p = n;
    for (const auto& c : m->window)
        for (int64_t id : c) put(id, 1);
    *n_l = n - *n_p;
    if (n > cap) return fail("assemble_kv: output buffer too small");
    return 0;
}

int orc_mem_dynamic(const orc_mem* m, int64_t* ids, float* scores, int64_t cap, int64_t* n) {
    if (m == nullptr) return fail("null memory");
    *n = static_cast<int64_t>(m->dynamic.size());
    if (*n > cap) return fail("buffer too small");
    for (int64_t i = 0; i < *n; ++i) {
        ids[i] = m->dynamic[i].first;
        scores[i] = m->dynamic[i].second;
    }
    return 0;
}

int64_t orc_mem_num_sinks(const orc_mem* m) { return m ? static_cast<int64_t>(m->sinks.size()) : -1; }

int orc_topc_select(const int64_t* ids, const float* scores, const uint8_t* is_sink, int64_t n,
                    int64_t capacity_c, uint8_t* kept) {
    if (n < 0 || capacity_c < 0) return fail("topc_select: bad arguments");
    std::vector<int64_t> order;
    int64_t n_sinks = 0;
    for (int64_t i = 0; i < n; ++i) {
        kept[i] = 0;
        if (is_sink && is_sink[i]) {
            kept[i] = 1;
            ++n_sinks;
        } else {
            order.push_back(i);
        }
    }
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return rank_before(ids[a], scores[a], ids[b], scores[b]);
    });
    const int64_t cap = std::max<int64_t>(0, capacity_c - n_sinks);
    for (int64_t r = 0; r < static_cast<int64_t>(order.size()) && r < cap; ++r) kept[order[r]] = 1;
    return 0;
}

}  // extern "C"
