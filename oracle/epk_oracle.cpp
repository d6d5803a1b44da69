// epk_oracle.cpp -- CPU ORACLE for the EpiCache block-prefill eviction step.
//
// TEST INFRASTRUCTURE ONLY.  This file is a plain-C++ restatement of the
// reference algorithm (the epikv header library under
// /root/reference/proj/include/epikv).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it, and only
// as the checker.  The product path (paper_2509_17396_b200/, include/) never
// links or calls anything in oracle/.
//
// Parity is pinned two ways:
//   * tests/test_oracle_vs_ref.py compares every function below against the
//     reference headers themselves, compiled from /root/reference by
//     oracle/Makefile into oracle/_ref/libepkref.so;
//   * tests/golden/ holds fixtures generated from that reference build
//     (tests/golden/make_golden.py) so the oracle stays pinned on machines
//     without /root/reference (the GPU box).
//
// Conventions shared with the CUDA path (one "layer" at a time):
//   head_off[h]..head_off[h+1]  rows of kv-head h (position-sorted, CSR)
//   k, v                        [n][d] row-major
//   q                           [Hq][p][d]   query head qh -> kv head qh / G
//   kp                          [Hkv][p][d]  prompt keys (causal self-columns)
//   scores                      [n]          one score per live cache row
//
// Built with -O2 -ffp-contract=off -fno-math-errno (the reference's own
// flags, proj/CMakeLists.txt:21-25) so no multiply-add is fused.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

using i64 = std::int64_t;

// ---------------------------------------------------------------------------
// a1 + a2: fp64 restatement of the attention-weight loop
// (toymodel.hpp:327-391: scale :257, visible = cache_len + t + 1 :339,
// running max :348-356, exp(l - m) :368-373, sequential denominator :372,
// w = e / den :376) followed by score_with_prompt (scoring.hpp:80-128:
// cache columns only :102, window Max/Avg :104-116, GQA max :117-123).
// ---------------------------------------------------------------------------
void score_layer_f64(int hq, int hkv, int d, int p, const i64* head_off, const double* q,
                     const double* k, const double* kp, int agg_max, double* out) {
    const int group = hq / hkv;
    const double scale = 1.0 / std::sqrt(double(d));
    const double kMasked = -std::numeric_limits<double>::infinity();
    std::vector<double> logits;
    std::vector<double> acc_col;
    for (int h = 0; h < hkv; ++h) {
        const i64 n = head_off[h + 1] - head_off[h];
        const double* kh = k + head_off[h] * d;
        const double* kph = kp + i64(h) * p * d;
        for (i64 j = 0; j < n; ++j) out[head_off[h] + j] = kMasked;  // filled by max below
        bool first_qh = true;
        for (int g = 0; g < group; ++g) {
            const int qh = h * group + g;
            acc_col.assign(size_t(n), agg_max ? kMasked : 0.0);
            logits.resize(size_t(n + p));
            for (int t = 0; t < p; ++t) {
                const double* qv = q + (i64(qh) * p + t) * d;
                const i64 visible = n + t + 1;
                double max_logit = kMasked;
                for (i64 j = 0; j < visible; ++j) {
                    const double* kv = j < n ? kh + j * d : kph + (j - n) * d;
                    double acc = 0.0;
                    for (int dd = 0; dd < d; ++dd) acc += qv[dd] * kv[dd];
                    const double s = acc * scale;
                    if (s > max_logit) max_logit = s;
                    logits[size_t(j)] = s;
                }
                double denom = 0.0;
                for (i64 j = 0; j < visible; ++j) {
                    const double e = std::exp(logits[size_t(j)] - max_logit);
                    logits[size_t(j)] = e;
                    denom += e;
                }
                for (i64 j = 0; j < n; ++j) {
                    const double w = logits[size_t(j)] / denom;
                    if (agg_max) {
                        acc_col[size_t(j)] = std::max(acc_col[size_t(j)], w);
                    } else {
                        acc_col[size_t(j)] += w;
                    }
                }
            }
            for (i64 j = 0; j < n; ++j) {
                double a = acc_col[size_t(j)];
                if (!agg_max) a /= double(p);
                double& slot = out[head_off[h] + j];
                if (first_qh || a > slot) slot = a;  // scoring.hpp:118-123
            }
            first_qh = false;
        }
    }
}

// ---------------------------------------------------------------------------
// EPK-F32 v1: the fp32 parity contract mirrored bit-for-bit by the CUDA
// parity scorer (paper_2509_17396_b200/csrc/score_f32.cu).  Same loop
// structure as the fp64 restatement above, with three fixed choices that make
// the result reproducible on any IEEE fp32 machine:
//   (1) sequential d-order dot, separate multiply and add (no FMA);
//   (2) epk_expf below (Cody-Waite + degree-7 Horner, explicit 2^k scaling);
//   (3) denominator = pairwise tree over 64-column sequential chunk sums
//       (the reference's sequential order is not safe in fp32 at 180K
//       columns, SURVEY.md section 7 "Hard parts" 3).
// ---------------------------------------------------------------------------
inline float bits_to_float(std::uint32_t b) {
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}

float epk_expf(float x) {
    if (x > 88.72283935546875f) return std::numeric_limits<float>::infinity();
    if (x < -103.97207641601562f) return 0.0f;
    const float t = x * 1.44269502162933349609375f;
    const float kf = std::rint(t);
    float r = x - kf * 0.693145751953125f;
    r = r - kf * 1.428606765330187045037746429443359375e-06f;
    float pz = 1.98412701138295233249664306640625e-04f;   // 1/5040
    pz = pz * r + 1.3888889225199818611145019531250e-03f;  // 1/720
    pz = pz * r + 8.3333337679505348205566406250000e-03f;  // 1/120
    pz = pz * r + 4.1666667908430099487304687500000e-02f;  // 1/24
    pz = pz * r + 1.6666667163372039794921875000000e-01f;  // 1/6
    pz = pz * r + 0.5f;
    pz = pz * r + 1.0f;
    pz = pz * r + 1.0f;
    const int ki = int(kf);
    if (ki > 127) return (pz * bits_to_float(std::uint32_t(127 + 127) << 23)) * 2.0f;
    if (ki >= -126) return pz * bits_to_float(std::uint32_t(ki + 127) << 23);
    return (pz * bits_to_float(std::uint32_t(ki + 127 + 64) << 23)) *
           bits_to_float(std::uint32_t(127 - 64) << 23);
}

constexpr int kChunk = 64;

float tree_sum_chunks(const float* e, i64 count, std::vector<float>& scratch) {
    const i64 nchunks = (count + kChunk - 1) / kChunk;
    scratch.resize(size_t(std::max<i64>(nchunks, 1)));
    for (i64 c = 0; c < nchunks; ++c) {
        float s = 0.0f;
        const i64 end = std::min<i64>(count, (c + 1) * kChunk);
        for (i64 j = c * kChunk; j < end; ++j) s = s + e[j];
        scratch[size_t(c)] = s;
    }
    i64 len = nchunks;
    while (len > 1) {
        const i64 half = len / 2;
        for (i64 i = 0; i < half; ++i) scratch[size_t(i)] = scratch[size_t(2 * i)] + scratch[size_t(2 * i + 1)];
        if (len & 1) scratch[size_t(half)] = scratch[size_t(len - 1)];
        len = (len + 1) / 2;
    }
    return scratch[0];
}

void score_layer_f32(int hq, int hkv, int d, int p, const i64* head_off, const float* q,
                     const float* k, const float* kp, int agg_max, float* out) {
    const int group = hq / hkv;
    const float scale = float(1.0 / std::sqrt(double(d)));
    const float kNegInf = -std::numeric_limits<float>::infinity();
    std::vector<float> e, acc_col, scratch;
    for (int h = 0; h < hkv; ++h) {
        const i64 n = head_off[h + 1] - head_off[h];
        const float* kh = k + head_off[h] * d;
        const float* kph = kp + i64(h) * p * d;
        for (i64 j = 0; j < n; ++j) out[head_off[h] + j] = kNegInf;
        for (int g = 0; g < group; ++g) {
            const int qh = h * group + g;
            acc_col.assign(size_t(n), agg_max ? kNegInf : 0.0f);
            e.resize(size_t(n + p));
            for (int t = 0; t < p; ++t) {
                const float* qv = q + (i64(qh) * p + t) * d;
                const i64 visible = n + t + 1;
                float m = kNegInf;
                for (i64 j = 0; j < visible; ++j) {
                    const float* kv = j < n ? kh + j * d : kph + (j - n) * d;
                    float acc = 0.0f;
                    for (int dd = 0; dd < d; ++dd) acc = acc + qv[dd] * kv[dd];
                    const float s = acc * scale;
                    if (s > m) m = s;
                    e[size_t(j)] = s;
                }
                for (i64 j = 0; j < visible; ++j) e[size_t(j)] = epk_expf(e[size_t(j)] - m);
                const float z = tree_sum_chunks(e.data(), visible, scratch);
                for (i64 j = 0; j < n; ++j) {
                    const float w = e[size_t(j)] / z;
                    if (agg_max) {
                        if (w > acc_col[size_t(j)]) acc_col[size_t(j)] = w;
                    } else {
                        acc_col[size_t(j)] = acc_col[size_t(j)] + w;
                    }
                }
            }
            for (i64 j = 0; j < n; ++j) {
                float a = acc_col[size_t(j)];
                if (!agg_max) a = a / float(p);
                float& slot = out[head_off[h] + j];
                if (a > slot) slot = a;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Multi-threaded forms of the two restatements above, for the parity tests at
// benchmark scale (a cfg5 layer is ~640 M dot products).  Same arithmetic:
// every logit is the same sequential-d chain, every row's max / exp /
// denominator the same sequence; only (a) four prompt rows' dot products are
// interleaved (independent chains, identical bits) and (b) query heads run on
// separate threads, each into its own window accumulator, combined afterwards
// in query-head order exactly as the single-threaded loops do.
// ---------------------------------------------------------------------------
template <typename T>
void qhead_window(int qh, int group, int d, int p, const i64* head_off, const T* q, const T* k, const T* kp,
                  int agg_max, T* acc_col) {
    const int h = qh / group;
    const i64 n = head_off[h + 1] - head_off[h];
    const T* kh = k + head_off[h] * d;
    const T* kph = kp + i64(h) * p * d;
    const T scale = T(1.0 / std::sqrt(double(d)));
    const T kNegInf = -std::numeric_limits<T>::infinity();
    std::vector<T> lg(size_t(4) * size_t(n + p));
    std::vector<float> scratch;
    for (i64 j = 0; j < n; ++j) acc_col[j] = agg_max ? kNegInf : T(0);
    for (int t0 = 0; t0 < p; t0 += 4) {
        const int nt = std::min(4, p - t0);
        const i64 vis_max = n + t0 + nt;
        const T* qv[4];
        for (int u = 0; u < 4; ++u) qv[u] = q + (i64(qh) * p + t0 + std::min(u, nt - 1)) * d;
        for (i64 j = 0; j < vis_max; ++j) {
            const T* kv = j < n ? kh + j * d : kph + (j - n) * d;
            T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            for (int dd = 0; dd < d; ++dd) {
                const T x = kv[dd];
                a0 = a0 + qv[0][dd] * x;
                a1 = a1 + qv[1][dd] * x;
                a2 = a2 + qv[2][dd] * x;
                a3 = a3 + qv[3][dd] * x;
            }
            lg[size_t(0 * (n + p) + j)] = a0 * scale;
            lg[size_t(1 * (n + p) + j)] = a1 * scale;
            lg[size_t(2 * (n + p) + j)] = a2 * scale;
            lg[size_t(3 * (n + p) + j)] = a3 * scale;
        }
        for (int u = 0; u < nt; ++u) {
            T* e = lg.data() + size_t(u) * size_t(n + p);
            const i64 visible = n + t0 + u + 1;
            T m = kNegInf;
            for (i64 j = 0; j < visible; ++j)
                if (e[j] > m) m = e[j];
            T den;
            if constexpr (sizeof(T) == 8) {
                den = 0.0;
                for (i64 j = 0; j < visible; ++j) {
                    const T x = std::exp(e[j] - m);
                    e[j] = x;
                    den += x;
                }
            } else {
                for (i64 j = 0; j < visible; ++j) e[j] = epk_expf(e[j] - m);
                den = tree_sum_chunks(e, visible, scratch);
            }
            for (i64 j = 0; j < n; ++j) {
                const T w = e[j] / den;
                if (agg_max) {
                    if constexpr (sizeof(T) == 8) acc_col[j] = std::max(acc_col[j], w);
                    else if (w > acc_col[j]) acc_col[j] = w;
                } else {
                    acc_col[j] = acc_col[j] + w;
                }
            }
        }
    }
}

template <typename T>
void score_layer_mt(int hq, int hkv, int d, int p, const i64* head_off, const T* q, const T* k, const T* kp,
                    int agg_max, T* out, int threads) {
    const int group = hq / hkv;
    std::vector<i64> acc_off(size_t(hq) + 1, 0);
    for (int qh = 0; qh < hq; ++qh) acc_off[qh + 1] = acc_off[qh] + (head_off[qh / group + 1] - head_off[qh / group]);
    std::vector<T> acc(size_t(acc_off[hq]));
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::min(threads, hq);
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w] {
            for (int qh = w; qh < hq; qh += threads)
                qhead_window<T>(qh, group, d, p, head_off, q, k, kp, agg_max, acc.data() + acc_off[qh]);
        });
    for (auto& th : pool) th.join();
    for (int h = 0; h < hkv; ++h) {
        const i64 n = head_off[h + 1] - head_off[h];
        for (int g = 0; g < group; ++g) {
            const T* a_col = acc.data() + acc_off[h * group + g];
            for (i64 j = 0; j < n; ++j) {
                T a = a_col[j];
                if (!agg_max) a = a / T(p);
                T& slot = out[head_off[h] + j];
                if (sizeof(T) == 8) {
                    if (g == 0 || a > slot) slot = a;  // scoring.hpp:118-123
                } else {
                    if (g == 0) slot = -std::numeric_limits<T>::infinity();
                    if (a > slot) slot = a;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// a4: evict_to_budget (kvcache.hpp:142-201).  Pooled over the layer's kv
// heads; pins (positions, live in any head) always kept; the remaining
// limit - pinned_live slots go to the best (score desc, position asc, head
// asc) candidates; per-head order preserved.  Returns
//   0  -> keep[] written (evicted)
//   1  -> under budget, returned unchanged (kvcache.hpp:148-151), keep[] = 1
//  -2  -> pinned entries exceed the layer limit (kvcache.hpp:175-178)
// ---------------------------------------------------------------------------
int evict_layer(int hkv, i64 budget, const i64* head_off, const i64* pos, const double* scores,
                const i64* pins, i64 npins, std::uint8_t* keep) {
    const i64 n = head_off[hkv];
    const i64 limit = i64(hkv) * budget;
    if (n <= limit) {
        std::fill(keep, keep + n, std::uint8_t(1));
        return 1;
    }
    std::unordered_set<i64> pinned(pins, pins + npins);
    struct Cand {
        double score;
        i64 position;
        int head;
        i64 row;
    };
    std::vector<Cand> cands;
    cands.reserve(size_t(n));
    i64 pinned_live = 0;
    for (int h = 0; h < hkv; ++h) {
        for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) {
            keep[r] = 0;
            if (pinned.count(pos[r])) {
                ++pinned_live;
                keep[r] = 1;
                continue;
            }
            cands.push_back({scores[r], pos[r], h, r});
        }
    }
    if (pinned_live > limit) return -2;
    const i64 slots = limit - pinned_live;
    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
        if (a.score != b.score) return a.score > b.score;
        if (a.position != b.position) return a.position < b.position;
        return a.head < b.head;
    });
    for (i64 i = 0; i < slots && i < i64(cands.size()); ++i) keep[cands[size_t(i)].row] = 1;
    return 0;
}

// a8: top_k_indices (numerics.hpp:111-125), applied per kv-head ("per-head"
// selection mode).  Ties to the lower index.
void topk_per_head(int hkv, i64 k, const i64* head_off, const double* scores, std::uint8_t* keep) {
    for (int h = 0; h < hkv; ++h) {
        const i64 n = head_off[h + 1] - head_off[h];
        const double* s = scores + head_off[h];
        std::vector<i64> idx(static_cast<size_t>(n));
        for (i64 i = 0; i < n; ++i) idx[size_t(i)] = i;
        for (i64 i = 0; i < n; ++i) keep[head_off[h] + i] = 0;
        if (k >= n) {
            for (i64 i = 0; i < n; ++i) keep[head_off[h] + i] = 1;
            continue;
        }
        std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), [&](i64 a, i64 b) {
            if (s[a] != s[b]) return s[a] > s[b];
            return a < b;
        });
        for (i64 i = 0; i < k; ++i) keep[head_off[h] + idx[size_t(i)]] = 1;
    }
}

// ---------------------------------------------------------------------------
// a9: kmeans (clustering.hpp:148-260).  The random stream is the standard
// mt19937_64 consumed exactly as epikv::Rng does (numerics.hpp:146-183):
// uniform() = (u64 >> 11) * 2^-53, uniform_index(n) = (u64 * n) >> 64.
// ---------------------------------------------------------------------------
double sq_distance(const double* a, const double* b, i64 dim) {
    double acc = 0.0;
    for (i64 i = 0; i < dim; ++i) {
        const double dd = a[i] - b[i];
        acc += dd * dd;
    }
    return acc;
}

struct OracleRng {
    std::mt19937_64 gen;
    explicit OracleRng(std::uint64_t s) : gen(s) {}
    double uniform() { return double(gen() >> 11) * 0x1.0p-53; }
    i64 uniform_index(i64 n) {
        return i64((static_cast<unsigned __int128>(gen()) * std::uint64_t(n)) >> 64);
    }
};

int kmeans(const double* pts, i64 n, i64 dim, i64 k, std::uint64_t seed, i64 max_iters,
           i64* assign_out, double* centroids_out, i64* iters_out, double* sse_out) {
    if (k < 1 || n < k) return -1;
    OracleRng rng(seed);
    std::vector<double> cent;
    cent.reserve(size_t(k * dim));
    auto push_point = [&](i64 i) { cent.insert(cent.end(), pts + i * dim, pts + (i + 1) * dim); };
    push_point(rng.uniform_index(n));
    std::vector<double> d2(static_cast<size_t>(n));
    i64 have = 1;
    while (have < k) {
        double total = 0.0;
        for (i64 i = 0; i < n; ++i) {
            double best = std::numeric_limits<double>::infinity();
            for (i64 c = 0; c < have; ++c)
                best = std::min(best, sq_distance(pts + i * dim, cent.data() + c * dim, dim));
            d2[size_t(i)] = best;
            total += best;
        }
        i64 chosen = 0;
        if (total > 0.0) {
            const double target = rng.uniform() * total;
            double acc = 0.0;
            chosen = n - 1;
            for (i64 i = 0; i < n; ++i) {
                acc += d2[size_t(i)];
                if (acc > target) {
                    chosen = i;
                    break;
                }
            }
        } else {
            chosen = rng.uniform_index(n);
        }
        push_point(chosen);
        ++have;
    }
    std::vector<i64> assignments(static_cast<size_t>(n), 0);
    i64 iters = 0;
    for (i64 iter = 0; iter < max_iters; ++iter) {
        bool changed = false;
        for (i64 i = 0; i < n; ++i) {
            i64 best = 0;
            double best_d = sq_distance(pts + i * dim, cent.data(), dim);
            for (i64 c = 1; c < k; ++c) {
                const double dd = sq_distance(pts + i * dim, cent.data() + c * dim, dim);
                if (dd < best_d) {
                    best_d = dd;
                    best = c;
                }
            }
            if (assignments[size_t(i)] != best) {
                assignments[size_t(i)] = best;
                changed = true;
            }
        }
        std::vector<i64> counts(size_t(k), 0);
        for (i64 a : assignments) ++counts[size_t(a)];
        for (i64 c = 0; c < k; ++c) {
            if (counts[size_t(c)] > 0) continue;
            i64 victim = 0;
            double worst = -1.0;
            for (i64 i = 0; i < n; ++i) {
                if (counts[size_t(assignments[size_t(i)])] <= 1) continue;
                const double dd =
                    sq_distance(pts + i * dim, cent.data() + assignments[size_t(i)] * dim, dim);
                if (dd > worst) {
                    worst = dd;
                    victim = i;
                }
            }
            --counts[size_t(assignments[size_t(victim)])];
            assignments[size_t(victim)] = c;
            ++counts[size_t(c)];
            changed = true;
        }
        for (i64 c = 0; c < k; ++c) {
            std::vector<double> mean(static_cast<size_t>(dim), 0.0);
            for (i64 i = 0; i < n; ++i) {
                if (assignments[size_t(i)] != c) continue;
                for (i64 dd = 0; dd < dim; ++dd) mean[size_t(dd)] += pts[i * dim + dd];
            }
            for (double& x : mean) x /= double(counts[size_t(c)]);
            std::copy(mean.begin(), mean.end(), cent.begin() + c * dim);
        }
        iters = iter + 1;
        double sse = 0.0;
        for (i64 i = 0; i < n; ++i)
            sse += sq_distance(pts + i * dim, cent.data() + assignments[size_t(i)] * dim, dim);
        if (sse_out) sse_out[iter] = sse;
        if (!changed) break;
    }
    std::copy(assignments.begin(), assignments.end(), assign_out);
    std::copy(cent.begin(), cent.end(), centroids_out);
    *iters_out = iters;
    return 0;
}

// ---------------------------------------------------------------------------
// a10: the sensitivity reduction of measure_sensitivity (allocation.hpp:80-100):
// sigma_l = mean over (h, t) of cosine(k_full, k_block) (numerics.hpp:75-87,
// clamp to [-1, 1]), zero-norm pairs skipped and counted; sigma = 1 when no
// pair counts.  Inputs are [L][Hkv][N][d].
// ---------------------------------------------------------------------------
void sensitivity(int layers, int hkv, i64 ntok, int d, const double* kf, const double* kb,
                 double* sigma, i64* skipped) {
    i64 skip = 0;
    for (int l = 0; l < layers; ++l) {
        double acc = 0.0;
        i64 counted = 0;
        for (int h = 0; h < hkv; ++h) {
            for (i64 t = 0; t < ntok; ++t) {
                const double* a = kf + ((i64(l) * hkv + h) * ntok + t) * d;
                const double* b = kb + ((i64(l) * hkv + h) * ntok + t) * d;
                double na = 0.0, nb = 0.0, dot = 0.0;
                for (int i = 0; i < d; ++i) na += a[i] * a[i];
                for (int i = 0; i < d; ++i) nb += b[i] * b[i];
                na = std::sqrt(na);
                nb = std::sqrt(nb);
                if (na == 0.0 || nb == 0.0) {
                    ++skip;
                    continue;
                }
                for (int i = 0; i < d; ++i) dot += a[i] * b[i];
                const double c = dot / (na * nb);
                acc += std::clamp(c, -1.0, 1.0);
                ++counted;
            }
        }
        sigma[l] = counted > 0 ? acc / double(counted) : 1.0;
    }
    *skipped = skip;
}

// §8(f) rank 1, KeyDiff baseline: keydiff_scores (scoring.hpp:186-221).  Per
// (layer, kv-head) the anchor is the mean key (per-dimension sum in entry
// order, then / n); each entry scores -cosine(key, anchor) (numerics.hpp:
// 52-87: sequential dot and norms, clamp to [-1, 1]), or 0 when the anchor or
// the key has zero norm.  One layer: rows of head h are [head_off[h],
// head_off[h+1]), keys [rows][d].
// ---------------------------------------------------------------------------
void keydiff_layer(int hkv, int d, const i64* head_off, const double* k, double* out) {
    std::vector<double> anchor(static_cast<size_t>(d));
    for (int h = 0; h < hkv; ++h) {
        const i64 r0 = head_off[h], r1 = head_off[h + 1];
        if (r1 <= r0) continue;
        std::fill(anchor.begin(), anchor.end(), 0.0);
        for (i64 r = r0; r < r1; ++r)
            for (int i = 0; i < d; ++i) anchor[size_t(i)] += k[r * d + i];
        for (int i = 0; i < d; ++i) anchor[size_t(i)] /= double(r1 - r0);
        double nb = 0.0;
        for (int i = 0; i < d; ++i) nb += anchor[size_t(i)] * anchor[size_t(i)];
        nb = std::sqrt(nb);
        for (i64 r = r0; r < r1; ++r) {
            const double* a = k + r * d;
            double na = 0.0, dot = 0.0;
            for (int i = 0; i < d; ++i) na += a[i] * a[i];
            na = std::sqrt(na);
            double score = 0.0;
            if (nb != 0.0 && na != 0.0) {
                for (int i = 0; i < d; ++i) dot += a[i] * anchor[size_t(i)];
                score = -std::clamp(dot / (na * nb), -1.0, 1.0);
            }
            out[r] = score;
        }
    }
}

// ---------------------------------------------------------------------------
// a11: allocate (allocation.hpp:120-198).  Returns 0, or -1 on error.
int allocate(const double* sens, int layers, i64 per_head_budget, double alpha, i64* budgets_out,
             double* weights_out) {
    if (layers < 1 || per_head_budget < 1 || alpha < 0.0) return -1;
    std::vector<double> powered(static_cast<size_t>(layers)), w(static_cast<size_t>(layers));
    double total = 0.0;
    for (int l = 0; l < layers; ++l) {
        powered[size_t(l)] = std::pow(std::max(0.0, sens[l]), alpha);
        total += powered[size_t(l)];
    }
    for (int l = 0; l < layers; ++l)
        w[size_t(l)] = total <= 0.0 ? 1.0 / double(layers) : powered[size_t(l)] / total;
    const i64 grand = i64(layers) * per_head_budget;
    std::vector<double> real(static_cast<size_t>(layers));
    std::vector<i64> b(static_cast<size_t>(layers));
    i64 assigned = 0;
    for (int l = 0; l < layers; ++l) {
        real[size_t(l)] = w[size_t(l)] * double(grand);
        b[size_t(l)] = i64(std::floor(real[size_t(l)]));
        assigned += b[size_t(l)];
    }
    std::vector<int> order(static_cast<size_t>(layers));
    for (int l = 0; l < layers; ++l) order[size_t(l)] = l;
    std::sort(order.begin(), order.end(), [&](int a, int c) {
        const double ra = real[size_t(a)] - std::floor(real[size_t(a)]);
        const double rc = real[size_t(c)] - std::floor(real[size_t(c)]);
        if (ra != rc) return ra > rc;
        return a < c;
    });
    for (i64 i = 0; assigned < grand; ++i) {
        ++b[size_t(order[size_t(i % layers)])];
        ++assigned;
    }
    for (int l = 0; l < layers; ++l) {
        while (b[size_t(l)] < 1) {
            int victim = 0;
            for (int j = 1; j < layers; ++j) {
                if (b[size_t(j)] > b[size_t(victim)] ||
                    (b[size_t(j)] == b[size_t(victim)] && w[size_t(j)] < w[size_t(victim)]))
                    victim = j;
            }
            if (b[size_t(victim)] <= 1) return -1;
            --b[size_t(victim)];
            ++b[size_t(l)];
        }
    }
    for (int l = 0; l < layers; ++l) {
        budgets_out[l] = b[size_t(l)];
        if (weights_out) weights_out[l] = w[size_t(l)];
    }
    return 0;
}

}  // namespace

extern "C" {

void orc_score_layer_f64(int hq, int hkv, int d, int p, const i64* head_off, const double* q,
                         const double* k, const double* kp, int agg_max, double* out) {
    score_layer_f64(hq, hkv, d, p, head_off, q, k, kp, agg_max, out);
}

void orc_score_layer_f32(int hq, int hkv, int d, int p, const i64* head_off, const float* q,
                         const float* k, const float* kp, int agg_max, float* out) {
    score_layer_f32(hq, hkv, d, p, head_off, q, k, kp, agg_max, out);
}

void orc_score_layer_f64_mt(int hq, int hkv, int d, int p, const i64* head_off, const double* q,
                            const double* k, const double* kp, int agg_max, double* out, int threads) {
    score_layer_mt<double>(hq, hkv, d, p, head_off, q, k, kp, agg_max, out, threads);
}

void orc_score_layer_f32_mt(int hq, int hkv, int d, int p, const i64* head_off, const float* q,
                            const float* k, const float* kp, int agg_max, float* out, int threads) {
    score_layer_mt<float>(hq, hkv, d, p, head_off, q, k, kp, agg_max, out, threads);
}

// The restated attention grids themselves (toymodel.hpp:327-391): grids for
// query head qh are p x (n_h + p), concatenated in qh order; masked = 0.
void orc_prompt_grids_f64(int hq, int hkv, int d, int p, const i64* head_off, const double* q,
                          const double* k, const double* kp, double* grids) {
    const int group = hq / hkv;
    const double scale = 1.0 / std::sqrt(double(d));
    const double kMasked = -std::numeric_limits<double>::infinity();
    std::vector<double> sc;
    double* g = grids;
    for (int qh = 0; qh < hq; ++qh) {
        const int h = qh / group;
        const i64 n = head_off[h + 1] - head_off[h];
        const i64 cols = n + p;
        sc.resize(size_t(cols));
        for (int t = 0; t < p; ++t) {
            const double* qv = q + (i64(qh) * p + t) * d;
            const i64 visible = n + t + 1;
            double m = kMasked;
            for (i64 j = 0; j < visible; ++j) {
                const double* kv = j < n ? k + (head_off[h] + j) * d : kp + (i64(h) * p + (j - n)) * d;
                double acc = 0.0;
                for (int dd = 0; dd < d; ++dd) acc += qv[dd] * kv[dd];
                const double s = acc * scale;
                if (s > m) m = s;
                sc[size_t(j)] = s;
            }
            double den = 0.0;
            for (i64 j = 0; j < visible; ++j) {
                const double e = std::exp(sc[size_t(j)] - m);
                sc[size_t(j)] = e;
                den += e;
            }
            for (i64 j = 0; j < cols; ++j) g[t * cols + j] = j < visible ? sc[size_t(j)] / den : 0.0;
        }
        g += i64(p) * cols;
    }
}

float orc_expf(float x) { return epk_expf(x); }

void orc_expf_many(const float* x, i64 n, float* out) {
    for (i64 i = 0; i < n; ++i) out[i] = epk_expf(x[i]);
}

float orc_tree_sum(const float* e, i64 n) {
    std::vector<float> scratch;
    return tree_sum_chunks(e, n, scratch);
}

int orc_evict_layer(int hkv, i64 budget, const i64* head_off, const i64* pos, const double* scores,
                    const i64* pins, i64 npins, std::uint8_t* keep) {
    return evict_layer(hkv, budget, head_off, pos, scores, pins, npins, keep);
}

void orc_topk_per_head(int hkv, i64 k, const i64* head_off, const double* scores,
                       std::uint8_t* keep) {
    topk_per_head(hkv, k, head_off, scores, keep);
}

int orc_kmeans(const double* pts, i64 n, i64 dim, i64 k, std::uint64_t seed, i64 max_iters,
               i64* assign_out, double* centroids_out, i64* iters_out, double* sse_out) {
    return kmeans(pts, n, dim, k, seed, max_iters, assign_out, centroids_out, iters_out, sse_out);
}

void orc_sensitivity(int layers, int hkv, i64 ntok, int d, const double* kf, const double* kb,
                     double* sigma, i64* skipped) {
    sensitivity(layers, hkv, ntok, d, kf, kb, sigma, skipped);
}

void orc_keydiff_layer(int hkv, int d, const i64* head_off, const double* k, double* out) {
    keydiff_layer(hkv, d, head_off, k, out);
}

int orc_allocate(const double* sens, int layers, i64 per_head_budget, double alpha,
                 i64* budgets_out, double* weights_out) {
    return allocate(sens, layers, per_head_budget, alpha, budgets_out, weights_out);
}

}  // extern "C"
