// multigpu.cu -- K4 over several GPUs: k-means (clustering.hpp:148-260) with
// the segment embeddings sharded in index order over one context per GPU,
// bit-identical to the single-GPU (and reference) result.
//
// The host orchestration of epk_kmeans lives here for any number of shards
// (epk_kmeans is the one-shard case), so one code path serves both:
//   seeding    k-means++ (clustering.hpp:160-191) on the host with the
//              reference RNG stream; every shard computes its points'
//              distances to the newest centroid, the host walks them in
//              global index order;
//   assign     per shard on its device (ties -> lower cluster);
//   repair     empty clusters steal the globally farthest point of a
//              multi-member cluster (clustering.hpp:213-232), host-side over
//              the shards' distances in index order;
//   update     the centroid sums as an ORDERED CHAIN: shard 0
//              sums its points in index order, hands (sums, counts) to shard
//              1, which keeps adding ITS points in index order on top, ...;
//              the last shard divides and broadcasts the centroids.  Each
//              add happens in exactly the single-GPU order, so the bits match;
//              an all-reduce would not (fp64 addition is not associative).
// Transport between shards: NCCL point-to-point (ncclSend / ncclRecv inside
// ncclGroupStart/End) plus ncclBroadcast over a communicator of the shards'
// devices (ncclCommInitAll, one host thread drives every rank) when the
// devices are distinct; device-to-device copies when shards share a device.
// libnccl.so.2 is loaded at first use (dlopen), so single-GPU users of
// libepk.so carry no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "epk_internal.cuh"

namespace epk {

int launch_km_dist(epk_ctx*, const double*, int64_t, int64_t, const double*, int64_t, double*);
int launch_km_assign(epk_ctx*, const double*, int64_t, int64_t, const double*, int64_t, int64_t*, double*);
int launch_km_sums(epk_ctx*, const double*, int64_t, int64_t, const int64_t*, int64_t, double*, int64_t*, int);
int launch_km_finalize(epk_ctx*, const double*, const int64_t*, int64_t, int64_t, double*);
int launch_km_sqdist(epk_ctx*, const double*, int64_t, int64_t, const double*, const int64_t*, double*);

// ---- NCCL, resolved at first use ---------------------------------------------
struct NcclApi {
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclBroadcast) bcast = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) err = nullptr;
};

static const NcclApi* nccl_api() {
    static std::once_flag once;
    static NcclApi api;
    static bool ok = false;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
        api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
        api.bcast = reinterpret_cast<decltype(api.bcast)>(dlsym(h, "ncclBroadcast"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
        api.err = reinterpret_cast<decltype(api.err)>(dlsym(h, "ncclGetErrorString"));
        ok = api.comm_init_all && api.send && api.recv && api.bcast && api.group_start && api.group_end && api.err;
    });
    return ok ? &api : nullptr;
}

#define EPK_NCCL_CHECK(api, expr)                                                                       \
    do {                                                                                                \
        ncclResult_t _r = (expr);                                                                       \
        if (_r != ncclSuccess) return fail(EPK_ERR_CUDA, std::string("NCCL: ") + (api)->err(_r) + " in " #expr); \
    } while (0)

// One communicator per distinct device list, created once per process.
static int nccl_comms(const NcclApi* api, const std::vector<int>& devs, std::vector<ncclComm_t>* out) {
    static std::mutex mu;
    static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(devs);
    if (it == cache.end()) {
        std::vector<ncclComm_t> comms(devs.size());
        EPK_NCCL_CHECK(api, api->comm_init_all(comms.data(), int(devs.size()), devs.data()));
        it = cache.emplace(devs, std::move(comms)).first;
    }
    *out = it->second;
    return EPK_OK;
}

// ---- host mirror of epikv::Rng (numerics.hpp:146-183) used by the seeding ----
struct KmRng {
    std::mt19937_64 gen;
    explicit KmRng(uint64_t s) : gen(s) {}
    double uniform() { return double(gen() >> 11) * 0x1.0p-53; }
    int64_t uniform_index(int64_t n) { return int64_t((static_cast<unsigned __int128>(gen()) * uint64_t(n)) >> 64); }
};

struct Shard {
    epk_ctx* ctx;
    const double* pts;
    int64_t n, start;
    double *cent, *sums, *d2;
    int64_t *assign, *counts;
};

static int use(const Shard& s) {
    EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
    return EPK_OK;
}

// Moves `bytes` from shard a's buffer to shard b's (b's stream waits for a's work).
static int hand_over(const Shard& a, const void* src, const Shard& b, void* dst, size_t bytes) {
    cudaEvent_t ev;
    EPK_CUDA_CHECK(cudaSetDevice(a.ctx->device));
    EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    EPK_CUDA_CHECK(cudaEventRecord(ev, a.ctx->stream));
    EPK_CUDA_CHECK(cudaSetDevice(b.ctx->device));
    EPK_CUDA_CHECK(cudaStreamWaitEvent(b.ctx->stream, ev, 0));
    EPK_CUDA_CHECK(cudaMemcpyPeerAsync(dst, b.ctx->device, src, a.ctx->device, bytes, b.ctx->stream));
    EPK_CUDA_CHECK(cudaEventDestroy(ev));
    return EPK_OK;
}

static int sync_all(const std::vector<Shard>& sh) {
    for (const Shard& s : sh) {
        EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
        EPK_CUDA_CHECK(cudaStreamSynchronize(s.ctx->stream));
    }
    return EPK_OK;
}

// Every shard's per-point values (distances) into host[global index].
static int gather_points(const std::vector<Shard>& sh, double* const Shard::*buf, std::vector<double>& host) {
    for (const Shard& s : sh) {
        if (s.n == 0) continue;
        EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
        EPK_CUDA_CHECK(cudaMemcpyAsync(host.data() + s.start, s.*buf, size_t(s.n) * 8, cudaMemcpyDeviceToHost,
                                       s.ctx->stream));
    }
    return sync_all(sh);
}

int kmeans_shards(epk_ctx* const* ctxs, int S, const double* const* points, const int64_t* ns, int64_t dim, int64_t k,
                  uint64_t seed, int64_t max_iters, int64_t* assign_out, double* cent_out, int64_t* iters_out,
                  double* sse_out) {
    if (S < 1 || !ctxs || !points || !ns) return fail(EPK_ERR_ARG, "kmeans: no shards");
    if (k < 1) return fail(EPK_ERR_ARG, "kmeans: cluster count must be >= 1");
    if (dim < 1) return fail(EPK_ERR_ARG, "kmeans: dimension must be >= 1");
    std::vector<Shard> sh(static_cast<size_t>(S));
    int64_t n = 0;
    std::vector<int> devs;
    for (int s = 0; s < S; ++s) {
        if (!ctxs[s]) return fail(EPK_ERR_ARG, "kmeans: null context");
        if (ns[s] < 0 || (ns[s] > 0 && !points[s])) return fail(EPK_ERR_ARG, "kmeans: bad shard");
        sh[size_t(s)] = Shard{ctxs[s], points[s], ns[s], n, nullptr, nullptr, nullptr, nullptr, nullptr};
        n += ns[s];
        devs.push_back(ctxs[s]->device);
    }
    if (n < k)
        return fail(EPK_ERR_ARG, "kmeans: fewer points (" + std::to_string(n) + ") than clusters (" +
                                     std::to_string(k) + ")");
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const NcclApi* api = nullptr;
    std::vector<ncclComm_t> comms;
    static const bool force_nccl = std::getenv("EPK_FORCE_NCCL") != nullptr;  // tests: the NCCL path on 1 GPU
    if (distinct && (S > 1 || force_nccl)) {
        api = nccl_api();
        if (!api) return fail(EPK_ERR_UNSUPPORTED, "kmeans: libnccl.so.2 not loadable (sharded k-means over GPUs)");
        int rc = nccl_comms(api, devs, &comms);
        if (rc) return rc;
    }
    // per-shard device state in each context's grow-only second workspace
    for (Shard& s : sh) {
        int rc = use(s);
        if (rc) return rc;
        const int64_t m = std::max<int64_t>(s.n, 1);
        rc = ws2_require(s.ctx, 2 * align_up(k * dim * 8, 256) + 2 * align_up(m * 8, 256) + align_up(k * 8, 256) + 1024);
        if (rc) return rc;
        WsCarver wc(s.ctx->ws2);
        s.cent = wc.take<double>(k * dim);
        s.sums = wc.take<double>(k * dim);
        s.d2 = wc.take<double>(m);
        s.assign = wc.take<int64_t>(m);
        s.counts = wc.take<int64_t>(k);
    }
    auto shard_of = [&](int64_t i) -> const Shard& {
        int s = 0;
        while (s + 1 < S && sh[size_t(s + 1)].start <= i) ++s;
        return sh[size_t(s)];
    };
    // centroid c := point i (the host relays it to every shard)
    std::vector<double> row(static_cast<size_t>(dim));
    auto set_centroid = [&](int64_t c, int64_t i) -> int {
        const Shard& o = shard_of(i);
        EPK_CUDA_CHECK(cudaSetDevice(o.ctx->device));
        EPK_CUDA_CHECK(cudaMemcpyAsync(row.data(), o.pts + (i - o.start) * dim, size_t(dim) * 8,
                                       cudaMemcpyDeviceToHost, o.ctx->stream));
        EPK_CUDA_CHECK(cudaStreamSynchronize(o.ctx->stream));
        for (const Shard& s : sh) {
            EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
            EPK_CUDA_CHECK(cudaMemcpyAsync(s.cent + c * dim, row.data(), size_t(dim) * 8, cudaMemcpyHostToDevice,
                                           s.ctx->stream));
        }
        return sync_all(sh);
    };

    // k-means++ seeding (clustering.hpp:160-191): distances on the devices,
    // the running min, the sequential total and the draw on the host.
    KmRng rng(seed);
    int rc = set_centroid(0, rng.uniform_index(n));
    if (rc) return rc;
    std::vector<double> best(static_cast<size_t>(n), std::numeric_limits<double>::infinity());
    std::vector<double> dd(static_cast<size_t>(n));
    for (int64_t have = 1; have < k; ++have) {
        for (const Shard& s : sh) {
            if (s.n == 0) continue;
            if ((rc = use(s)) || (rc = launch_km_dist(s.ctx, s.pts, s.n, dim, s.cent + (have - 1) * dim, 1, s.d2)))
                return rc;
        }
        if ((rc = gather_points(sh, &Shard::d2, dd))) return rc;
        double total = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            best[size_t(i)] = std::min(best[size_t(i)], dd[size_t(i)]);
            total += best[size_t(i)];
        }
        int64_t chosen = 0;
        if (total > 0.0) {
            const double target = rng.uniform() * total;
            double acc = 0.0;
            chosen = n - 1;
            for (int64_t i = 0; i < n; ++i) {
                acc += best[size_t(i)];
                if (acc > target) {
                    chosen = i;
                    break;
                }
            }
        } else {
            chosen = rng.uniform_index(n);
        }
        if ((rc = set_centroid(have, chosen))) return rc;
    }

    // Lloyd iterations (clustering.hpp:195-255).
    std::vector<int64_t> assign(static_cast<size_t>(n), 0), prev(static_cast<size_t>(n), 0);
    std::vector<int64_t> counts(static_cast<size_t>(k));
    auto upload_assign = [&]() -> int {
        for (const Shard& s : sh) {
            if (s.n == 0) continue;
            EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
            EPK_CUDA_CHECK(cudaMemcpyAsync(s.assign, assign.data() + s.start, size_t(s.n) * 8,
                                           cudaMemcpyHostToDevice, s.ctx->stream));
        }
        return EPK_OK;
    };
    int64_t iters = 0;
    for (int64_t iter = 0; iter < max_iters; ++iter) {
        for (const Shard& s : sh) {
            if (s.n == 0) continue;
            if ((rc = use(s)) || (rc = launch_km_assign(s.ctx, s.pts, s.n, dim, s.cent, k, s.assign, nullptr)))
                return rc;
        }
        for (const Shard& s : sh) {
            if (s.n == 0) continue;
            EPK_CUDA_CHECK(cudaSetDevice(s.ctx->device));
            EPK_CUDA_CHECK(cudaMemcpyAsync(assign.data() + s.start, s.assign, size_t(s.n) * 8,
                                           cudaMemcpyDeviceToHost, s.ctx->stream));
        }
        if ((rc = sync_all(sh))) return rc;
        bool changed = false;
        for (int64_t i = 0; i < n; ++i)
            if (assign[size_t(i)] != prev[size_t(i)]) changed = true;
        std::fill(counts.begin(), counts.end(), 0);
        for (int64_t a : assign) ++counts[size_t(a)];
        bool repaired = false;
        for (int64_t c = 0; c < k; ++c) {
            if (counts[size_t(c)] > 0) continue;
            // distances to the current centroids under the current assignment
            if ((rc = upload_assign())) return rc;
            for (const Shard& s : sh) {
                if (s.n == 0) continue;
                if ((rc = use(s)) || (rc = launch_km_sqdist(s.ctx, s.pts, s.n, dim, s.cent, s.assign, s.d2)))
                    return rc;
            }
            if ((rc = gather_points(sh, &Shard::d2, dd))) return rc;
            int64_t victim = 0;
            double worst = -1.0;
            for (int64_t i = 0; i < n; ++i) {
                if (counts[size_t(assign[size_t(i)])] <= 1) continue;
                if (dd[size_t(i)] > worst) {
                    worst = dd[size_t(i)];
                    victim = i;
                }
            }
            --counts[size_t(assign[size_t(victim)])];
            assign[size_t(victim)] = c;
            ++counts[size_t(c)];
            changed = true;
            repaired = true;
        }
        if (repaired && (rc = upload_assign())) return rc;
        // the ordered chain of partial sums (points in global index order)
        for (int s = 0; s < S; ++s) {
            const Shard& cur = sh[size_t(s)];
            if (s > 0) {
                const Shard& prv = sh[size_t(s - 1)];
                if (api) {
                    EPK_NCCL_CHECK(api, api->group_start());
                    EPK_NCCL_CHECK(api, api->send(prv.sums, size_t(k * dim), ncclFloat64, s, comms[size_t(s - 1)],
                                                  prv.ctx->stream));
                    EPK_NCCL_CHECK(api, api->send(prv.counts, size_t(k), ncclInt64, s, comms[size_t(s - 1)],
                                                  prv.ctx->stream));
                    EPK_NCCL_CHECK(api, api->recv(cur.sums, size_t(k * dim), ncclFloat64, s - 1, comms[size_t(s)],
                                                  cur.ctx->stream));
                    EPK_NCCL_CHECK(api, api->recv(cur.counts, size_t(k), ncclInt64, s - 1, comms[size_t(s)],
                                                  cur.ctx->stream));
                    EPK_NCCL_CHECK(api, api->group_end());
                } else {
                    if ((rc = hand_over(prv, prv.sums, cur, cur.sums, size_t(k * dim) * 8)) ||
                        (rc = hand_over(prv, prv.counts, cur, cur.counts, size_t(k) * 8)))
                        return rc;
                }
            }
            if ((rc = use(cur)) ||
                (rc = launch_km_sums(cur.ctx, cur.pts, cur.n, dim, cur.assign, k, cur.sums, cur.counts, s > 0 ? 1 : 0)))
                return rc;
        }
        const Shard& last = sh[size_t(S - 1)];
        if ((rc = use(last)) || (rc = launch_km_finalize(last.ctx, last.sums, last.counts, k, dim, last.cent)))
            return rc;
        if (S > 1 || api) {
            if (api) {
                EPK_NCCL_CHECK(api, api->group_start());
                for (int s = 0; s < S; ++s)
                    EPK_NCCL_CHECK(api, api->bcast(last.cent, sh[size_t(s)].cent, size_t(k * dim), ncclFloat64, S - 1,
                                                   comms[size_t(s)], sh[size_t(s)].ctx->stream));
                EPK_NCCL_CHECK(api, api->group_end());
            } else {
                for (int s = 0; s + 1 < S; ++s)
                    if ((rc = hand_over(last, last.cent, sh[size_t(s)], sh[size_t(s)].cent, size_t(k * dim) * 8)))
                        return rc;
            }
        }
        iters = iter + 1;
        for (const Shard& s : sh) {
            if (s.n == 0) continue;
            if ((rc = use(s)) || (rc = launch_km_sqdist(s.ctx, s.pts, s.n, dim, s.cent, s.assign, s.d2))) return rc;
        }
        if ((rc = gather_points(sh, &Shard::d2, dd))) return rc;
        double sse = 0.0;
        for (int64_t i = 0; i < n; ++i) sse += dd[size_t(i)];
        if (sse_out) sse_out[iter] = sse;
        prev = assign;
        if (!changed) break;
    }
    std::memcpy(assign_out, assign.data(), size_t(n) * 8);
    EPK_CUDA_CHECK(cudaSetDevice(sh.back().ctx->device));
    EPK_CUDA_CHECK(cudaMemcpy(cent_out, sh.back().cent, size_t(k * dim) * 8, cudaMemcpyDeviceToHost));
    *iters_out = iters;
    return EPK_OK;
}

}  // namespace epk

extern "C" int epk_kmeans_sharded(epk_ctx* const* ctxs, int32_t nshards, const double* const* points,
                                  const int64_t* n_per_shard, int64_t dim, int64_t k, uint64_t seed,
                                  int64_t max_iters, int64_t* assign_out, double* centroids_out,
                                  int64_t* iterations_out, double* sse_out) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int rc = epk::kmeans_shards(ctxs, nshards, points, n_per_shard, dim, k, seed, max_iters, assign_out,
                                      centroids_out, iterations_out, sse_out);
    cudaSetDevice(dev);  // the caller's current device is left as it was
    return rc;
}
