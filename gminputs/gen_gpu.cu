// gen_gpu.cu -- GPU implementation of the seeded input generators in gminputs/__init__.py.
//
// Same counter-based generator (splitmix64 finaliser keyed by seed and stream) and the
// same arithmetic as the numpy code, so the edge lists are bit-identical for the same
// seed (checked by tests/test_gpu_parity.py::test_gpu_generator_matches_numpy).  Holds
// no subgraph-matching arithmetic: it only draws graphs and labels, for workloads too
// large to generate on the host (R-MAT scale >= 22).
#include <cuda_runtime.h>
#include <stdint.h>

#define GEN_API extern "C" __attribute__((visibility("default")))

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
__host__ __device__ __forceinline__ uint64_t mix64h(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
static uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64h(seed ^ (stream * 0xD1B54A32D192ED03ull)); }

__device__ __forceinline__ double unit(uint64_t key, uint64_t i) {
    return (double)(mix64(key + i * 0x9E3779B97F4A7C15ull) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_rmat(uint64_t m, int scale, uint64_t key, double t1, double t2, double t3,
                       uint64_t A, uint64_t B, uint32_t *src, uint32_t *dst) {
    const uint64_t mask = (scale == 64) ? ~0ull : ((1ull << scale) - 1);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0, d = 0;
        for (int k = 0; k < scale; ++k) {
            const double u = unit(key, e * (uint64_t)scale + (uint64_t)k);
            const uint64_t bit = 1ull << (scale - 1 - k);
            if (u >= t2) s |= bit;                              // quadrants c, d
            if ((u >= t1 && u < t2) || u >= t3) d |= bit;       // quadrants b, d
        }
        s = (s * A + B) & mask;
        d = (d * A + B) & mask;
        src[e] = (uint32_t)s;
        dst[e] = (uint32_t)d;
    }
}

__global__ void k_er(uint64_t m, uint64_t n, uint64_t key, uint32_t *src, uint32_t *dst) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        src[e] = (uint32_t)(mix64(key + (2 * e) * 0x9E3779B97F4A7C15ull) % n);
        dst[e] = (uint32_t)(mix64(key + (2 * e + 1) * 0x9E3779B97F4A7C15ull) % n);
    }
}

__global__ void k_labels(uint64_t n, uint32_t S, uint64_t key, uint32_t *lab) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        lab[v] = S <= 1 ? 0 : (uint32_t)(mix64(key + v * 0x9E3779B97F4A7C15ull) % S);
}

// Edges incident to a vertex set (bitmap over vertices): writes the matching (src,dst)
// pairs -- used to grow query graphs on device-resident edge lists.
__global__ void k_incident(uint64_t m, const uint32_t *src, const uint32_t *dst, const uint32_t *bits,
                           uint32_t *out_s, uint32_t *out_d, unsigned long long *cnt, uint64_t cap) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = src[e], b = dst[e];
        if (((bits[a >> 5] >> (a & 31)) & 1u) || ((bits[b >> 5] >> (b & 31)) & 1u)) {
            const unsigned long long k = atomicAdd(cnt, 1ull);
            if (k < cap) { out_s[k] = a; out_d[k] = b; }
        }
    }
}

// The other endpoints of all edges incident to vertex v (duplicates / self loops included;
// the caller dedups) -- neighbour lists of a device-resident edge list, for query growth.
__global__ void k_neighbors(uint64_t m, const uint32_t *src, const uint32_t *dst, uint32_t v, uint32_t *out,
                            unsigned long long *cnt, uint64_t cap) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = src[e], b = dst[e];
        if (a == v || b == v) {
            const unsigned long long k = atomicAdd(cnt, 1ull);
            if (k < cap) out[k] = a == v ? b : a;
        }
    }
}

static int grid(uint64_t work) {
    uint64_t g = (work + 255) / 256;
    if (g > 148ull * 64) g = 148ull * 64;
    return (int)(g ? g : 1);
}

GEN_API int gen_rmat(int scale, uint64_t m, uint64_t seed, double t1, double t2, double t3, uint64_t A, uint64_t B,
                     uint32_t *src, uint32_t *dst, void *stream) {
    k_rmat<<<grid(m), 256, 0, (cudaStream_t)stream>>>(m, scale, stream_key(seed, 1), t1, t2, t3, A, B, src, dst);
    return (int)cudaGetLastError();
}

GEN_API int gen_er(uint64_t n, uint64_t m, uint64_t seed, uint32_t *src, uint32_t *dst, void *stream) {
    k_er<<<grid(m), 256, 0, (cudaStream_t)stream>>>(m, n, stream_key(seed, 2), src, dst);
    return (int)cudaGetLastError();
}

GEN_API int gen_labels(uint64_t n, uint32_t S, uint64_t seed, uint32_t *lab, void *stream) {
    k_labels<<<grid(n), 256, 0, (cudaStream_t)stream>>>(n, S, stream_key(seed, 3), lab);
    return (int)cudaGetLastError();
}

GEN_API int gen_neighbors(uint64_t m, const uint32_t *src, const uint32_t *dst, uint32_t v, uint32_t *out,
                          unsigned long long *cnt, uint64_t cap, void *stream) {
    k_neighbors<<<grid(m), 256, 0, (cudaStream_t)stream>>>(m, src, dst, v, out, cnt, cap);
    return (int)cudaGetLastError();
}

GEN_API int gen_incident(uint64_t m, const uint32_t *src, const uint32_t *dst, const uint32_t *bits,
                         uint32_t *out_s, uint32_t *out_d, unsigned long long *cnt, uint64_t cap, void *stream) {
    k_incident<<<grid(m), 256, 0, (cudaStream_t)stream>>>(m, src, dst, bits, out_s, out_d, cnt, cap);
    return (int)cudaGetLastError();
}
