/*
 * tc_philox.h — counter-based random numbers shared by host, device and the
 * CPU oracle, so every side draws identical synthetic inputs, initial
 * parameters and dropout masks without transferring them.
 *
 *   Philox-4x32-10 (Salmon et al., SC'11), key = (seed, stream), 128-bit counter.
 *
 * Streams and counters:
 *   labels     y_n      = philox(seed, LABEL,    {n_global, iter, 0, 0})[0] mod K
 *   centroids  mu_k[e]  = u01(philox(seed, CENTROID, {e/4, k, 0, 0})[e%4])
 *   images     x_n[e]   = mu_{y_n}[e] + 0.1 * z,  z = Box-Muller of
 *                         philox(seed, IMAGE, {e/2, n_global, iter, 0})[0..1], cos for even e, sin for odd
 *   params     Xavier   U(-a, a), a = sqrt(6/(fan_in+fan_out)) from philox(seed, PARAM+i, {j/4,0,0,0})[j%4]
 *   dropout    keep     = u01(philox(seed, DROPOUT+var, {e/4, n_global, iter, 0})[e%4]) >= rate
 *              value    = keep ? 1/(1-rate) : 0          (inverted dropout; e = element within a sample)
 * u01(r) = ((r >> 8) + 0.5) * 2^-24 is exact in fp32, so masks are bit-identical everywhere.
 */
#ifndef TC_PHILOX_H
#define TC_PHILOX_H

#include <stdint.h>

#if defined(__CUDACC__)
#define TCP_FN __host__ __device__ __forceinline__
#else
#define TCP_FN static inline
#endif

enum { TCP_STREAM_LABEL = 1, TCP_STREAM_CENTROID = 2, TCP_STREAM_IMAGE = 3, TCP_STREAM_PARAM = 0x100,
       TCP_STREAM_DROPOUT = 0x100000 };

typedef struct tcp_u4 { uint32_t x, y, z, w; } tcp_u4;

TCP_FN uint32_t tcp_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
    const uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    return (uint32_t)p;
}

TCP_FN tcp_u4 tcp_philox(uint32_t k0, uint32_t k1, tcp_u4 c) {
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        const uint32_t lo0 = tcp_mulhilo(0xD2511F53u, c.x, &hi0);
        const uint32_t lo1 = tcp_mulhilo(0xCD9E8D57u, c.z, &hi1);
        tcp_u4 n;
        n.x = hi1 ^ c.y ^ k0;
        n.y = lo1;
        n.z = hi0 ^ c.w ^ k1;
        n.w = lo0;
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

TCP_FN uint32_t tcp_word(tcp_u4 v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

TCP_FN float tcp_u01(uint32_t r) { return ((float)(r >> 8) + 0.5f) * (1.0f / 16777216.0f); }

TCP_FN tcp_u4 tcp_draw(uint64_t seed, uint32_t stream, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    tcp_u4 c;
    c.x = c0; c.y = c1; c.z = c2; c.w = c3;
    return tcp_philox((uint32_t)seed, (uint32_t)(seed >> 32) ^ stream, c);
}

TCP_FN uint32_t tcp_label(uint64_t seed, uint32_t n_global, uint32_t iter, uint32_t classes) {
    return tcp_draw(seed, TCP_STREAM_LABEL, n_global, iter, 0, 0).x % classes;
}

TCP_FN float tcp_centroid(uint64_t seed, uint32_t k, uint32_t e) {
    return tcp_u01(tcp_word(tcp_draw(seed, TCP_STREAM_CENTROID, e >> 2, k, 0, 0), (int)(e & 3)));
}

/* Standard normal for element e of sample n at iteration iter (fp64 math on the host). */
TCP_FN void tcp_uniform_pair(uint64_t seed, uint32_t n_global, uint32_t iter, uint32_t e, float* u1, float* u2) {
    const tcp_u4 r = tcp_draw(seed, TCP_STREAM_IMAGE, e >> 1, n_global, iter, 0);
    *u1 = tcp_u01(r.x);
    *u2 = tcp_u01(r.y);
}

TCP_FN float tcp_dropout_value(uint64_t seed, uint32_t var, uint32_t n_global, uint32_t iter, uint32_t e, float rate) {
    const tcp_u4 r = tcp_draw(seed, TCP_STREAM_DROPOUT + var, e >> 2, n_global, iter, 0);
    return tcp_u01(tcp_word(r, (int)(e & 3))) >= rate ? 1.0f / (1.0f - rate) : 0.0f;
}

TCP_FN float tcp_param_uniform(uint64_t seed, uint32_t param_index, uint32_t j) {
    return tcp_u01(tcp_word(tcp_draw(seed, TCP_STREAM_PARAM + param_index, j >> 2, 0, 0, 0), (int)(j & 3)));
}

#endif /* TC_PHILOX_H */
