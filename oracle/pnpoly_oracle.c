/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the PnPoly kernel.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this; the product path never does.
 *
 * Parity status: UNPINNED by the reference. /root/reference (jouletune) has
 * no PnPoly code at all; the algorithm restated here is
 * the paper's Kernel-Tuner PnPoly benchmark: the crossing-number test
 *
 *   inside ^= ((vy_k > py) != (vy_j > py)) && (px < x_k(py)),  j = k-1 (cyclic)
 *
 * evaluated in IEEE float32, one rounding per operation, no contraction
 * (build with -ffp-contract=off), with the three crossing formulas the
 * kernel offers (csrc/kernels/pnpoly.cu METHOD):
 *   0: x = (dx * (py - vy_k)) / dy + vx_k
 *   1: x = fmaf(slope, py - vy_k, vx_k)          slope = dx / dy
 *   2: x = fmaf(slope, py, icpt)                 icpt  = fmaf(-slope, vy_k, vx_k)
 * with dx = vx_j - vx_k, dy = vy_j - vy_k, and
 *   3: formula 2 with every comparison taken as the sign bit of an exactly
 *      rounded float32 difference: crossing = sign((py - vy_k) ^ (py - vy_j))
 *      & sign(px - x). Equal to formula 2 unless a coordinate is -0.0.
 * The edge table is rebuilt here independently from the raw vertices.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static float edge_x(int method, float vxk, float vyk, float dx, float dy, float slope, float icpt, float py) {
    if (method == 0) {
        volatile float t = py - vyk;
        volatile float m = dx * t;
        volatile float q = m / dy;
        return q + vxk;
    }
    if (method == 1) {
        volatile float t = py - vyk;
        return fmaf(slope, t, vxk);
    }
    return fmaf(slope, py, icpt);
}

typedef struct {
    const float *points, *vx, *vy, *dx, *dy, *sl, *ic;
    long long begin, end;
    int nv, method;
    int32_t *out;
} span_t;

static uint32_t bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

static void *run_span(void *arg) {
    const span_t *s = (const span_t *)arg;
    const int nv = s->nv;
    if (s->method == 3) {
        for (long long i = s->begin; i < s->end; ++i) {
            const float px = s->points[2 * i], py = s->points[2 * i + 1];
            volatile float dprev = py - s->vy[nv - 1];
            uint32_t acc = 0;
            for (int k = 0; k < nv; ++k) {
                volatile float d = py - s->vy[k];
                volatile float x = fmaf(s->sl[k], py, s->ic[k]);
                volatile float e = px - x;
                acc ^= (bits(d) ^ bits(dprev)) & bits(e);
                dprev = d;
            }
            s->out[i] = (int32_t)(acc >> 31);
        }
        return 0;
    }
    for (long long i = s->begin; i < s->end; ++i) {
        const float px = s->points[2 * i], py = s->points[2 * i + 1];
        int c = 0;
        for (int k = 0, j = nv - 1; k < nv; j = k++) {
            if ((s->vy[k] > py) != (s->vy[j] > py)) {
                if (px < edge_x(s->method, s->vx[k], s->vy[k], s->dx[k], s->dy[k], s->sl[k], s->ic[k], py)) c = !c;
            }
        }
        s->out[i] = c;
    }
    return 0;
}

/* points: n x 2 float32 (x, y interleaved); vx, vy: nv vertices; out: n int32.
 * `threads` host threads split the points into contiguous spans. */
int pnpoly_oracle(const float *points, long long n, const float *vx, const float *vy, int nv, int method,
                  int32_t *out, int threads) {
    if (nv < 3 || method < 0 || method > 3) return 1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    float *dx = malloc(sizeof(float) * nv), *dy = malloc(sizeof(float) * nv);
    float *sl = malloc(sizeof(float) * nv), *ic = malloc(sizeof(float) * nv);
    if (!dx || !dy || !sl || !ic) return 2;
    for (int k = 0; k < nv; ++k) {
        int j = (k + nv - 1) % nv;
        dx[k] = vx[j] - vx[k];
        dy[k] = vy[j] - vy[k];
        volatile float s = dx[k] / dy[k];
        sl[k] = s;
        ic[k] = fmaf(-sl[k], vy[k], vx[k]);
    }
    pthread_t tid[256];
    span_t span[256];
    long long chunk = (n + threads - 1) / threads;
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        long long b = t * chunk, e = b + chunk < n ? b + chunk : n;
        span[t] = (span_t){points, vx, vy, dx, dy, sl, ic, b, e > b ? e : b, nv, method, out};
        if (threads == 1) {
            run_span(&span[t]);
        } else if (pthread_create(&tid[t], 0, run_span, &span[t]) == 0) {
            ++started;
        } else {
            run_span(&span[t]);
            tid[t] = 0;
        }
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t)
            if (tid[t]) pthread_join(tid[t], 0);
    free(dx);
    free(dy);
    free(sl);
    free(ic);
    return 0;
}
