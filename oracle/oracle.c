/*
 * oracle.c -- CPU float64 DIRECT (spatial) convolution oracle for the OaA layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_1601_06815_b200/csrc).
 *
 * What it computes is the plain definition of the convolution layer that OaA
 * reaches exactly ("create the same results as a traditional spacial
 * convolution", PAPER.md:18 (§2); "the methods are equivalent"
 * (§3.1, Table 2)).  Every sum is written out as the definition, in float64,
 * with no blocking, transform or reordering:
 *
 *   forward   (§1 "KC convolutions"; SPEC.md:205 true convolution,
 *              SPEC.md:188 crop):
 *       Full[b,k,I,J] = sum_c sum_{u,v} x[b,c,I-u,J-v] * w[k,c,u,v]   (x = 0 outside)
 *       y[b,k,i,j]    = Full[b,k,i+o,j+o]
 *   bwd_data  ("one convolution to propagate the error"):
 *       dx[b,c,a1,a2] = sum_k sum_{u,v} G[b,k,a1+u,a2+v] * w[k,c,u,v]
 *       with G[b,k] the (N+n-1)^2 frame holding dy at [o,o+M)^2 and 0 elsewhere
 *   bwd_filter ("another to calculate the change in weight"):
 *       dw[k,c,u,v]   = sum_b sum_{a1,a2} x[b,c,a1,a2] * G[b,k,a1+u,a2+v]
 *
 * bwd_data / bwd_filter are the exact adjoints of the forward map (the layer's
 * gradients); tests pin them with the dot-product identity, torch autograd and
 * finite differences (tests/test_oracle_direct.py).
 *
 * Crop (reading R5/R6): 0 = Full (M = N+n-1, o = 0),
 * 1 = Valid (M = N-n+1, o = n-1), 2 = Same (M = N, o = floor((n-1)/2)).
 * Shapes may be rectangular (rows, cols) so SPEC's 1-D embedded examples
 * are expressible; the product ABI is square.
 *
 * Parallelism: OpenMP over independent outputs only (each output element is one
 * thread's plain sum), so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- crop bookkeeping ------------------------------------ */
int oracle_out_size(int N, int n, int crop) {
    if (N < 1 || n < 1) return -1;
    if (crop == 0) return N + n - 1;
    if (crop == 1) return (n <= N) ? N - n + 1 : -1;
    if (crop == 2) return N;
    return -1;
}
int oracle_crop_offset(int n, int crop) {
    if (crop == 0) return 0;
    if (crop == 1) return n - 1;
    if (crop == 2) return (n - 1) / 2;
    return -1;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- forward: y = crop(Full(x * w)) ------------------------------------ */
/* x[B][C][Nr][Nc], w[K][C][nr][nc], y[B][K][Mr][Mc]                          */
static double fwd_elem(const double* x, const double* w, int C, int Nr, int Nc,
                       int nr, int nc, int b, int k, int I, int J) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) {
        const double* xc = x + ((size_t)b * C + c) * Nr * Nc;
        const double* wk = w + ((size_t)k * C + c) * nr * nc;
        for (int u = 0; u < nr; ++u) {
            int r = I - u;
            if (r < 0 || r >= Nr) continue;
            for (int v = 0; v < nc; ++v) {
                int q = J - v;
                if (q < 0 || q >= Nc) continue;
                s += xc[(size_t)r * Nc + q] * wk[u * nc + v];
            }
        }
    }
    return s;
}

int oracle_conv_fwd_rect(const double* x, const double* w, double* y, int B, int C, int K,
                         int Nr, int Nc, int nr, int nc, int crop, int nthreads) {
    int Mr = oracle_out_size(Nr, nr, crop), Mc = oracle_out_size(Nc, nc, crop);
    if (Mr < 1 || Mc < 1) return -1;
    int orr = oracle_crop_offset(nr, crop), oc = oracle_crop_offset(nc, crop);
    set_threads(nthreads);
    long total = (long)B * K * Mr;
#pragma omp parallel for schedule(dynamic, 4)
    for (long t = 0; t < total; ++t) {
        int i = (int)(t % Mr);
        int k = (int)((t / Mr) % K);
        int b = (int)(t / ((long)Mr * K));
        double* yr = y + (((size_t)b * K + k) * Mr + i) * Mc;
        for (int j = 0; j < Mc; ++j) yr[j] = fwd_elem(x, w, C, Nr, Nc, nr, nc, b, k, i + orr, j + oc);
    }
    return 0;
}

int oracle_conv_fwd(const double* x, const double* w, double* y, int B, int C, int K, int N,
                    int n, int crop, int nthreads) {
    return oracle_conv_fwd_rect(x, w, y, B, C, K, N, N, n, n, crop, nthreads);
}

/* ---- bwd_data: dx[b,c,a] = sum_k sum_{u,v} G[b,k,a+(u,v)] w[k,c,u,v] ------ */
/* G[b,k,p] = dy[b,k,p-o] if p-o in [0,M) else 0                              */
static double bwd_data_elem(const double* dy, const double* w, int C, int K, int Mr, int Mc,
                            int nr, int nc, int orr, int oc, int b, int c, int a1, int a2) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) {
        const double* g = dy + ((size_t)b * K + k) * Mr * Mc;
        const double* wk = w + ((size_t)k * C + c) * nr * nc;
        for (int u = 0; u < nr; ++u) {
            int r = a1 + u - orr;
            if (r < 0 || r >= Mr) continue;
            for (int v = 0; v < nc; ++v) {
                int q = a2 + v - oc;
                if (q < 0 || q >= Mc) continue;
                s += g[(size_t)r * Mc + q] * wk[u * nc + v];
            }
        }
    }
    return s;
}

int oracle_conv_bwd_data_rect(const double* dy, const double* w, double* dx, int B, int C,
                              int K, int Nr, int Nc, int nr, int nc, int crop, int nthreads) {
    int Mr = oracle_out_size(Nr, nr, crop), Mc = oracle_out_size(Nc, nc, crop);
    if (Mr < 1 || Mc < 1) return -1;
    int orr = oracle_crop_offset(nr, crop), oc = oracle_crop_offset(nc, crop);
    set_threads(nthreads);
    long total = (long)B * C * Nr;
#pragma omp parallel for schedule(dynamic, 4)
    for (long t = 0; t < total; ++t) {
        int a1 = (int)(t % Nr);
        int c = (int)((t / Nr) % C);
        int b = (int)(t / ((long)Nr * C));
        double* row = dx + (((size_t)b * C + c) * Nr + a1) * Nc;
        for (int a2 = 0; a2 < Nc; ++a2)
            row[a2] = bwd_data_elem(dy, w, C, K, Mr, Mc, nr, nc, orr, oc, b, c, a1, a2);
    }
    return 0;
}

int oracle_conv_bwd_data(const double* dy, const double* w, double* dx, int B, int C, int K,
                         int N, int n, int crop, int nthreads) {
    return oracle_conv_bwd_data_rect(dy, w, dx, B, C, K, N, N, n, n, crop, nthreads);
}

/* ---- bwd_filter: dw[k,c,u,v] = sum_b sum_a x[b,c,a] G[b,k,a+(u,v)] ------- */
static double bwd_filter_elem(const double* x, const double* dy, int B, int C, int K, int Nr,
                              int Nc, int Mr, int Mc, int orr, int oc, int k, int c, int u,
                              int v) {
    double s = 0.0;
    for (int b = 0; b < B; ++b) {
        const double* xc = x + ((size_t)b * C + c) * Nr * Nc;
        const double* g = dy + ((size_t)b * K + k) * Mr * Mc;
        for (int a1 = 0; a1 < Nr; ++a1) {
            int r = a1 + u - orr;
            if (r < 0 || r >= Mr) continue;
            for (int a2 = 0; a2 < Nc; ++a2) {
                int q = a2 + v - oc;
                if (q < 0 || q >= Mc) continue;
                s += xc[(size_t)a1 * Nc + a2] * g[(size_t)r * Mc + q];
            }
        }
    }
    return s;
}

int oracle_conv_bwd_filter_rect(const double* x, const double* dy, double* dw, int B, int C,
                                int K, int Nr, int Nc, int nr, int nc, int crop, int nthreads) {
    int Mr = oracle_out_size(Nr, nr, crop), Mc = oracle_out_size(Nc, nc, crop);
    if (Mr < 1 || Mc < 1) return -1;
    int orr = oracle_crop_offset(nr, crop), oc = oracle_crop_offset(nc, crop);
    set_threads(nthreads);
    long total = (long)K * C * nr * nc;
#pragma omp parallel for schedule(dynamic, 1)
    for (long t = 0; t < total; ++t) {
        int v = (int)(t % nc);
        int u = (int)((t / nc) % nr);
        int c = (int)((t / ((long)nc * nr)) % C);
        int k = (int)(t / ((long)nc * nr * C));
        dw[t] = bwd_filter_elem(x, dy, B, C, K, Nr, Nc, Mr, Mc, orr, oc, k, c, u, v);
    }
    return 0;
}

int oracle_conv_bwd_filter(const double* x, const double* dy, double* dw, int B, int C, int K,
                           int N, int n, int crop, int nthreads) {
    return oracle_conv_bwd_filter_rect(x, dy, dw, B, C, K, N, N, n, n, crop, nthreads);
}

/* ---- sampled single-element evaluation on fp32 inputs -------------------
 * For parity checks at full BASELINE sizes, where the whole oracle output is
 * too slow: the same definitions evaluated one element at a time, reading the
 * fp32 input values directly (promoted to double per term).                 */
static double fwd_elem_f(const float* x, const float* w, int C, int N, int n, int b, int k,
                         int I, int J) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) {
        const float* xc = x + ((size_t)b * C + c) * N * N;
        const float* wk = w + ((size_t)k * C + c) * n * n;
        for (int u = 0; u < n; ++u) {
            int r = I - u;
            if (r < 0 || r >= N) continue;
            for (int v = 0; v < n; ++v) {
                int q = J - v;
                if (q < 0 || q >= N) continue;
                s += (double)xc[(size_t)r * N + q] * (double)wk[u * n + v];
            }
        }
    }
    return s;
}

/* idx: count tuples (b, k, i, j) in cropped output coordinates */
int oracle_fwd_sample(const float* x, const float* w, int B, int C, int K, int N, int n,
                      int crop, const int64_t* idx, long count, double* out, int nthreads) {
    int M = oracle_out_size(N, n, crop);
    if (M < 1) return -1;
    int o = oracle_crop_offset(n, crop);
    set_threads(nthreads);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (long s = 0; s < count; ++s) {
        int b = (int)idx[4 * s], k = (int)idx[4 * s + 1], i = (int)idx[4 * s + 2],
            j = (int)idx[4 * s + 3];
        if (b < 0 || b >= B || k < 0 || k >= K || i < 0 || i >= M || j < 0 || j >= M) {
            bad = 1;
            out[s] = NAN;
            continue;
        }
        out[s] = fwd_elem_f(x, w, C, N, n, b, k, i + o, j + o);
    }
    return bad ? -2 : 0;
}

/* idx: (b, c, a1, a2) */
int oracle_bwd_data_sample(const float* dy, const float* w, int B, int C, int K, int N, int n,
                           int crop, const int64_t* idx, long count, double* out,
                           int nthreads) {
    int M = oracle_out_size(N, n, crop);
    if (M < 1) return -1;
    int o = oracle_crop_offset(n, crop);
    set_threads(nthreads);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (long s = 0; s < count; ++s) {
        int b = (int)idx[4 * s], c = (int)idx[4 * s + 1], a1 = (int)idx[4 * s + 2],
            a2 = (int)idx[4 * s + 3];
        if (b < 0 || b >= B || c < 0 || c >= C || a1 < 0 || a1 >= N || a2 < 0 || a2 >= N) {
            bad = 1;
            out[s] = NAN;
            continue;
        }
        double acc = 0.0;
        for (int k = 0; k < K; ++k) {
            const float* g = dy + ((size_t)b * K + k) * M * M;
            const float* wk = w + ((size_t)k * C + c) * n * n;
            for (int u = 0; u < n; ++u) {
                int r = a1 + u - o;
                if (r < 0 || r >= M) continue;
                for (int v = 0; v < n; ++v) {
                    int q = a2 + v - o;
                    if (q < 0 || q >= M) continue;
                    acc += (double)g[(size_t)r * M + q] * (double)wk[u * n + v];
                }
            }
        }
        out[s] = acc;
    }
    return bad ? -2 : 0;
}

/* idx: (k, c, u, v); each element sums over the whole batch */
int oracle_bwd_filter_sample(const float* x, const float* dy, int B, int C, int K, int N,
                             int n, int crop, const int64_t* idx, long count, double* out,
                             int nthreads) {
    int M = oracle_out_size(N, n, crop);
    if (M < 1) return -1;
    int o = oracle_crop_offset(n, crop);
    set_threads(nthreads);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
    for (long s = 0; s < count; ++s) {
        int k = (int)idx[4 * s], c = (int)idx[4 * s + 1], u = (int)idx[4 * s + 2],
            v = (int)idx[4 * s + 3];
        if (k < 0 || k >= K || c < 0 || c >= C || u < 0 || u >= n || v < 0 || v >= n) {
            bad = 1;
            out[s] = NAN;
            continue;
        }
        double acc = 0.0;
        for (int b = 0; b < B; ++b) {
            const float* xc = x + ((size_t)b * C + c) * N * N;
            const float* g = dy + ((size_t)b * K + k) * M * M;
            for (int a1 = 0; a1 < N; ++a1) {
                int r = a1 + u - o;
                if (r < 0 || r >= M) continue;
                for (int a2 = 0; a2 < N; ++a2) {
                    int q = a2 + v - o;
                    if (q < 0 || q >= M) continue;
                    acc += (double)xc[(size_t)a1 * N + a2] * (double)g[(size_t)r * M + q];
                }
            }
        }
        out[s] = acc;
    }
    return bad ? -2 : 0;
}

/* ---- whole-layer step on fp32 inputs, for the CPU baseline ---------------
 * One fwd + bwd_data + bwd_filter over B images, reading fp32 inputs and
 * writing fp64 outputs: exactly the three definitions above, used by bench.py
 * to time "the oracle as it stands" on the host cores.                      */
int oracle_step_f32(const float* x, const float* w, const float* dy, double* y, double* dx,
                    double* dw, int B, int C, int K, int N, int n, int crop, int nthreads) {
    int M = oracle_out_size(N, n, crop);
    if (M < 1) return -1;
    int o = oracle_crop_offset(n, crop);
    set_threads(nthreads);
    long tot_y = (long)B * K * M;
#pragma omp parallel for schedule(dynamic, 4)
    for (long t = 0; t < tot_y; ++t) {
        int i = (int)(t % M), k = (int)((t / M) % K), b = (int)(t / ((long)M * K));
        double* yr = y + (((size_t)b * K + k) * M + i) * M;
        for (int j = 0; j < M; ++j) yr[j] = fwd_elem_f(x, w, C, N, n, b, k, i + o, j + o);
    }
    long tot_dx = (long)B * C * N;
#pragma omp parallel for schedule(dynamic, 4)
    for (long t = 0; t < tot_dx; ++t) {
        int a1 = (int)(t % N), c = (int)((t / N) % C), b = (int)(t / ((long)N * C));
        double* row = dx + (((size_t)b * C + c) * N + a1) * N;
        for (int a2 = 0; a2 < N; ++a2) {
            double acc = 0.0;
            for (int k = 0; k < K; ++k) {
                const float* g = dy + ((size_t)b * K + k) * M * M;
                const float* wk = w + ((size_t)k * C + c) * n * n;
                for (int u = 0; u < n; ++u) {
                    int r = a1 + u - o;
                    if (r < 0 || r >= M) continue;
                    for (int v = 0; v < n; ++v) {
                        int q = a2 + v - o;
                        if (q < 0 || q >= M) continue;
                        acc += (double)g[(size_t)r * M + q] * (double)wk[u * n + v];
                    }
                }
            }
            row[a2] = acc;
        }
    }
    long tot_dw = (long)K * C * n * n;
#pragma omp parallel for schedule(dynamic, 1)
    for (long t = 0; t < tot_dw; ++t) {
        int v = (int)(t % n), u = (int)((t / n) % n), c = (int)((t / ((long)n * n)) % C),
            k = (int)(t / ((long)n * n * C));
        double acc = 0.0;
        for (int b = 0; b < B; ++b) {
            const float* xc = x + ((size_t)b * C + c) * N * N;
            const float* g = dy + ((size_t)b * K + k) * M * M;
            for (int a1 = 0; a1 < N; ++a1) {
                int r = a1 + u - o;
                if (r < 0 || r >= M) continue;
                for (int a2 = 0; a2 < N; ++a2) {
                    int q = a2 + v - o;
                    if (q < 0 || q >= M) continue;
                    acc += (double)xc[(size_t)a1 * N + a2] * (double)g[(size_t)r * M + q];
                }
            }
        }
        dw[t] = acc;
    }
    return 0;
}
