/*
 * oracle.c -- plain single-threaded CPU oracle (TEST INFRASTRUCTURE ONLY; see
 * oracle.h).  Every function is the plain definition written out as a loop
 * over edges in ascending edge id, with double accumulation and a single
 * rounding to float at the end.  No blocking, fusion or reordering.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see
 * oracle/__init__.py).  -ffp-contract=off keeps "w * x" a single float
 * multiply for the MAX path (reading Q4/Q10): the argmax decision is taken on
 * the float message the GPU also computes.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int check_index(const int64_t* idx, int64_t E, int64_t n) {
    for (int64_t k = 0; k < E; ++k)
        if (idx[k] < 0 || idx[k] >= n) return ORC_ERR_OOB;
    return ORC_OK;
}

int orc_degree(const int64_t* index, int64_t E, int64_t n, int64_t* deg) {
    if (E < 0 || n < 0 || (E > 0 && !index) || (n > 0 && !deg)) return ORC_ERR_INVALID;
    if (check_index(index, E, n)) return ORC_ERR_OOB;
    for (int64_t i = 0; i < n; ++i) deg[i] = 0;
    for (int64_t k = 0; k < E; ++k) deg[index[k]] += 1; /* count of incident edges */
    return ORC_OK;
}

int orc_csr(const int64_t* dst, int64_t E, int64_t n, int64_t* rowptr, int64_t* perm) {
    if (E < 0 || n < 0 || !rowptr || (E > 0 && (!dst || !perm))) return ORC_ERR_INVALID;
    if (check_index(dst, E, n)) return ORC_ERR_OOB;
    /* counting sort: rowptr = exclusive prefix sum of in-degrees */
    for (int64_t i = 0; i <= n; ++i) rowptr[i] = 0;
    for (int64_t k = 0; k < E; ++k) rowptr[dst[k] + 1] += 1;
    for (int64_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
    int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!next) return ORC_ERR_INVALID;
    for (int64_t i = 0; i < n; ++i) next[i] = rowptr[i];
    for (int64_t k = 0; k < E; ++k) perm[next[dst[k]]++] = k; /* ascending k => stable */
    free(next);
    return ORC_OK;
}

/* ---- the reduction core shared by scatter / propagate / pooling --------- */
/* The caller supplies, for edge k and output column c, the message value as
 * a float (what MAX compares, reading Q4) and as a double (what SUM/MEAN
 * accumulate: the exact product for weighted messages). */
typedef struct {
    /* propagate inputs */
    const float* x_src; int64_t ldx;
    const float* x_dst; int64_t ldxd;
    const float* edge_attr; int64_t D;
    const float* w;
    int64_t F; int concat_xi;
    /* scatter input */
    const float* src; int64_t lds;
    const int64_t* src_idx; /* NULL for scatter */
    const int64_t* dst_idx;
} msg_ctx;

/* Column layout of the propagate message: [x_i (F, if concat) | w x_j (F) | e (D)] */
static void message(const msg_ctx* m, int64_t k, int64_t c, float* mf, double* md) {
    if (!m->src_idx) { /* scatter: the message is the edge-space row itself */
        float v = m->src[k * m->lds + c];
        *mf = v; *md = (double)v;
        return;
    }
    int64_t j = m->src_idx[k], i = m->dst_idx[k];
    int64_t off = 0;
    if (m->concat_xi) {
        if (c < m->F) {
            const float* xd = m->x_dst ? m->x_dst : m->x_src;
            int64_t ld = m->x_dst ? m->ldxd : m->ldx;
            float v = xd[i * ld + c];
            *mf = v; *md = (double)v;
            return;
        }
        off = m->F;
    }
    if (c < off + m->F) {
        float x = m->x_src[j * m->ldx + (c - off)];
        if (m->w) {
            float wk = m->w[k];
            *mf = wk * x;                     /* one float multiply (MAX decision) */
            *md = (double)wk * (double)x;      /* exact product (SUM / MEAN) */
        } else {
            *mf = x; *md = (double)x;
        }
        return;
    }
    float e = m->edge_attr[k * m->D + (c - off - m->F)];
    *mf = e; *md = (double)e;
}

static int reduce_core(const msg_ctx* m, int64_t E, int64_t n_out, int64_t F_out, int reduce,
                       float* out, int64_t* arg, double* abs_sum) {
    size_t cells = (size_t)n_out * (size_t)F_out;
    int64_t* deg = (int64_t*)calloc((size_t)(n_out > 0 ? n_out : 1), sizeof(int64_t));
    if (!deg) return ORC_ERR_INVALID;
    for (int64_t k = 0; k < E; ++k) deg[m->dst_idx[k]] += 1;
    if (abs_sum)
        for (size_t t = 0; t < cells; ++t) abs_sum[t] = 0.0;

    if (reduce == ORC_SUM || reduce == ORC_MEAN) {
        double* acc = (double*)calloc(cells ? cells : 1, sizeof(double));
        if (!acc) { free(deg); return ORC_ERR_INVALID; }
        for (int64_t k = 0; k < E; ++k) {
            int64_t i = m->dst_idx[k];
            for (int64_t c = 0; c < F_out; ++c) {
                float mf; double md;
                message(m, k, c, &mf, &md);
                acc[i * F_out + c] += md;
                if (abs_sum) abs_sum[i * F_out + c] += fabs(md);
            }
        }
        for (int64_t i = 0; i < n_out; ++i)
            for (int64_t c = 0; c < F_out; ++c) {
                double a = acc[i * F_out + c];
                if (reduce == ORC_MEAN) /* mean = sum / integer in-degree; deg 0 -> 0 (Q6) */
                    out[i * F_out + c] = deg[i] > 0 ? (float)(a / (double)deg[i]) : 0.0f;
                else
                    out[i * F_out + c] = (float)a;
                if (abs_sum && reduce == ORC_MEAN && deg[i] > 0)
                    abs_sum[i * F_out + c] /= (double)deg[i];
            }
        free(acc);
    } else if (reduce == ORC_MAX) {
        /* scan k ascending; take m if the segment is empty so far or m > best
         * (strict IEEE) => arg = lowest edge id among equal maxima (Q4);
         * empty segment -> out 0, arg E (Q2, Q3). */
        float* best = (float*)malloc((cells ? cells : 1) * sizeof(float));
        if (!best) { free(deg); return ORC_ERR_INVALID; }
        for (size_t t = 0; t < cells; ++t) { best[t] = 0.0f; arg[t] = E; }
        for (int64_t k = 0; k < E; ++k) {
            int64_t i = m->dst_idx[k];
            for (int64_t c = 0; c < F_out; ++c) {
                float mf; double md;
                message(m, k, c, &mf, &md);
                size_t t = (size_t)(i * F_out + c);
                if (arg[t] == E || mf > best[t]) { best[t] = mf; arg[t] = k; }
            }
        }
        for (size_t t = 0; t < cells; ++t) out[t] = (arg[t] == E) ? 0.0f : best[t];
        free(best);
    } else {
        free(deg);
        return ORC_ERR_INVALID;
    }
    free(deg);
    return ORC_OK;
}

int orc_scatter(const float* src, int64_t E, int64_t F, int64_t lds, const int64_t* index,
                int64_t dim_size, int reduce, float* out, int64_t* arg, double* abs_sum) {
    if (E < 0 || F < 0 || dim_size < 0 || lds < F) return ORC_ERR_DIMENSION;
    if (reduce < ORC_SUM || reduce > ORC_MAX) return ORC_ERR_INVALID;
    if ((E > 0 && (!index || (F > 0 && !src))) || (dim_size * F > 0 && !out)) return ORC_ERR_INVALID;
    if (reduce == ORC_MAX && dim_size * F > 0 && !arg) return ORC_ERR_INVALID;
    if (check_index(index, E, dim_size)) return ORC_ERR_OOB;
    msg_ctx m;
    memset(&m, 0, sizeof m);
    m.src = src; m.lds = lds; m.dst_idx = index; m.F = F;
    return reduce_core(&m, E, dim_size, F, reduce, out, arg, abs_sum);
}

int orc_propagate(const float* x_src, int64_t n_src, int64_t F, int64_t ldx, const float* x_dst,
                  int64_t ldxd, int64_t n_dst, const int64_t* edge_index, int64_t E,
                  const float* edge_attr, int64_t D, const float* edge_weight, int reduce,
                  int concat_xi, float* out, int64_t* arg, double* abs_sum) {
    if (E < 0 || F < 0 || D < 0 || n_src < 0 || n_dst < 0 || ldx < F) return ORC_ERR_DIMENSION;
    if (x_dst && ldxd < F) return ORC_ERR_DIMENSION;
    if (concat_xi && !x_dst && n_dst > n_src) return ORC_ERR_DIMENSION;
    if (reduce < ORC_SUM || reduce > ORC_MAX) return ORC_ERR_INVALID;
    if (D > 0 && E > 0 && !edge_attr) return ORC_ERR_INVALID;
    int64_t F_out = (concat_xi ? F : 0) + F + D;
    if (n_dst * F_out > 0 && !out) return ORC_ERR_INVALID;
    if (reduce == ORC_MAX && n_dst * F_out > 0 && !arg) return ORC_ERR_INVALID;
    if (E > 0 && !edge_index) return ORC_ERR_INVALID;
    const int64_t* src_idx = edge_index;
    const int64_t* dst_idx = edge_index + E;
    if (check_index(src_idx, E, n_src) || check_index(dst_idx, E, n_dst)) return ORC_ERR_OOB;
    msg_ctx m;
    memset(&m, 0, sizeof m);
    m.x_src = x_src; m.ldx = ldx; m.x_dst = x_dst; m.ldxd = ldxd;
    m.edge_attr = edge_attr; m.D = D; m.w = edge_weight; m.F = F; m.concat_xi = concat_xi;
    m.src_idx = src_idx; m.dst_idx = dst_idx;
    return reduce_core(&m, E, n_dst, F_out, reduce, out, arg, abs_sum);
}

int orc_scatter_backward(const float* grad_out, int64_t F, const int64_t* index, int64_t E,
                         int64_t dim_size, int reduce, const int64_t* arg, float* grad_src) {
    if (E < 0 || F < 0 || dim_size < 0) return ORC_ERR_DIMENSION;
    if (reduce < ORC_SUM || reduce > ORC_MAX) return ORC_ERR_INVALID;
    if (reduce == ORC_MAX && dim_size * F > 0 && !arg) return ORC_ERR_INVALID;
    if (check_index(index, E, dim_size)) return ORC_ERR_OOB;
    int64_t* deg = (int64_t*)calloc((size_t)(dim_size > 0 ? dim_size : 1), sizeof(int64_t));
    if (!deg) return ORC_ERR_INVALID;
    for (int64_t k = 0; k < E; ++k) deg[index[k]] += 1;
    for (int64_t k = 0; k < E; ++k) {
        int64_t i = index[k];
        for (int64_t c = 0; c < F; ++c) {
            float g = grad_out[i * F + c];
            float r;
            if (reduce == ORC_SUM) r = g;                         /* gather of grad */
            else if (reduce == ORC_MEAN) r = g / (float)deg[i];   /* scaled by 1/count */
            else r = (arg[i * F + c] == k) ? g : 0.0f;             /* routed to argmax */
            grad_src[k * F + c] = r;
        }
    }
    free(deg);
    return ORC_OK;
}

int orc_propagate_backward(const float* x_src, int64_t n_src, int64_t F, int64_t ldx,
                           int64_t n_dst, const int64_t* edge_index, int64_t E, int64_t D,
                           const float* edge_weight, int reduce, int concat_xi,
                           const float* grad_out, const int64_t* arg, float* grad_x_src,
                           float* grad_x_dst, float* grad_edge_attr, float* grad_edge_weight,
                           double* abs_sum_x_src) {
    if (E < 0 || F < 0 || D < 0 || n_src < 0 || n_dst < 0 || ldx < F) return ORC_ERR_DIMENSION;
    if (reduce < ORC_SUM || reduce > ORC_MAX) return ORC_ERR_INVALID;
    int64_t F_out = (concat_xi ? F : 0) + F + D;
    if (reduce == ORC_MAX && n_dst * F_out > 0 && !arg) return ORC_ERR_INVALID;
    if (grad_edge_weight && !x_src && E * F > 0) return ORC_ERR_INVALID;
    const int64_t* src_idx = edge_index;
    const int64_t* dst_idx = edge_index + E;
    if (check_index(src_idx, E, n_src) || check_index(dst_idx, E, n_dst)) return ORC_ERR_OOB;
    int64_t off1 = concat_xi ? F : 0, off2 = off1 + F;

    int64_t* deg = (int64_t*)calloc((size_t)(n_dst > 0 ? n_dst : 1), sizeof(int64_t));
    double* gxs = (double*)calloc((size_t)(n_src * F > 0 ? n_src * F : 1), sizeof(double));
    double* gxd = (double*)calloc((size_t)(n_dst * F > 0 ? n_dst * F : 1), sizeof(double));
    if (!deg || !gxs || !gxd) { free(deg); free(gxs); free(gxd); return ORC_ERR_INVALID; }
    for (int64_t k = 0; k < E; ++k) deg[dst_idx[k]] += 1;
    if (abs_sum_x_src)
        for (int64_t t = 0; t < n_src * F; ++t) abs_sum_x_src[t] = 0.0;

    for (int64_t k = 0; k < E; ++k) {
        int64_t j = src_idx[k], i = dst_idx[k];
        double wk = edge_weight ? (double)edge_weight[k] : 1.0;
        double gw = 0.0;
        for (int64_t c = 0; c < F_out; ++c) {
            /* dL/dm_k[c]: the adjoint of the reduction */
            double g = (double)grad_out[i * F_out + c];
            double gm;
            if (reduce == ORC_SUM) gm = g;
            else if (reduce == ORC_MEAN) gm = g / (double)deg[i];
            else gm = (arg[i * F_out + c] == k) ? g : 0.0;
            if (c < off1) {
                gxd[i * F + c] += gm;                       /* x_i block */
            } else if (c < off2) {
                double t = wk * gm;                         /* w_k x_j block */
                gxs[j * F + (c - off1)] += t;
                if (abs_sum_x_src) abs_sum_x_src[j * F + (c - off1)] += fabs(t);
                if (grad_edge_weight) gw += (double)x_src[j * ldx + (c - off1)] * gm;
            } else if (grad_edge_attr) {
                grad_edge_attr[k * D + (c - off2)] = (float)gm; /* e_ji block */
            }
        }
        if (grad_edge_weight) grad_edge_weight[k] = (float)gw;
    }
    if (grad_x_src)
        for (int64_t t = 0; t < n_src * F; ++t) grad_x_src[t] = (float)gxs[t];
    if (grad_x_dst && concat_xi)
        for (int64_t t = 0; t < n_dst * F; ++t) grad_x_dst[t] = (float)gxd[t];
    if (grad_edge_attr && E == 0) { /* nothing */ }
    free(deg); free(gxs); free(gxd);
    return ORC_OK;
}

int orc_gcn_norm(const int64_t* edge_index, int64_t E, int64_t N, const float* edge_weight,
                 int64_t* ei_src_out, int64_t* ei_dst_out, float* w_out, int64_t* E_out) {
    if (E < 0 || N < 0) return ORC_ERR_DIMENSION;
    const int64_t* src = edge_index;
    const int64_t* dst = edge_index + E;
    if (check_index(src, E, N) || check_index(dst, E, N)) return ORC_ERR_OOB;
    /* 1. add remaining self-loops (reading Q8) */
    char* has_loop = (char*)calloc((size_t)(N > 0 ? N : 1), 1);
    double* deg = (double*)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
    if (!has_loop || !deg) { free(has_loop); free(deg); return ORC_ERR_INVALID; }
    for (int64_t k = 0; k < E; ++k)
        if (src[k] == dst[k]) has_loop[src[k]] = 1;
    int64_t e = 0;
    for (int64_t k = 0; k < E; ++k) {
        ei_src_out[e] = src[k]; ei_dst_out[e] = dst[k];
        w_out[e] = edge_weight ? edge_weight[k] : 1.0f;
        ++e;
    }
    for (int64_t i = 0; i < N; ++i)
        if (!has_loop[i]) { ei_src_out[e] = i; ei_dst_out[e] = i; w_out[e] = 1.0f; ++e; }
    *E_out = e;
    /* 2. deg_hat[i] = sum of edge weights into i (reading Q7) */
    for (int64_t k = 0; k < e; ++k) deg[ei_dst_out[k]] += (double)w_out[k];
    /* 3. w'_k = deg^-1/2[src] * w_k * deg^-1/2[dst] */
    for (int64_t k = 0; k < e; ++k) {
        double ds = deg[ei_src_out[k]], dd = deg[ei_dst_out[k]];
        double is = ds > 0 ? 1.0 / sqrt(ds) : 0.0;
        double id = dd > 0 ? 1.0 / sqrt(dd) : 0.0;
        w_out[k] = (float)(is * (double)w_out[k] * id);
    }
    free(has_loop); free(deg);
    return ORC_OK;
}

int orc_collate(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr,
                const int64_t* local_ei, int64_t* ei, int64_t* batch, int64_t* node_ptr) {
    if (G <= 0 || !num_nodes || !edge_ptr) return ORC_ERR_INVALID; /* empty list */
    if (edge_ptr[0] != 0) return ORC_ERR_INVALID;
    for (int64_t g = 0; g < G; ++g)
        if (num_nodes[g] < 0 || edge_ptr[g + 1] < edge_ptr[g]) return ORC_ERR_INVALID;
    int64_t Etot = edge_ptr[G];
    /* node offsets = exclusive prefix sum of N_g */
    node_ptr[0] = 0;
    for (int64_t g = 0; g < G; ++g) node_ptr[g + 1] = node_ptr[g] + num_nodes[g];
    for (int64_t g = 0; g < G; ++g) {
        for (int64_t k = edge_ptr[g]; k < edge_ptr[g + 1]; ++k) {
            int64_t s = local_ei[k], d = local_ei[Etot + k];
            if (s < 0 || s >= num_nodes[g] || d < 0 || d >= num_nodes[g]) return ORC_ERR_OOB;
            ei[k] = s + node_ptr[g];          /* block-diagonal offset */
            ei[Etot + k] = d + node_ptr[g];
        }
        for (int64_t v = node_ptr[g]; v < node_ptr[g + 1]; ++v) batch[v] = g; /* assignment vector */
    }
    return ORC_OK;
}

int orc_global_pool(const float* x, int64_t N, int64_t F, const int64_t* batch, int64_t G,
                    int reduce, float* out, int64_t* arg) {
    return orc_scatter(x, N, F, F, batch, G, reduce, out, arg, NULL);
}

/* ---- NEXT-1: segment softmax and GAT attention aggregation ---------------- */
/* segment_softmax (the "optimized sparse softmax kernels" of P:239):
 * for every segment i = {k : index[k] == i} and column h, with m = max_k src[k][h],
 *   out[k][h] = exp(src[k][h] - m) / sum_{k' in i} exp(src[k'][h] - m),
 * in double (three plain passes over the edges: max, sum, divide), rounded once. */
int orc_segment_softmax(const float* src, int64_t E, int64_t H, const int64_t* index, int64_t n, float* out) {
    if (E < 0 || H < 0 || n < 0 || (E * H > 0 && (!src || !index || !out))) return ORC_ERR_INVALID;
    if (check_index(index, E, n)) return ORC_ERR_OOB;
    size_t nh = (size_t)(n * H > 0 ? n * H : 1);
    double* m = (double*)malloc(sizeof(double) * nh);
    double* s = (double*)malloc(sizeof(double) * nh);
    if (!m || !s) { free(m); free(s); return ORC_ERR_INVALID; }
    for (size_t t = 0; t < nh; ++t) { m[t] = -INFINITY; s[t] = 0.0; }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) {
            double v = (double)src[k * H + h];
            if (v > m[index[k] * H + h]) m[index[k] * H + h] = v;
        }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) s[index[k] * H + h] += exp((double)src[k * H + h] - m[index[k] * H + h]);
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h)
            out[k * H + h] = (float)(exp((double)src[k * H + h] - m[index[k] * H + h]) / s[index[k] * H + h]);
    free(m);
    free(s);
    return ORC_OK;
}

/* softmax backward (chain rule of the definition above, "differentiable"):
 *   grad_src[k][h] = out[k][h] * (g[k][h] - sum_{k' in seg(k)} out[k'][h] * g[k'][h]).
 * abs (optional, double [E x H]): out[k][h] * (|g[k][h]| + sum |out g|) -- the magnitude of the
 * terms, for the summation tolerance (reading Q11). */
int orc_segment_softmax_backward(const float* out, const float* grad, int64_t E, int64_t H, const int64_t* index,
                                 int64_t n, float* grad_src, double* abs_out) {
    if (E < 0 || H < 0 || n < 0 || (E * H > 0 && (!out || !grad || !index || !grad_src))) return ORC_ERR_INVALID;
    if (check_index(index, E, n)) return ORC_ERR_OOB;
    size_t nh = (size_t)(n * H > 0 ? n * H : 1);
    double* t = (double*)calloc(nh, sizeof(double));
    double* ta = (double*)calloc(nh, sizeof(double));
    if (!t || !ta) { free(t); free(ta); return ORC_ERR_INVALID; }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) {
            t[index[k] * H + h] += (double)out[k * H + h] * (double)grad[k * H + h];
            ta[index[k] * H + h] += fabs((double)out[k * H + h] * (double)grad[k * H + h]);
        }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) {
            double a = (double)out[k * H + h];
            grad_src[k * H + h] = (float)(a * ((double)grad[k * H + h] - t[index[k] * H + h]));
            if (abs_out) abs_out[k * H + h] = a * (fabs((double)grad[k * H + h]) + ta[index[k] * H + h]);
        }
    free(t);
    free(ta);
    return ORC_OK;
}

static double leaky(double v, double slope) { return v > 0.0 ? v : slope * v; }

/* GAT attention coefficients in double: for edge k = (j -> i) and head h,
 *   logit[k][h] = leaky_relu(s_src[j][h] + s_dst[i][h], slope),
 *   alpha[k][h] = softmax of the logits over the segment of target i (as orc_segment_softmax). */
static int gat_alpha(const float* s_src, const float* s_dst, int64_t H, int64_t n_dst, const int64_t* ei, int64_t E,
                     double slope, double* alpha) {
    const int64_t* src = ei;
    const int64_t* dst = ei + E;
    size_t nh = (size_t)(n_dst * H > 0 ? n_dst * H : 1);
    double* m = (double*)malloc(sizeof(double) * nh);
    double* s = (double*)malloc(sizeof(double) * nh);
    if (!m || !s) { free(m); free(s); return ORC_ERR_INVALID; }
    for (size_t t = 0; t < nh; ++t) { m[t] = -INFINITY; s[t] = 0.0; }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) {
            double l = leaky((double)s_src[src[k] * H + h] + (double)s_dst[dst[k] * H + h], slope);
            alpha[k * H + h] = l;
            if (l > m[dst[k] * H + h]) m[dst[k] * H + h] = l;
        }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) {
            alpha[k * H + h] = exp(alpha[k * H + h] - m[dst[k] * H + h]);
            s[dst[k] * H + h] += alpha[k * H + h];
        }
    for (int64_t k = 0; k < E; ++k)
        for (int64_t h = 0; h < H; ++h) alpha[k * H + h] /= s[dst[k] * H + h];
    free(m);
    free(s);
    return ORC_OK;
}

/* GAT aggregation ("output_i = sum alpha z_j (weighted scatter-add)"):
 *   out[i][h*C + c] = sum_{k : dst_k = i} alpha[k][h] * z[src_k][h*C + c]   (double, rounded once)
 * z [n_src x H*C] packed; s_src [n_src x H]; s_dst [n_dst x H]; alpha_out [E x H] (optional,
 * rounded alpha); abs (optional) = sum alpha |z| for the tolerance.  Empty segment -> 0 (Q2). */
int orc_gat(const float* z, int64_t n_src, int64_t H, int64_t C, const float* s_src, const float* s_dst,
            int64_t n_dst, const int64_t* ei, int64_t E, double slope, float* out, float* alpha_out,
            double* abs_out) {
    if (n_src < 0 || H <= 0 || C < 0 || n_dst < 0 || E < 0) return ORC_ERR_INVALID;
    if (E > 0 && (!z || !s_src || !s_dst || !ei)) return ORC_ERR_INVALID;
    if (check_index(ei, E, n_src) || check_index(ei + E, E, n_dst)) return ORC_ERR_OOB;
    const int64_t F = H * C;
    double* alpha = (double*)malloc(sizeof(double) * (size_t)(E * H > 0 ? E * H : 1));
    double* acc = (double*)calloc((size_t)(n_dst * F > 0 ? n_dst * F : 1), sizeof(double));
    if (!alpha || !acc) { free(alpha); free(acc); return ORC_ERR_INVALID; }
    int st = gat_alpha(s_src, s_dst, H, n_dst, ei, E, slope, alpha);
    if (st) { free(alpha); free(acc); return st; }
    if (abs_out)
        for (int64_t t = 0; t < n_dst * F; ++t) abs_out[t] = 0.0;
    for (int64_t k = 0; k < E; ++k) {
        const int64_t j = ei[k], i = ei[E + k];
        for (int64_t h = 0; h < H; ++h)
            for (int64_t c = 0; c < C; ++c) {
                double v = alpha[k * H + h] * (double)z[j * F + h * C + c];
                acc[i * F + h * C + c] += v;
                if (abs_out) abs_out[i * F + h * C + c] += fabs(v);
            }
    }
    for (int64_t t = 0; t < n_dst * F; ++t) out[t] = (float)acc[t];
    if (alpha_out)
        for (int64_t t = 0; t < E * H; ++t) alpha_out[t] = (float)alpha[t];
    free(alpha);
    free(acc);
    return ORC_OK;
}

/* GAT backward (chain rule of orc_gat, double throughout; g = dL/dout [n_dst x H*C]):
 *   grad_z[j][h*C+c]  = sum_{k: src_k = j} alpha[k][h] * g[dst_k][h*C+c]
 *   da[k][h]          = sum_c g[dst_k][h*C+c] * z[src_k][h*C+c]            (per-edge SDDMM)
 *   dl[k][h]          = alpha[k][h] * (da[k][h] - sum_{k' in seg(dst_k)} alpha[k'][h] da[k'][h])
 *   dp[k][h]          = dl[k][h] * (pre > 0 ? 1 : slope),  pre = s_src[j][h] + s_dst[i][h]
 *   grad_s_src[j][h]  = sum_{k: src_k = j} dp[k][h];  grad_s_dst[i][h] = sum_{k: dst_k = i} dp[k][h].
 * abs_* (optional, double): the same sums over the magnitudes of their terms (tolerance). */
int orc_gat_backward(const float* z, int64_t n_src, int64_t H, int64_t C, const float* s_src, const float* s_dst,
                     int64_t n_dst, const int64_t* ei, int64_t E, double slope, const float* g, float* grad_z,
                     float* grad_s_src, float* grad_s_dst, double* abs_z, double* abs_ssrc, double* abs_sdst) {
    if (n_src < 0 || H <= 0 || C < 0 || n_dst < 0 || E < 0) return ORC_ERR_INVALID;
    if (E > 0 && (!z || !s_src || !s_dst || !ei || !g)) return ORC_ERR_INVALID;
    if (check_index(ei, E, n_src) || check_index(ei + E, E, n_dst)) return ORC_ERR_OOB;
    const int64_t F = H * C;
    const size_t eh = (size_t)(E * H > 0 ? E * H : 1), nh = (size_t)(n_dst * H > 0 ? n_dst * H : 1);
    double* alpha = (double*)malloc(sizeof(double) * eh);
    double* da = (double*)malloc(sizeof(double) * eh);
    double* daa = (double*)malloc(sizeof(double) * eh);
    double* t = (double*)calloc(nh, sizeof(double));
    double* ta = (double*)calloc(nh, sizeof(double));
    double* gz = (double*)calloc((size_t)(n_src * F > 0 ? n_src * F : 1), sizeof(double));
    double* gs = (double*)calloc((size_t)(n_src * H > 0 ? n_src * H : 1), sizeof(double));
    double* gd = (double*)calloc(nh, sizeof(double));
    int st = (!alpha || !da || !daa || !t || !ta || !gz || !gs || !gd) ? ORC_ERR_INVALID : ORC_OK;
    if (!st) st = gat_alpha(s_src, s_dst, H, n_dst, ei, E, slope, alpha);
    if (!st) {
        if (abs_z) for (int64_t q = 0; q < n_src * F; ++q) abs_z[q] = 0.0;
        if (abs_ssrc) for (int64_t q = 0; q < n_src * H; ++q) abs_ssrc[q] = 0.0;
        if (abs_sdst) for (int64_t q = 0; q < n_dst * H; ++q) abs_sdst[q] = 0.0;
        for (int64_t k = 0; k < E; ++k) {
            const int64_t j = ei[k], i = ei[E + k];
            for (int64_t h = 0; h < H; ++h) {
                double d = 0.0, dab = 0.0;
                for (int64_t c = 0; c < C; ++c) {
                    const double gv = (double)g[i * F + h * C + c];
                    d += gv * (double)z[j * F + h * C + c];
                    dab += fabs(gv * (double)z[j * F + h * C + c]);
                    gz[j * F + h * C + c] += alpha[k * H + h] * gv;
                    if (abs_z) abs_z[j * F + h * C + c] += alpha[k * H + h] * fabs(gv);
                }
                da[k * H + h] = d;
                daa[k * H + h] = dab;
                t[i * H + h] += alpha[k * H + h] * d;
                ta[i * H + h] += alpha[k * H + h] * dab;
            }
        }
        for (int64_t k = 0; k < E; ++k) {
            const int64_t j = ei[k], i = ei[E + k];
            for (int64_t h = 0; h < H; ++h) {
                const double pre = (double)s_src[j * H + h] + (double)s_dst[i * H + h];
                const double lk = pre > 0.0 ? 1.0 : slope;
                const double dp = alpha[k * H + h] * (da[k * H + h] - t[i * H + h]) * lk;
                const double ab = alpha[k * H + h] * (daa[k * H + h] + ta[i * H + h]) * fabs(lk);
                gs[j * H + h] += dp;
                gd[i * H + h] += dp;
                if (abs_ssrc) abs_ssrc[j * H + h] += ab;
                if (abs_sdst) abs_sdst[i * H + h] += ab;
            }
        }
        if (grad_z) for (int64_t q = 0; q < n_src * F; ++q) grad_z[q] = (float)gz[q];
        if (grad_s_src) for (int64_t q = 0; q < n_src * H; ++q) grad_s_src[q] = (float)gs[q];
        if (grad_s_dst) for (int64_t q = 0; q < n_dst * H; ++q) grad_s_dst[q] = (float)gd[q];
    }
    free(alpha); free(da); free(daa); free(t); free(ta); free(gz); free(gs); free(gd);
    return st;
}

/* ---- NEXT-2: APPNP / SGC K-step propagation ---------------------------------- */
/* APPNP ("Approximate Personalized Propagation of Neural Predictions";
 * S:439-447): z_0 = h; z_{k+1} = (1 - alpha) * S z_k + alpha * h; out = z_K, with
 * (S z)[i] = sum_{k : dst_k = i} w_k z[src_k] (w = 1 when edge_weight is NULL).
 * The state is kept in double through all K steps and rounded once. alpha = 0 is
 * SGC's S^K h. */
int orc_appnp(const float* h, int64_t n, int64_t F, const int64_t* ei, int64_t E, const float* edge_weight,
              int64_t K, double alpha, float* out) {
    if (n < 0 || F < 0 || E < 0 || K < 0 || (n * F > 0 && (!h || !out)) || (E > 0 && !ei)) return ORC_ERR_INVALID;
    if (alpha < 0.0 || alpha > 1.0) return ORC_ERR_INVALID;
    if (check_index(ei, E, n) || check_index(ei + E, E, n)) return ORC_ERR_OOB;
    size_t nf = (size_t)(n * F > 0 ? n * F : 1);
    double* z = (double*)malloc(sizeof(double) * nf);
    double* t = (double*)malloc(sizeof(double) * nf);
    if (!z || !t) { free(z); free(t); return ORC_ERR_INVALID; }
    for (int64_t q = 0; q < n * F; ++q) z[q] = (double)h[q];
    for (int64_t it = 0; it < K; ++it) {
        for (int64_t q = 0; q < n * F; ++q) t[q] = 0.0;
        for (int64_t k = 0; k < E; ++k) {
            const int64_t j = ei[k], i = ei[E + k];
            const double w = edge_weight ? (double)edge_weight[k] : 1.0;
            for (int64_t c = 0; c < F; ++c) t[i * F + c] += w * z[j * F + c];
        }
        for (int64_t q = 0; q < n * F; ++q) z[q] = (1.0 - alpha) * t[q] + alpha * (double)h[q];
    }
    for (int64_t q = 0; q < n * F; ++q) out[q] = (float)z[q];
    free(z);
    free(t);
    return ORC_OK;
}

/* ---- NEXT-2: dense feature transform ------------------------------------------ */
/* Y[m][n] = row_scale[m] * sum_k X[m][k] W[n][k] + bias[n] (the x W of GCN / SGC / APPNP, P:49-54;
 * W in the [out x in] layout), in double, rounded once; abs = sum_k |X[m][k] W[n][k]| * |row_scale|. */
int orc_dense_transform(const float* X, int64_t M, int64_t K, const float* W, int64_t N, const float* bias,
                        const float* row_scale, float* Y, double* abs_out) {
    if (M < 0 || K < 0 || N < 0 || (M * N > 0 && (!X || !W || !Y))) return ORC_ERR_INVALID;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0, ab = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                const double p = (double)X[m * K + k] * (double)W[n * K + k];
                acc += p;
                ab += fabs(p);
            }
            const double rs = row_scale ? (double)row_scale[m] : 1.0;
            acc = acc * rs + (bias ? (double)bias[n] : 0.0);
            Y[m * N + n] = (float)acc;
            if (abs_out) abs_out[m * N + n] = ab * fabs(rs);
        }
    return ORC_OK;
}
