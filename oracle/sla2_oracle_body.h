/*
 * sla2_oracle_body.h -- element-type-generic body of the CPU oracle (TEST INFRASTRUCTURE).
 * Included twice by sla2_oracle.c with T/S/ACC/EXP/LOG/SQRT bound to the float and double
 * instantiations of the reference templates. See sla2_oracle.h for the contract.
 *
 * Every loop below keeps the reference's iteration order and its separate multiply/add
 * roundings (the file is compiled with -ffp-contract=off).
 */

#define FN2(a, b) a##_##b
#define FN1(a, b) FN2(a, b)
#define FN(name) FN1(name, S)

/* matrix.hpp:235-244 colmean: serial sums over rows (ascending), then *= T(1)/rows. */
void FN(sla2o_colmean)(const T* x, size_t rows, size_t cols, T* out) {
    for (size_t j = 0; j < cols; ++j) out[j] = (T)0;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) out[j] += x[i * cols + j];
    const T inv = (T)1 / (T)rows;
    for (size_t j = 0; j < cols; ++j) out[j] *= inv;
}

/* quant.hpp:88-96 smooth_k: K~ = K - colmean(K). */
void FN(sla2o_smooth_k)(const T* k, size_t rows, size_t cols, T* ktilde, T* mean) {
    FN(sla2o_colmean)(k, rows, cols, mean);
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) ktilde[i * cols + j] = k[i * cols + j] - mean[j];
}

/* matrix.hpp:174-195 mean_pool: wide accumulator (double for float, long double for
 * double), rows of a group added in ascending order, then (T)(acc / (ACC)block). */
int FN(sla2o_mean_pool)(const T* x, size_t rows, size_t cols, size_t block, T* out) {
    if (block == 0 || rows % block != 0) return SLA2O_SHAPE;
    return FN(sla2o_mean_pool_ragged)(x, rows, cols, block, out);
}

/* RAGGED EXTENSION (not in the reference, which rejects rows % block != 0 at
 * matrix.hpp:176-179): ceil(rows / block) groups, the last one averaging
 * only its cnt = rows - g * block rows: (T)(acc / (ACC)cnt). Identical to mean_pool when
 * block divides rows (same loop, cnt == block). */
int FN(sla2o_mean_pool_ragged)(const T* x, size_t rows, size_t cols, size_t block, T* out) {
    if (block == 0) return SLA2O_SHAPE;
    const size_t out_rows = (rows + block - 1) / block;
    ACC* acc = (ACC*)malloc(sizeof(ACC) * (cols ? cols : 1));
    for (size_t g = 0; g < out_rows; ++g) {
        const size_t cnt = rows - g * block < block ? rows - g * block : block;
        for (size_t c = 0; c < cols; ++c) acc[c] = (ACC)0;
        for (size_t r = 0; r < cnt; ++r) {
            const T* in = x + (g * block + r) * cols;
            for (size_t c = 0; c < cols; ++c) acc[c] += (ACC)in[c];
        }
        for (size_t c = 0; c < cols; ++c) out[g * cols + c] = (T)(acc[c] / (ACC)cnt);
    }
    free(acc);
    return SLA2O_OK;
}

/* matrix.hpp:101-135 matmul. transpose_b: acc = 0; acc += a[i][k]*b[j][k] (k ascending).
 * Otherwise i-k-j: out[i][j] += a[i][k]*b[k][j] with k ascending per element. */
int FN(sla2o_matmul)(const T* a, size_t ar, size_t ac, const T* b, size_t br, size_t bc,
                     int transpose_b, T* out) {
    const size_t inner = transpose_b ? bc : br;
    const size_t n_out = transpose_b ? br : bc;
    if (ac != inner) return SLA2O_SHAPE;
    if (transpose_b) {
        for (size_t i = 0; i < ar; ++i) {
            const T* arow = a + i * ac;
            for (size_t j = 0; j < n_out; ++j) {
                const T* brow = b + j * bc;
                T acc = (T)0;
                for (size_t k = 0; k < inner; ++k) acc += arow[k] * brow[k];
                out[i * n_out + j] = acc;
            }
        }
    } else {
        for (size_t i = 0; i < ar * n_out; ++i) out[i] = (T)0;
        for (size_t i = 0; i < ar; ++i) {
            const T* arow = a + i * ac;
            T* orow = out + i * n_out;
            for (size_t k = 0; k < inner; ++k) {
                const T aik = arow[k];
                const T* brow = b + k * n_out;
                for (size_t j = 0; j < n_out; ++j) orow[j] += aik * brow[j];
            }
        }
    }
    return SLA2O_OK;
}

/* matrix.hpp:138-155 row_softmax: m = running std::max, o = exp(x - m), serial sum,
 * inv = 1/sum, o *= inv. exp is libm expf/exp (std::exp overloads). */
void FN(sla2o_row_softmax)(const T* s, size_t rows, size_t cols, T* out) {
    for (size_t i = 0; i < rows; ++i) {
        const T* in = s + i * cols;
        T* o = out + i * cols;
        T m = in[0];
        for (size_t j = 1; j < cols; ++j) m = (m < in[j]) ? in[j] : m; /* std::max(m, x) */
        T sum = (T)0;
        for (size_t j = 0; j < cols; ++j) {
            o[j] = EXP(in[j] - m);
            sum += o[j];
        }
        const T inv = (T)1 / sum;
        for (size_t j = 0; j < cols; ++j) o[j] *= inv;
    }
}

/* matrix.hpp:272-277 scale. */
void FN(sla2o_scale)(const T* a, size_t n, T s, T* out) {
    for (size_t i = 0; i < n; ++i) out[i] = a[i] * s;
}

/* router.hpp:87-102 block_scores: softmax((pool(q) proj_q)(pool(k) proj_k)^T * (1/sqrt(d))).
 * RouterParams::validate (router.hpp:27-33) is applied first. */
int FN(sla2o_block_scores)(const T* q, const T* k, size_t n, size_t d, const T* proj_q,
                           const T* proj_k, T tau, size_t bq, size_t bk, T* pc) {
    if (!(tau > (T)0)) return SLA2O_NUMERIC;
    if (bq == 0 || bk == 0 || n % bq || n % bk) return SLA2O_SHAPE;
    return FN(sla2o_block_scores_ragged)(q, k, n, d, proj_q, proj_k, tau, bq, bk, pc);
}

/* RAGGED EXTENSION of block_scores: tm = ceil(n/bq), tn = ceil(n/bk), partial last blocks pooled
 * over their own rows (sla2o_mean_pool_ragged); everything after the pooling unchanged. */
int FN(sla2o_block_scores_ragged)(const T* q, const T* k, size_t n, size_t d, const T* proj_q,
                                  const T* proj_k, T tau, size_t bq, size_t bk, T* pc) {
    if (!(tau > (T)0)) return SLA2O_NUMERIC;
    if (bq == 0 || bk == 0 || n == 0) return SLA2O_SHAPE;
    const size_t tm = (n + bq - 1) / bq, tn = (n + bk - 1) / bk;
    T* qbar = (T*)malloc(sizeof(T) * tm * d);
    T* kbar = (T*)malloc(sizeof(T) * tn * d);
    T* qp = (T*)malloc(sizeof(T) * tm * d);
    T* kp = (T*)malloc(sizeof(T) * tn * d);
    T* sc = (T*)malloc(sizeof(T) * tm * tn);
    FN(sla2o_mean_pool_ragged)(q, n, d, bq, qbar);
    FN(sla2o_mean_pool_ragged)(k, n, d, bk, kbar);
    FN(sla2o_matmul)(qbar, tm, d, proj_q, d, d, 0, qp);
    FN(sla2o_matmul)(kbar, tn, d, proj_k, d, d, 0, kp);
    FN(sla2o_matmul)(qp, tm, d, kp, tn, d, 1, sc);
    FN(sla2o_scale)(sc, tm * tn, (T)1 / SQRT((T)d), sc);
    FN(sla2o_row_softmax)(sc, tm, tn, pc);
    free(qbar); free(kbar); free(qp); free(kp); free(sc);
    return SLA2O_OK;
}

/* router.hpp:106-125 hard_topk: per row, std::stable_sort of column indices by pc
 * descending (equal values keep the lower index first), the first kappa set to 1.
 * Implemented as a stable merge sort with the same strict comparator pc[a] > pc[b]. */
static void FN(oracle_merge_sort_desc)(const T* row, size_t* idx, size_t* tmp, size_t n) {
    for (size_t width = 1; width < n; width *= 2) {
        for (size_t lo = 0; lo < n; lo += 2 * width) {
            size_t mid = lo + width < n ? lo + width : n;
            size_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            size_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                /* take right only if strictly greater: keeps stability */
                if (row[idx[j]] > row[idx[i]]) tmp[o++] = idx[j++];
                else tmp[o++] = idx[i++];
            }
            while (i < mid) tmp[o++] = idx[i++];
            while (j < hi) tmp[o++] = idx[j++];
        }
        memcpy(idx, tmp, sizeof(size_t) * n);
    }
}

int FN(sla2o_hard_topk)(const T* pc, size_t tm, size_t tn, double k_percent, uint8_t* mask,
                        size_t* kappa_out) {
    if (!(k_percent > 0.0 && k_percent <= 100.0)) return SLA2O_SHAPE;
    const size_t kappa = sla2o_topk_budget(k_percent, tn);
    size_t* idx = (size_t*)malloc(sizeof(size_t) * (tn ? tn : 1));
    size_t* tmp = (size_t*)malloc(sizeof(size_t) * (tn ? tn : 1));
    memset(mask, 0, tm * tn);
    for (size_t i = 0; i < tm; ++i) {
        for (size_t j = 0; j < tn; ++j) idx[j] = j;
        FN(oracle_merge_sort_desc)(pc + i * tn, idx, tmp, tn);
        for (size_t r = 0; r < kappa; ++r) mask[i * tn + idx[r]] = 1;
    }
    free(idx); free(tmp);
    if (kappa_out) *kappa_out = kappa;
    return SLA2O_OK;
}

/* quant.hpp:31-50 quantize: absmax = running std::max(|x|); zero block -> scale = T-min;
 * scale = absmax/127; inv = 1/scale; code = clamp(lround((double)(x*inv)), -127, 127). */
int FN(sla2o_quantize)(const T* x, size_t n, int8_t* codes, T* scale) {
    T absmax = (T)0;
    for (size_t i = 0; i < n; ++i) {
        const T a = FABS(x[i]);
        absmax = (absmax < a) ? a : absmax;
    }
    memset(codes, 0, n);
    if (absmax == (T)0) {
        *scale = TMIN;
        return SLA2O_OK;
    }
    *scale = absmax / (T)127;
    const T inv = (T)1 / *scale;
    for (size_t i = 0; i < n; ++i) {
        long r = lround((double)(x[i] * inv));
        if (r < -127) r = -127;
        if (r > 127) r = 127;
        codes[i] = (int8_t)r;
    }
    return SLA2O_OK;
}

/* quant.hpp:62-83 quantized_product: int32 accumulate, out = (T)acc * (sa*sb). */
int FN(sla2o_quantized_product)(const int8_t* a, size_t ar, size_t ac, T sa, const int8_t* b,
                                size_t br, size_t bc, T sb, int transpose_b, T* out) {
    const size_t inner = transpose_b ? bc : br;
    const size_t n_out = transpose_b ? br : bc;
    if (ac != inner) return SLA2O_SHAPE;
    const T s = sa * sb;
    for (size_t i = 0; i < ar; ++i) {
        for (size_t j = 0; j < n_out; ++j) {
            int32_t acc = 0;
            for (size_t k = 0; k < inner; ++k) {
                const int32_t av = a[i * ac + k];
                const int32_t bv = transpose_b ? b[j * bc + k] : b[k * bc + j];
                acc += av * bv;
            }
            out[i * n_out + j] = (T)acc * s;
        }
    }
    return SLA2O_OK;
}

/* attention.hpp:17-22 sigmoid with clamp to [T-min, 1 - eps/2]. */
T FN(sla2o_sigmoid)(T x) {
    T v = (T)1 / ((T)1 + EXP(-x));
    const T lo = TMIN, hi = (T)1 - TEPS / (T)2;
    if (v < lo) v = lo;
    if (hi < v) v = hi;
    return v;
}

/* ---- sla2_forward_blockwise (attention.hpp:423-560), hard BlockMask routing ---- */

typedef struct {
    const T *q, *ktilde, *v, *rho, *q_phi, *h, *z;
    const uint8_t* mask;
    size_t n, d, bq, bk, tm, tn;
    int quant;
    T *out, *o_s, *o_l, *big_l;
} FN(oracle_fwd_ctx);

/* attention.hpp:372-394 block_scores_qk and 396-415 block_product_pv are inlined below. */
static void FN(oracle_fwd_qblock)(const FN(oracle_fwd_ctx) * c, size_t i) {
    const size_t d = c->d, bk = c->bk, tn = c->tn;
    const size_t r0 = i * c->bq;
    /* rows of this query block: bq, or fewer for the ragged tail (n % bq != 0) */
    const size_t bq = c->n - r0 < c->bq ? c->n - r0 : c->bq;
    const T inv_sqrt_d = (T)1 / SQRT((T)d);
    T* m_run = (T*)malloc(sizeof(T) * bq);
    T* l_run = (T*)calloc(bq, sizeof(T));
    T* o_acc = (T*)calloc(bq * d, sizeof(T));
    T* h_i = (T*)calloc(d * d, sizeof(T));
    T* z_i = (T*)calloc(d, sizeof(T));
    T* s = (T*)malloc(sizeof(T) * bq * bk);
    T* p = (T*)malloc(sizeof(T) * bq * bk);
    T* pv = (T*)malloc(sizeof(T) * bq * d);
    int8_t* qa = (int8_t*)malloc(bq * d);
    int8_t* qb = (int8_t*)malloc(bk * d);
    int8_t* qpc = (int8_t*)malloc(bq * bk);
    int8_t* qv = (int8_t*)malloc(bk * d);
    for (size_t r = 0; r < bq; ++r) m_run[r] = -INFINITY;

    for (size_t j = 0; j < tn; ++j) {
        const T w = (T)c->mask[i * tn + j];
        const T cw = (T)(1 - c->mask[i * tn + j]);
        if (cw > (T)0) { /* attention.hpp:495-502 */
            for (size_t f = 0; f < d; ++f) {
                z_i[f] += cw * c->z[j * d + f];
                const T* hsrc = c->h + (j * d + f) * d;
                T* hdst = h_i + f * d;
                for (size_t cc = 0; cc < d; ++cc) hdst[cc] += cw * hsrc[cc];
            }
        }
        if (w <= (T)0) continue;
        /* keys of this block: bk, or fewer for the ragged tail; S is bq x kc, kept packed with
         * row stride kc (the reference's layout when kc == bk) */
        const size_t kc = c->n - j * bk < bk ? c->n - j * bk : bk;
        /* S = Q_i K~_j^T / sqrt(d) (attention.hpp:372-394) */
        if (c->quant) {
            T sa, sb;
            FN(sla2o_quantize)(c->q + r0 * d, bq * d, qa, &sa);
            FN(sla2o_quantize)(c->ktilde + j * bk * d, kc * d, qb, &sb);
            FN(sla2o_quantized_product)(qa, bq, d, sa, qb, kc, d, sb, 1, s);
            FN(sla2o_scale)(s, bq * kc, inv_sqrt_d, s);
        } else {
            for (size_t r = 0; r < bq; ++r) {
                const T* qrow = c->q + (r0 + r) * d;
                for (size_t t = 0; t < kc; ++t) {
                    const T* krow = c->ktilde + (j * bk + t) * d;
                    T acc = (T)0;
                    for (size_t f = 0; f < d; ++f) acc += qrow[f] * krow[f];
                    s[r * kc + t] = acc * inv_sqrt_d;
                }
            }
        }
        /* online softmax (attention.hpp:506-523) */
        for (size_t r = 0; r < bq; ++r) {
            T mx = s[r * kc];
            for (size_t t = 1; t < kc; ++t) mx = (mx < s[r * kc + t]) ? s[r * kc + t] : mx;
            const T m_new = (m_run[r] < mx) ? mx : m_run[r];
            const T rescale = EXP(m_run[r] - m_new);
            T rs = (T)0;
            for (size_t t = 0; t < kc; ++t) {
                p[r * kc + t] = EXP(s[r * kc + t] - m_new);
                rs += p[r * kc + t];
            }
            l_run[r] = rescale * l_run[r] + w * rs;
            T* orow = o_acc + r * d;
            for (size_t cc = 0; cc < d; ++cc) orow[cc] *= rescale;
            m_run[r] = m_new;
        }
        /* PV (attention.hpp:396-415) */
        if (c->quant) {
            T sp, sv;
            FN(sla2o_quantize)(p, bq * kc, qpc, &sp);
            FN(sla2o_quantize)(c->v + j * bk * d, kc * d, qv, &sv);
            FN(sla2o_quantized_product)(qpc, bq, kc, sp, qv, kc, d, sv, 0, pv);
        } else {
            for (size_t r = 0; r < bq * d; ++r) pv[r] = (T)0;
            for (size_t r = 0; r < bq; ++r) {
                T* orow = pv + r * d;
                for (size_t t = 0; t < kc; ++t) {
                    const T prt = p[r * kc + t];
                    const T* vrow = c->v + (j * bk + t) * d;
                    for (size_t cc = 0; cc < d; ++cc) orow[cc] += prt * vrow[cc];
                }
            }
        }
        for (size_t r = 0; r < bq; ++r) {
            T* orow = o_acc + r * d;
            const T* pvrow = pv + r * d;
            for (size_t cc = 0; cc < d; ++cc) orow[cc] += w * pvrow[cc];
        }
    }

    /* epilogue (attention.hpp:532-557) */
    int full_row = 1;
    for (size_t j = 0; j < tn; ++j)
        if (!c->mask[i * tn + j]) { full_row = 0; break; }
    const T a = full_row ? (T)1 : FN(sla2o_sigmoid)(c->rho[i]);
    for (size_t r = 0; r < bq; ++r) {
        const T inv_l = (T)1 / l_run[r];
        const T bigl = m_run[r] + LOG(l_run[r]);
        if (c->big_l) c->big_l[r0 + r] = bigl;
        T* os = c->o_s + (r0 + r) * d;
        const T* oa = o_acc + r * d;
        for (size_t cc = 0; cc < d; ++cc) os[cc] = oa[cc] * inv_l;
        T* ol = c->o_l + (r0 + r) * d;
        if (!full_row) {
            const T* qp = c->q_phi + (r0 + r) * d;
            T denom = (T)0;
            for (size_t f = 0; f < d; ++f) denom += qp[f] * z_i[f];
            for (size_t cc = 0; cc < d; ++cc) {
                T num = (T)0;
                for (size_t f = 0; f < d; ++f) num += qp[f] * h_i[f * d + cc];
                ol[cc] = num / denom;
            }
        }
        T* orow = c->out + (r0 + r) * d;
        for (size_t cc = 0; cc < d; ++cc)
            orow[cc] = full_row ? os[cc] : a * os[cc] + ((T)1 - a) * ol[cc];
    }
    free(m_run); free(l_run); free(o_acc); free(h_i); free(z_i); free(s); free(p); free(pv);
    free(qa); free(qb); free(qpc); free(qv);
}

typedef struct {
    const FN(oracle_fwd_ctx) * ctx;
    size_t begin, end;
} FN(oracle_fwd_job);

static void* FN(oracle_fwd_worker)(void* arg) {
    const FN(oracle_fwd_job)* job = (const FN(oracle_fwd_job)*)arg;
    for (size_t i = job->begin; i < job->end; ++i) FN(oracle_fwd_qblock)(job->ctx, i);
    return NULL;
}

int FN(sla2o_forward_blockwise)(const T* q, const T* k, const T* v, size_t n, size_t d, size_t bq,
                                size_t bk, const uint8_t* mask, const T* rho, int quant,
                                int smooth, T* out, T* o_s, T* o_l, T* big_l) {
    /* validation (attention.hpp:427-447, AttentionInputs::validate 36-43) */
    if (bq == 0 || bk == 0 || n % bq || n % bk) return SLA2O_SHAPE;
    return FN(sla2o_forward_blockwise_ragged)(q, k, v, n, d, bq, bk, mask, rho, quant, smooth, out,
                                              o_s, o_l, big_l);
}

/* RAGGED EXTENSION of sla2_forward_blockwise: tm = ceil(n/bq), tn = ceil(n/bk); the tail query
 * block has n - (tm-1) bq rows, the tail key block n - (tn-1) bk keys (h_j, z_j, S, P and PV over
 * those keys only). Same code path as forward_blockwise, which it equals when the blocks divide n. */
int FN(sla2o_forward_blockwise_ragged)(const T* q, const T* k, const T* v, size_t n, size_t d,
                                       size_t bq, size_t bk, const uint8_t* mask, const T* rho,
                                       int quant, int smooth, T* out, T* o_s, T* o_l, T* big_l) {
    if (bq == 0 || bk == 0 || n == 0) return SLA2O_SHAPE;
    const size_t tm = (n + bq - 1) / bq, tn = (n + bk - 1) / bk;
    for (size_t i = 0; i < tm; ++i) {
        int any = 0;
        for (size_t j = 0; j < tn; ++j) any |= (mask[i * tn + j] != 0);
        if (!any) return SLA2O_SHAPE;
    }
    T* ktilde = (T*)malloc(sizeof(T) * n * d);
    T* mean = (T*)malloc(sizeof(T) * d);
    if (smooth) FN(sla2o_smooth_k)(k, n, d, ktilde, mean);
    else memcpy(ktilde, k, sizeof(T) * n * d);
    T* q_phi = (T*)malloc(sizeof(T) * n * d);
    T* k_phi = (T*)malloc(sizeof(T) * n * d);
    FN(sla2o_row_softmax)(q, n, d, q_phi);
    FN(sla2o_row_softmax)(ktilde, n, d, k_phi);
    /* per-key-block h_j = phi(K~_j)^T V_j, z_j = colsum phi(K~_j) (attention.hpp:459-475) */
    T* h = (T*)calloc(tn * d * d, sizeof(T));
    T* z = (T*)calloc(tn * d, sizeof(T));
    for (size_t j = 0; j < tn; ++j) {
        const size_t kc = n - j * bk < bk ? n - j * bk : bk;
        for (size_t t = 0; t < kc; ++t) {
            const T* kp = k_phi + (j * bk + t) * d;
            const T* vr = v + (j * bk + t) * d;
            for (size_t f = 0; f < d; ++f) {
                z[j * d + f] += kp[f];
                const T kf = kp[f];
                T* hrow = h + (j * d + f) * d;
                for (size_t cc = 0; cc < d; ++cc) hrow[cc] += kf * vr[cc];
            }
        }
    }
    T* os_buf = o_s ? o_s : (T*)malloc(sizeof(T) * n * d);
    T* ol_buf = o_l ? o_l : (T*)malloc(sizeof(T) * n * d);
    memset(os_buf, 0, sizeof(T) * n * d);
    memset(ol_buf, 0, sizeof(T) * n * d);
    FN(oracle_fwd_ctx) ctx = {q, ktilde, v, rho, q_phi, h, z, mask, n, d, bq, bk, tm, tn, quant,
                              out, os_buf, ol_buf, big_l};
    size_t threads = (size_t)oracle_threads();
    if (threads > tm) threads = tm;
    if (threads <= 1) {
        for (size_t i = 0; i < tm; ++i) FN(oracle_fwd_qblock)(&ctx, i);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
        FN(oracle_fwd_job)* jobs = (FN(oracle_fwd_job)*)malloc(sizeof(FN(oracle_fwd_job)) * threads);
        const size_t chunk = (tm + threads - 1) / threads;
        for (size_t t = 0; t < threads; ++t) {
            jobs[t].ctx = &ctx;
            jobs[t].begin = t * chunk < tm ? t * chunk : tm;
            jobs[t].end = (t + 1) * chunk < tm ? (t + 1) * chunk : tm;
            pthread_create(&th[t], NULL, FN(oracle_fwd_worker), &jobs[t]);
        }
        for (size_t t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        free(th); free(jobs);
    }
    if (!o_s) free(os_buf);
    if (!o_l) free(ol_buf);
    free(ktilde); free(mean); free(q_phi); free(k_phi); free(h); free(z);
    return SLA2O_OK;
}

/* ---- sla2_forward_naive (attention.hpp:260-339), hard mask: dense N x N oracle ---- */
int FN(sla2o_forward_naive)(const T* q, const T* k, const T* v, size_t n, size_t d, size_t bq,
                            size_t bk, const uint8_t* mask, const T* rho, int smooth, T* out,
                            T* o_s, T* o_l) {
    if (bq == 0 || bk == 0 || n % bq || n % bk) return SLA2O_SHAPE;
    const size_t tm = n / bq, tn = n / bk;
    for (size_t i = 0; i < tm; ++i) {
        int any = 0;
        for (size_t j = 0; j < tn; ++j) any |= (mask[i * tn + j] != 0);
        if (!any) return SLA2O_SHAPE;
    }
    T* kt = (T*)malloc(sizeof(T) * n * d);
    T* mean = (T*)malloc(sizeof(T) * d);
    if (smooth) FN(sla2o_smooth_k)(k, n, d, kt, mean);
    else memcpy(kt, k, sizeof(T) * n * d);
    T* s = (T*)malloc(sizeof(T) * n * n);
    T* p = (T*)malloc(sizeof(T) * n * n);
    /* attention_scores (attention.hpp:65-68) */
    FN(sla2o_matmul)(q, n, d, kt, n, d, 1, s);
    FN(sla2o_scale)(s, n * n, (T)1 / SQRT((T)d), s);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j)
            if (!mask[(i / bq) * tn + j / bk]) s[i * n + j] -= (T)1e9; /* kMaskNegInf, 155 */
    FN(sla2o_row_softmax)(s, n, n, p);
    T* os = (T*)malloc(sizeof(T) * n * d);
    FN(sla2o_matmul)(p, n, n, v, n, d, 0, os);
    /* linear branch on the complement */
    T* phq = (T*)malloc(sizeof(T) * n * d);
    T* phk = (T*)malloc(sizeof(T) * n * d);
    FN(sla2o_row_softmax)(q, n, d, phq);
    FN(sla2o_row_softmax)(kt, n, d, phk);
    FN(sla2o_matmul)(phq, n, d, phk, n, d, 1, s);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) s[i * n + j] *= (T)(1 - mask[(i / bq) * tn + j / bk]);
    /* normalize_rows_or_zero (attention.hpp:157-170) via rowsum (matrix.hpp:225-233) */
    for (size_t i = 0; i < n; ++i) {
        T sum = (T)0;
        for (size_t j = 0; j < n; ++j) sum += s[i * n + j];
        if (sum != (T)0) {
            const T inv = (T)1 / sum;
            for (size_t j = 0; j < n; ++j) p[i * n + j] = s[i * n + j] * inv;
        } else {
            for (size_t j = 0; j < n; ++j) p[i * n + j] = (T)0;
        }
    }
    T* ol = (T*)malloc(sizeof(T) * n * d);
    FN(sla2o_matmul)(p, n, n, v, n, d, 0, ol);
    for (size_t i = 0; i < n; ++i) {
        const size_t blk = i / bq;
        int full = 1;
        for (size_t j = 0; j < tn; ++j)
            if (!mask[blk * tn + j]) { full = 0; break; }
        const T a = full ? (T)1 : FN(sla2o_sigmoid)(rho[blk]);
        for (size_t cc = 0; cc < d; ++cc)
            out[i * d + cc] = full ? os[i * d + cc] : a * os[i * d + cc] + ((T)1 - a) * ol[i * d + cc];
    }
    if (o_s) memcpy(o_s, os, sizeof(T) * n * d);
    if (o_l) memcpy(o_l, ol, sizeof(T) * n * d);
    free(kt); free(mean); free(s); free(p); free(os); free(phq); free(phk); free(ol);
    return SLA2O_OK;
}

/* attention.hpp:71-75 full_attention = softmax(QK^T/sqrt d) V (the dense baseline). */
int FN(sla2o_full_attention)(const T* q, const T* k, const T* v, size_t n, size_t d, T* out) {
    T* s = (T*)malloc(sizeof(T) * n * n);
    T* p = (T*)malloc(sizeof(T) * n * n);
    FN(sla2o_matmul)(q, n, d, k, n, d, 1, s);
    FN(sla2o_scale)(s, n * n, (T)1 / SQRT((T)d), s);
    FN(sla2o_row_softmax)(s, n, n, p);
    FN(sla2o_matmul)(p, n, n, v, n, d, 0, out);
    free(s); free(p);
    return SLA2O_OK;
}

/* tape.hpp:263-272 Tape::sla2_attention forward composition:
 * smooth_k -> block_scores(q, K~) -> hard_topk -> sla2_forward_blockwise. */
int FN(sla2o_attention)(const T* q, const T* k, const T* v, size_t n, size_t d, size_t bq,
                        size_t bk, const T* proj_q, const T* proj_k, const T* rho,
                        double k_percent, int quant, int smooth, T* out, uint8_t* mask,
                        T* o_s, T* o_l, T* big_l) {
    if (bq == 0 || bk == 0 || n % bq || n % bk) return SLA2O_SHAPE;
    const size_t tm = n / bq, tn = n / bk;
    T* kt = (T*)malloc(sizeof(T) * n * d);
    T* mean = (T*)malloc(sizeof(T) * d);
    if (smooth) FN(sla2o_smooth_k)(k, n, d, kt, mean);
    else memcpy(kt, k, sizeof(T) * n * d);
    T* pc = (T*)malloc(sizeof(T) * tm * tn);
    int rc = FN(sla2o_block_scores)(q, kt, n, d, proj_q, proj_k, (T)0.1, bq, bk, pc);
    if (rc == SLA2O_OK) rc = FN(sla2o_hard_topk)(pc, tm, tn, k_percent, mask, NULL);
    if (rc == SLA2O_OK)
        rc = FN(sla2o_forward_blockwise)(q, k, v, n, d, bq, bk, mask, rho, quant, smooth, out, o_s,
                                         o_l, big_l);
    free(kt); free(mean); free(pc);
    return rc;
}

/* RAGGED EXTENSION of the tape.hpp:263-272 composition for n not divisible by the blocks:
 * smooth_k (colmean over all n rows) -> block_scores_ragged -> hard_topk -> forward_blockwise_ragged. */
int FN(sla2o_attention_ragged)(const T* q, const T* k, const T* v, size_t n, size_t d, size_t bq,
                               size_t bk, const T* proj_q, const T* proj_k, const T* rho,
                               double k_percent, int quant, int smooth, T* out, uint8_t* mask,
                               T* o_s, T* o_l, T* big_l) {
    if (bq == 0 || bk == 0 || n == 0) return SLA2O_SHAPE;
    const size_t tm = (n + bq - 1) / bq, tn = (n + bk - 1) / bk;
    T* kt = (T*)malloc(sizeof(T) * n * d);
    T* mean = (T*)malloc(sizeof(T) * d);
    if (smooth) FN(sla2o_smooth_k)(k, n, d, kt, mean);
    else memcpy(kt, k, sizeof(T) * n * d);
    T* pc = (T*)malloc(sizeof(T) * tm * tn);
    int rc = FN(sla2o_block_scores_ragged)(q, kt, n, d, proj_q, proj_k, (T)0.1, bq, bk, pc);
    if (rc == SLA2O_OK) rc = FN(sla2o_hard_topk)(pc, tm, tn, k_percent, mask, NULL);
    if (rc == SLA2O_OK)
        rc = FN(sla2o_forward_blockwise_ragged)(q, k, v, n, d, bq, bk, mask, rho, quant, smooth, out,
                                                o_s, o_l, big_l);
    free(kt); free(mean); free(pc);
    return rc;
}

/* test_util.hpp:11-28 */
/* The bounds / stddev are T-typed parameters in the reference, widened to double. */
void FN(sla2o_random_matrix)(T* out, size_t n, uint64_t seed, double lo, double hi) {
    sla2o_rng r;
    sla2o_rng_seed(&r, seed);
    const double dlo = (double)(T)lo, dhi = (double)(T)hi;
    for (size_t i = 0; i < n; ++i) out[i] = (T)sla2o_rng_uniform(&r, dlo, dhi);
}
void FN(sla2o_gaussian_matrix)(T* out, size_t n, uint64_t seed, double sd) {
    sla2o_rng r;
    sla2o_rng_seed(&r, seed);
    const double dsd = (double)(T)sd;
    for (size_t i = 0; i < n; ++i) out[i] = (T)sla2o_rng_normal(&r, 0.0, dsd);
}

#undef FN
#undef FN1
#undef FN2
