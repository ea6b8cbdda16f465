// plan.cu -- one-time preprocessing: the stable sort of edges by target (CSR,
// "Compressed Row Storage", row = target; App. A).  The paper
// notes coalescing is "expensive to compute on GPUs and should be hence performed
// as part of the pre-processing" -- the plan is built once per graph, outside the
// timed aggregation, and reused by every forward/backward call.
//
// Steps (all on `stream`, one synchronisation at the end to read back the sizes the
// host needs for launch geometry):
//   1. keys = row_index as int32, vals = 0..E-1 (+ index-range validation);
//   2. LSD radix sort of (key, edge id) pairs over ceil(log2 n_rows) bits (CUB
//      onesweep; LSD radix sort is stable => edges of a row keep ascending ids,
//      which is what the max tie rule needs);
//   3. rowptr from the sorted keys (boundary scatter), col = col_index[perm];
//   4. rows longer than kHeavyThreshold (power-law hubs) are listed, in ascending
//      row order, with the prefix sum of their chunk counts.
#include <algorithm>

#include <cub/cub.cuh>

#include "kernels.cuh"

namespace pyg {

namespace {

int grid_for(int64_t work, int threads = 256) {
    int64_t b = cdiv(work, threads);
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

#define GRID_STRIDE(t, total) \
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (total); t += (int64_t)gridDim.x * blockDim.x)

// key = row, or (source block, row) as block * n_rows + row for source-blocked plans.
// Out-of-range indices raise the flag and are clamped so the build stays in bounds.
__global__ void keys_init(const int64_t* __restrict__ row, const int64_t* __restrict__ col, int64_t E,
                          int64_t n_rows, int64_t n_cols, int64_t col_block, int32_t* keys, int32_t* vals,
                          int* flag) {
    GRID_STRIDE(k, E) {
        int64_t r = row[k];
        if (r < 0 || r >= n_rows) { *flag = 1; r = 0; }
        int64_t key = r;
        if (col) {
            int64_t c = col[k];
            if (c < 0 || c >= n_cols) { *flag = 1; c = 0; }
            if (col_block > 0) key = (c / col_block) * n_rows + r;
        }
        keys[k] = (int32_t)key;
        vals[k] = (int32_t)k;
    }
}

__global__ void rowptr_fill(const int32_t* __restrict__ sk, int64_t E, int64_t n_rows, int64_t* rowptr) {
    // rowptr[r] = first position p with sk[p] >= r
    GRID_STRIDE(p, E + 1) {
        const int64_t prev = p > 0 ? (int64_t)sk[p - 1] : -1;
        const int64_t cur = p < E ? (int64_t)sk[p] : n_rows;
        for (int64_t r = prev + 1; r <= cur; ++r) rowptr[r] = p;
    }
}

__global__ void col_gather(const int64_t* __restrict__ col, const int32_t* __restrict__ perm, int64_t E,
                           int32_t* out, int* not_identity) {
    GRID_STRIDE(p, E) {
        const int32_t k = perm[p];
        if (col) out[p] = (int32_t)col[k];
        if (k != (int32_t)p) *not_identity = 1;
    }
}

__global__ void block_deg_kernel(const int64_t* __restrict__ rowptr, int64_t nb, int64_t n_rows, int32_t* deg) {
    GRID_STRIDE(r, n_rows) {
        int64_t d = 0;
        for (int64_t b = 0; b < nb; ++b) d += rowptr[b * n_rows + r + 1] - rowptr[b * n_rows + r];
        deg[r] = (int32_t)d;
    }
}

__global__ void heavy_flags(const int64_t* __restrict__ rowptr, int64_t n_rows, int thr, int32_t* flag_heavy) {
    GRID_STRIDE(r, n_rows) flag_heavy[r] = (rowptr[r + 1] - rowptr[r]) > thr ? 1 : 0;
}

__global__ void heavy_compact(const int32_t* __restrict__ flag_heavy, const int32_t* __restrict__ pos,
                              int64_t n_rows, int32_t* heavy_rows) {
    GRID_STRIDE(r, n_rows) if (flag_heavy[r]) heavy_rows[pos[r]] = (int32_t)r;
}

// key = 31 - degree bucket (bucket = bit length of the degree): larger rows sort first
// (also counts empty rows into *n_empty: they sort last, the tail the zero-fill kernel visits)
__global__ void order_keys(const int64_t* __restrict__ rowptr, int64_t n_rows, int32_t* keys, int32_t* vals,
                           int* n_empty) {
    GRID_STRIDE(r, n_rows) {
        const int64_t d = rowptr[r + 1] - rowptr[r];
        const int bucket = d > 0 ? 64 - __clzll((unsigned long long)d) : 0;
        keys[r] = 31 - min(bucket, 31);
        vals[r] = (int32_t)r;
        if (d == 0) atomicAdd(n_empty, 1);
    }
}

// pos_row[p] = row owning sorted position p (one thread per row, writes its positions)
__global__ void pos_row_fill(const int64_t* __restrict__ rowptr, int64_t n_rows, int32_t* pos_row) {
    GRID_STRIDE(r, n_rows) {
        for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) pos_row[p] = (int32_t)r;
    }
}

__global__ void heavy_counts(const int32_t* __restrict__ heavy_rows, int64_t n_heavy,
                             const int64_t* __restrict__ rowptr, int chunk, int64_t* cnt) {
    GRID_STRIDE(h, n_heavy) {
        const int64_t r = heavy_rows[h];
        cnt[h] = cdiv(rowptr[r + 1] - rowptr[r], chunk);
    }
}

}  // namespace

// Split parameters of a plan: rows longer than `thr` positions are cut into `chunk`-position pieces
// (separate work items, fp32 partials combined in fp64): 2048 / 512 (reading Q12).  (Splitting the
// rows of few-row, high-degree graphs above 32 positions was measured: Fig. 3's 10,000-node ER graph
// at degree 128 went from 35 to 53 ms per 1000 runs -- the extra launches and the combine cost more
// than the parallelism gained -- so the thresholds are fixed.)
static void split_params(int64_t E, int64_t V, int64_t n_blocks, int64_t* thr, int64_t* chunk) {
    (void)E;
    (void)V;
    (void)n_blocks;
    *thr = kHeavyThreshold;
    *chunk = kChunk;
}

struct PlanLayout {
    int32_t *keys, *vals, *skeys, *perm, *col, *flag_heavy, *pos, *heavy_rows, *deg;
    int32_t *order, *okeys, *okeys_out, *ovals, *pos_row, *task_item;
    int64_t *rowptr, *cnt, *item_ptr, *ldeg, *task_pos;
    size_t task_cap;
    int* flags2;
    void* cub_tmp;
    size_t cub_bytes;
};

// V = n_blocks * n_rows virtual rows (n_blocks = 1 unless source-blocked)
static size_t plan_layout(void* ws, size_t bytes, int64_t E, int64_t n_rows, int64_t n_blocks, bool has_col,
                          PlanLayout& L) {
    Carver cv(ws, bytes);
    const size_t e = (size_t)std::max<int64_t>(E, 1);
    const size_t v = (size_t)std::max<int64_t>(n_rows * n_blocks, 1);
    // kept arrays first
    L.rowptr = cv.take<int64_t>(v + 1);
    L.perm = cv.take<int32_t>(e);
    L.col = has_col ? cv.take<int32_t>(e) : nullptr;
    L.heavy_rows = cv.take<int32_t>(v);
    L.item_ptr = cv.take<int64_t>(v + 1);
    L.deg = n_blocks > 1 ? cv.take<int32_t>((size_t)std::max<int64_t>(n_rows, 1)) : nullptr;
    L.flags2 = cv.take<int>(3);  // [0] perm not identity, [1] empty rows, [2] index out of range
    // scratch
    L.keys = cv.take<int32_t>(e);
    L.vals = cv.take<int32_t>(e);
    L.skeys = cv.take<int32_t>(e);
    L.flag_heavy = cv.take<int32_t>(v);
    L.pos = cv.take<int32_t>(v);
    L.cnt = cv.take<int64_t>(v + 1);
    // light-row order (unblocked plans only)
    const size_t vo = n_blocks == 1 ? v : 1;
    L.order = cv.take<int32_t>(vo);
    L.okeys = cv.take<int32_t>(vo);
    L.okeys_out = cv.take<int32_t>(vo);
    L.ovals = cv.take<int32_t>(vo);
    L.ldeg = cv.take<int64_t>(1);
    L.pos_row = n_blocks == 1 ? cv.take<int32_t>(e) : nullptr;
    // closed tasks hold > kTaskPositions - thr positions; hub rows add one cut each
    int64_t thr = 0, chk = 0;
    split_params(E, n_rows * n_blocks, n_blocks, &thr, &chk);
    L.task_cap = n_blocks == 1 ? (e / (kTaskPositions - thr) + 2 * (e / thr) + e / chk + 4) : 1;
    L.task_pos = cv.take<int64_t>(2 * L.task_cap);
    L.task_item = cv.take<int32_t>(L.task_cap);
    size_t b1 = 0, b2 = 0, b3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)e, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, b2, (int32_t*)nullptr, (int32_t*)nullptr, (int)v);
    cub::DeviceScan::ExclusiveSum(nullptr, b3, (int64_t*)nullptr, (int64_t*)nullptr, (int)v + 1);
    size_t b5 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b5, (int64_t*)nullptr, (int64_t*)nullptr, (int)vo + 1);
    b3 = std::max(b3, b5);
    size_t b4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b4, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)vo, 0, 5);
    L.cub_bytes = std::max(std::max(b1, b4), std::max(b2, b3));
    L.cub_tmp = cv.take<char>(L.cub_bytes);
    return cv.off;
}

#define LAUNCH_CHECK()                  \
    do {                                \
        PYG_LAUNCHED();                 \
        PYG_CUDA(cudaGetLastError());   \
    } while (0)

static int64_t n_blocks_for(int64_t n_cols, int64_t col_block) {
    return col_block > 0 ? std::max<int64_t>(1, cdiv(n_cols, col_block)) : 1;
}

pyg_status_t plan_workspace(int64_t E, int64_t n_rows, int64_t n_cols, int64_t col_block, size_t* bytes) {
    PlanLayout L;
    const int64_t nb = n_blocks_for(n_cols, col_block);
    if (nb * n_rows > 0x7ffffffeLL) return fail(PYG_ERR_UNSUPPORTED, "plan: n_blocks * n_rows must be < 2^31");
    *bytes = plan_layout(nullptr, 0, E, n_rows, nb, true, L) + 1024;
    return PYG_OK;
}

pyg_status_t plan_slice_impl(const pyg_plan* p, int64_t lo, int64_t hi, pyg_plan** out);

pyg_status_t plan_build_impl(const int64_t* row, const int64_t* col, int64_t E, int64_t n_rows, int64_t n_cols,
                             int64_t col_block, void* ws, size_t bytes, pyg_plan** out, cudaStream_t s) {
    PlanLayout L;
    if (!col) col_block = 0;
    const int64_t nb = n_blocks_for(n_cols, col_block);
    if (nb * n_rows > 0x7ffffffeLL) return fail(PYG_ERR_UNSUPPORTED, "plan: n_blocks * n_rows must be < 2^31");
    const int64_t V = nb * n_rows;  // virtual rows
    const size_t need = plan_layout(ws, bytes, E, n_rows, nb, col != nullptr, L);
    int64_t thr = 0, chunk = 0;
    split_params(E, V, nb, &thr, &chunk);
    if (!ws || need > bytes) return fail(PYG_ERR_NO_MEMORY, "plan workspace too small (%zu < %zu)", bytes, need);
    // the out-of-range flag lives in the plan's own workspace (no process-wide state)
    int* flag = L.flags2 + 2;
    PYG_CUDA(cudaMemsetAsync(L.flags2, 0, 3 * sizeof(int), s));
    if (E > 0) {
        keys_init<<<grid_for(E), 256, 0, s>>>(row, col, E, n_rows, n_cols, nb > 1 ? col_block : 0, L.keys, L.vals,
                                              flag);
        LAUNCH_CHECK();
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) < V) ++bits;
        size_t cb = L.cub_bytes;
        PYG_CUDA(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cb, L.keys, L.skeys, L.vals, L.perm, (int)E, 0, bits, s));
        PYG_LAUNCHED();
    }
    rowptr_fill<<<grid_for(E + 1), 256, 0, s>>>(L.skeys, E, V, L.rowptr);
    LAUNCH_CHECK();
    if (E > 0) {
        col_gather<<<grid_for(E), 256, 0, s>>>(col, L.perm, E, L.col, L.flags2);
        LAUNCH_CHECK();
    }
    if (nb > 1) {  // total in-degree = sum of the row's lengths over the blocks (clamped keys: in bounds)
        block_deg_kernel<<<grid_for(n_rows), 256, 0, s>>>(L.rowptr, nb, n_rows, L.deg);
        LAUNCH_CHECK();
    }
    std::vector<int64_t> h_rowptr;
    if (nb == 1 && V > 0) {
        order_keys<<<grid_for(V), 256, 0, s>>>(L.rowptr, V, L.okeys, L.ovals, L.flags2 + 1);
        LAUNCH_CHECK();
        size_t cb = L.cub_bytes;
        PYG_CUDA(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cb, L.okeys, L.okeys_out, L.ovals, L.order, (int)V, 0, 5,
                                                 s));
        PYG_LAUNCHED();
        if (E > 0) {
            pos_row_fill<<<grid_for(V), 256, 0, s>>>(L.rowptr, V, L.pos_row);
            LAUNCH_CHECK();
        }
        h_rowptr.resize((size_t)V + 1);
        PYG_CUDA(cudaMemcpyAsync(h_rowptr.data(), L.rowptr, 8 * ((size_t)V + 1), cudaMemcpyDeviceToHost, s));
    }
    int64_t n_heavy = 0;
    if (V > 0) {
        heavy_flags<<<grid_for(V), 256, 0, s>>>(L.rowptr, V, (int)thr, L.flag_heavy);
        LAUNCH_CHECK();
        size_t cb = L.cub_bytes;
        PYG_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.flag_heavy, L.pos, (int)V, s));
        PYG_LAUNCHED();
        heavy_compact<<<grid_for(V), 256, 0, s>>>(L.flag_heavy, L.pos, V, L.heavy_rows);
        LAUNCH_CHECK();
        int32_t last_pos = 0, last_flag = 0;
        PYG_CUDA(cudaMemcpyAsync(&last_pos, L.pos + V - 1, 4, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaMemcpyAsync(&last_flag, L.flag_heavy + V - 1, 4, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        n_heavy = (int64_t)last_pos + last_flag;
    }
    std::vector<int32_t> h_rows((size_t)n_heavy);
    std::vector<int64_t> h_ptr((size_t)n_heavy + 1, 0);
    if (n_heavy > 0) {
        heavy_counts<<<grid_for(n_heavy), 256, 0, s>>>(L.heavy_rows, n_heavy, L.rowptr, (int)chunk, L.cnt);
        LAUNCH_CHECK();
        PYG_CUDA(cudaMemsetAsync(L.cnt + n_heavy, 0, sizeof(int64_t), s));
        size_t cb = L.cub_bytes;
        PYG_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.cnt, L.item_ptr, (int)n_heavy + 1, s));
        PYG_LAUNCHED();
        PYG_CUDA(cudaMemcpyAsync(h_rows.data(), L.heavy_rows, 4 * (size_t)n_heavy, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaMemcpyAsync(h_ptr.data(), L.item_ptr, 8 * ((size_t)n_heavy + 1), cudaMemcpyDeviceToHost, s));
    } else {
        PYG_CUDA(cudaMemsetAsync(L.item_ptr, 0, sizeof(int64_t), s));
    }
    // task partition of the light positions (host greedy over the row pointers; preprocessing):
    // a task is a run of consecutive light rows with <= kTaskPositions positions, cut before a row
    // that would overflow it and at every split hub row, so its positions are contiguous.
    // Hub rows contribute one task per kChunk-position chunk, tagged with its split-row item id
    // (items are numbered in row order exactly like heavy_item_ptr) so the TMA kernel can write
    // the chunk's partial for the fp64 combine.
    int64_t n_tasks = 0, n_light_tasks = 0;
    if (nb == 1 && V > 0 && E > 0) {
        std::vector<int64_t> tp, hp;  // light tasks first, then the hub chunk tasks
        std::vector<int32_t> ti, hi;
        tp.reserve(2 * (L.task_cap));
        ti.reserve(L.task_cap);
        int64_t t0 = -1, t1 = -1, item = 0;
        auto close = [&]() {
            if (t0 >= 0) { tp.push_back(t0); tp.push_back(t1); ti.push_back(-1); t0 = -1; }
        };
        for (int64_t r = 0; r < V; ++r) {
            const int64_t b = h_rowptr[(size_t)r], e = h_rowptr[(size_t)r + 1], d = e - b;
            if (d > thr) {
                close();
                for (int64_t c = b; c < e; c += chunk) {
                    hp.push_back(c);
                    hp.push_back(std::min<int64_t>(c + chunk, e));
                    hi.push_back((int32_t)item++);
                }
                continue;
            }
            if (d == 0) continue;
            if (t0 >= 0 && (e - t0) > kTaskPositions) close();
            if (t0 < 0) t0 = b;
            t1 = e;
        }
        close();
        n_light_tasks = (int64_t)ti.size();
        tp.insert(tp.end(), hp.begin(), hp.end());
        ti.insert(ti.end(), hi.begin(), hi.end());
        n_tasks = (int64_t)ti.size();
        if ((size_t)n_tasks > L.task_cap) return fail(PYG_ERR_INVALID_ARGUMENT, "internal: task capacity");
        if (n_tasks > 0) {
            PYG_CUDA(cudaMemcpyAsync(L.task_pos, tp.data(), tp.size() * 8, cudaMemcpyHostToDevice, s));
            PYG_CUDA(cudaMemcpyAsync(L.task_item, ti.data(), ti.size() * 4, cudaMemcpyHostToDevice, s));
        }
        PYG_CUDA(cudaStreamSynchronize(s));  // tp / ti are locals
    }
    int flags2[3] = {0, 0, 0};
    PYG_CUDA(cudaMemcpyAsync(flags2, L.flags2, sizeof(flags2), cudaMemcpyDeviceToHost, s));
    PYG_CUDA(cudaStreamSynchronize(s));
    if (flags2[2]) return fail(PYG_ERR_INDEX_OUT_OF_BOUNDS, "plan_build: index out of range");

    pyg_plan root;
    root.n_rows = V;
    root.n_cols = n_cols;
    root.E = E;
    root.row_offset = 0;
    root.rowptr = L.rowptr;
    root.col = col ? L.col : nullptr;
    root.perm = L.perm;
    root.perm_identity = flags2[0] == 0;
    root.heavy_rows = L.heavy_rows;
    root.heavy_item_ptr = L.item_ptr;
    root.h_heavy_rows = std::move(h_rows);
    root.h_heavy_item_ptr = std::move(h_ptr);
    root.h_lo = 0;
    root.h_hi = n_heavy;
    root.item_lo = 0;
    root.item_hi = root.h_heavy_item_ptr[(size_t)n_heavy];
    root.heavy_threshold = (int32_t)thr;
    root.chunk = (int32_t)chunk;
    if (nb == 1) {
        root.row_order = L.order;
        root.order_len = V;
        root.task_pos = n_tasks > 0 ? L.task_pos : nullptr;
        root.task_item = n_tasks > 0 ? L.task_item : nullptr;
        root.n_light_tasks = n_light_tasks;
        root.pos_row = L.pos_row;
        root.n_tasks = n_tasks;
        root.n_empty = flags2[1];
        root.empty_begin = V - flags2[1];
    }
    if (nb == 1) {
        *out = new pyg_plan(std::move(root));
        return PYG_OK;
    }
    // source-blocked: the user-facing plan has n_rows real rows and one part per block
    pyg_plan* p = new pyg_plan();
    p->n_rows = n_rows;
    p->n_cols = n_cols;
    p->E = E;
    p->col = root.col;
    p->perm = root.perm;
    p->perm_identity = 0;
    p->heavy_threshold = (int32_t)thr;
    p->chunk = (int32_t)chunk;
    p->col_block = col_block;
    p->deg = L.deg;
    for (int64_t b = 0; b < nb; ++b) {
        pyg_plan* part = nullptr;
        PYG_TRY(plan_slice_impl(&root, b * n_rows, (b + 1) * n_rows, &part));
        p->parts.push_back(std::move(*part));
        delete part;
    }
    p->rowptr = p->parts[0].rowptr;
    for (const auto& q : p->parts) {
        p->item_hi += q.item_hi - q.item_lo;
        p->h_hi += q.h_hi - q.h_lo;
    }
    *out = p;
    return PYG_OK;
}

namespace {
__global__ void export_kernel(const int64_t* __restrict__ rp, int64_t n_rows, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ perm, int64_t* rowptr, int64_t* col_out, int64_t* perm_out) {
    const int64_t b = rp[0], e = rp[n_rows];
    GRID_STRIDE(t, n_rows + 1) if (rowptr) rowptr[t] = rp[t] - b;
    GRID_STRIDE(p, e - b) {
        if (col_out) col_out[p] = col[b + p];
        if (perm_out) perm_out[p] = perm[b + p];
    }
}
}  // namespace

pyg_status_t plan_export_impl(const pyg_plan* p, int64_t* rowptr, int64_t* col, int64_t* perm, cudaStream_t s) {
    export_kernel<<<grid_for(std::max<int64_t>(p->n_rows + 1, p->E)), 256, 0, s>>>(p->rowptr, p->n_rows, p->col,
                                                                                  p->perm, rowptr, col, perm);
    LAUNCH_CHECK();
    return PYG_OK;
}

pyg_status_t plan_slice_impl(const pyg_plan* p, int64_t lo, int64_t hi, pyg_plan** out) {
    if (!p->parts.empty()) {
        pyg_plan* q = new pyg_plan();
        q->n_rows = hi - lo;
        q->n_cols = p->n_cols;
        q->E = p->E;
        q->row_offset = p->row_offset + lo;
        q->col = p->col;
        q->perm = p->perm;
        q->heavy_threshold = p->heavy_threshold;
        q->chunk = p->chunk;
        q->col_block = p->col_block;
        q->pass_base = p->pass_base;
        q->n_passes = p->n_passes;
        q->deg = p->deg + lo;
        for (const auto& part : p->parts) {
            pyg_plan* sub = nullptr;
            PYG_TRY(plan_slice_impl(&part, lo, hi, &sub));
            q->parts.push_back(std::move(*sub));
            delete sub;
        }
        q->rowptr = q->parts[0].rowptr;
        for (const auto& r : q->parts) {
            q->item_hi += r.item_hi - r.item_lo;
            q->h_hi += r.h_hi - r.h_lo;
        }
        *out = q;
        return PYG_OK;
    }
    pyg_plan* q = new pyg_plan(*p);
    q->row_offset = p->row_offset + lo;
    q->rowptr = p->rowptr + lo;
    q->n_rows = hi - lo;
    const auto& hr = p->h_heavy_rows;
    const int64_t glo = q->row_offset, ghi = q->row_offset + (hi - lo);
    const auto first = hr.begin() + p->h_lo, last = hr.begin() + p->h_hi;
    const int64_t a = std::lower_bound(first, last, (int32_t)glo) - hr.begin();
    const int64_t b = std::lower_bound(first, last, (int32_t)std::min<int64_t>(ghi, INT32_MAX)) - hr.begin();
    q->h_lo = a;
    q->h_hi = std::max(a, b);
    q->item_lo = p->h_heavy_item_ptr[(size_t)q->h_lo];
    q->item_hi = p->h_heavy_item_ptr[(size_t)q->h_hi];
    *out = q;
    return PYG_OK;
}

// Pass view: the source blocks [lo, hi) of a source-blocked plan (or of a slice of one); calls made
// with the views of consecutive ranges, in order, equal one call with the whole plan.
pyg_status_t plan_passes_impl(const pyg_plan* p, int64_t lo, int64_t hi, pyg_plan** out) {
    pyg_plan* q = new pyg_plan(*p);
    q->parts.assign(p->parts.begin() + lo, p->parts.begin() + hi);
    q->n_passes = p->n_passes > 0 ? p->n_passes : (int64_t)p->parts.size();
    q->pass_base = p->pass_base + lo;
    q->rowptr = q->parts.empty() ? p->rowptr : q->parts[0].rowptr;
    q->item_lo = q->item_hi = q->h_lo = q->h_hi = 0;
    for (const auto& r : q->parts) {
        q->item_hi += r.item_hi - r.item_lo;
        q->h_hi += r.h_hi - r.h_lo;
    }
    *out = q;
    return PYG_OK;
}

}  // namespace pyg
