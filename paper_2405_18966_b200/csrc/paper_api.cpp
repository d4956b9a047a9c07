// paper_api.cpp -- the paper's C interface (include/svdsc_paper.h)
// and Matrix Market I/O, host-side C++ over the libsvdsc
// C ABI: layout conversion (1-based four-array CSR -> 0-based row_ptr CSR),
// output allocation, and the host-buffer solve entry points.  No compute here.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "../../include/svdsc_paper.h"

namespace {

thread_local std::string g_err;

svdsc_status fail(svdsc_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

template <typename T>
T *xmalloc(size_t n) {
    return static_cast<T *>(std::malloc(std::max<size_t>(n, 1) * sizeof(T)));
}

bool alloc_mat(svdsc_mat *M, int64_t r, int64_t c) {
    M->nrows = r;
    M->ncols = c;
    M->d = xmalloc<double>((size_t)r * (size_t)c);
    return M->d != nullptr;
}

// one handle per call on the current device, default stream
struct Handle {
    svdsc_handle *h = nullptr;
    svdsc_status st = SVDSC_OK;
    Handle() { st = svdsc_create(&h, nullptr); }
    ~Handle() {
        if (h) svdsc_destroy(h);
    }
};

svdsc_opts make_opts(int k, double tol, int t, int r) {
    svdsc_opts o;
    std::memset(&o, 0, sizeof(o));
    o.k = k;
    o.tol = tol;
    o.t = t;
    o.maxit = r;
    o.seed = 0;
    o.v0 = nullptr;  // library start vector (reading Q8)
    o.fixed_passes = 0;
    o.reorth = 2;
    return o;
}

// the solve shared by the sparse and dense paper entry points: outputs are
// allocated here and filled by the host-buffer C-ABI solve
template <typename Solve>
svdsc_status paper_solve(int64_t m, int64_t n, int k, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, Solve &&solve) {
    if (!U || !S || !V) return fail(SVDSC_EINVAL, "U, S and V must be non-NULL");
    if (k < 1) return fail(SVDSC_EINVAL, "k must be >= 1");
    U->d = S->d = V->d = nullptr;
    if (!alloc_mat(U, m, k) || !alloc_mat(S, k, 1) || !alloc_mat(V, n, k)) {
        svdsc_mat_free(U);
        svdsc_mat_free(S);
        svdsc_mat_free(V);
        return fail(SVDSC_ENOMEM, "host allocation of the outputs failed");
    }
    Handle H;
    if (H.st != SVDSC_OK) {
        svdsc_mat_free(U);
        svdsc_mat_free(S);
        svdsc_mat_free(V);
        return fail(H.st, "svdsc_create failed (no CUDA device?)");
    }
    std::vector<double> resid(k);
    svdsc_info info;
    const svdsc_status st = solve(H.h, S->d, U->d, V->d, resid.data(), &info);
    if (st < 0) {
        g_err = svdsc_last_error(H.h);
        svdsc_mat_free(U);
        svdsc_mat_free(S);
        svdsc_mat_free(V);
    }
    return st;
}

}  // namespace

extern "C" {

const char *svdsc_paper_last_error(void) { return g_err.c_str(); }

void svdsc_mat_free(svdsc_mat *M) {
    if (!M) return;
    std::free(M->d);
    M->d = nullptr;
}

void svdsc_mat_csr_free(svdsc_mat_csr *A) {
    if (!A) return;
    std::free(A->values);
    std::free(A->cols);
    std::free(A->pointerB);
    std::free(A->pointerE);
    A->values = nullptr;
    A->cols = A->pointerB = A->pointerE = nullptr;
}

svdsc_status svdsc_paper_csr_to_csr(const svdsc_mat_csr *A, int64_t **row_ptr, int32_t **col_idx, double **values,
                                    int64_t *nnz_kept) {
    if (!A || !row_ptr || !col_idx || !values || !nnz_kept) return fail(SVDSC_EINVAL, "NULL argument");
    if (A->nrows < 0 || A->ncols < 0 || A->nnz < 0) return fail(SVDSC_EINVAL, "negative dimension");
    if (A->nrows > 0 && (!A->pointerB || !A->pointerE)) return fail(SVDSC_EINVAL, "pointerB/pointerE are NULL");
    if (A->nnz > 0 && (!A->cols || !A->values)) return fail(SVDSC_EINVAL, "cols/values are NULL");
    int64_t kept = 0;
    for (int64_t i = 0; i < A->nrows; i++) {
        const int64_t b = A->pointerB[i], e = A->pointerE[i];
        if (e < b || b < 1 || e > A->nnz + 1)
            return fail(SVDSC_EINVAL, "row " + std::to_string(i) + ": pointerB/pointerE inconsistent (" +
                                          std::to_string(b) + ", " + std::to_string(e) + ")");
        kept += e - b;
    }
    int64_t *rp = xmalloc<int64_t>(A->nrows + 1);
    int32_t *ci = xmalloc<int32_t>(kept);
    double *va = xmalloc<double>(kept);
    if (!rp || !ci || !va) {
        std::free(rp);
        std::free(ci);
        std::free(va);
        return fail(SVDSC_ENOMEM, "host allocation failed");
    }
    int64_t p = 0;
    rp[0] = 0;
    for (int64_t i = 0; i < A->nrows; i++) {
        for (int64_t q = A->pointerB[i] - 1; q < A->pointerE[i] - 1; q++) {
            const int c = A->cols[q];
            if (c < 1 || c > A->ncols) {
                std::free(rp);
                std::free(ci);
                std::free(va);
                return fail(SVDSC_EINVAL, "row " + std::to_string(i) + ": column index " + std::to_string(c) +
                                              " outside 1.." + std::to_string(A->ncols));
            }
            ci[p] = c - 1;
            va[p] = A->values[q];
            p++;
        }
        rp[i + 1] = p;
    }
    *row_ptr = rp;
    *col_idx = ci;
    *values = va;
    *nnz_kept = kept;
    return SVDSC_OK;
}

svdsc_status svds_C_opt(const svdsc_mat_csr *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k, double tol, int t,
                        int r) {
    if (!A) return fail(SVDSC_EINVAL, "A is NULL");
    int64_t *rp = nullptr;
    int32_t *ci = nullptr;
    double *va = nullptr;
    int64_t nnz = 0;
    svdsc_status st = svdsc_paper_csr_to_csr(A, &rp, &ci, &va, &nnz);
    if (st != SVDSC_OK) return st;
    const svdsc_opts o = make_opts(k, tol, t, r);
    st = paper_solve(A->nrows, A->ncols, k, U, S, V,
                     [&](svdsc_handle *h, double *Sd, double *Ud, double *Vd, double *res, svdsc_info *info) {
                         return svdsc_solve_host_csr(h, A->nrows, A->ncols, nnz, rp, ci, va, &o, Sd, Ud, Vd, res,
                                                     info);
                     });
    std::free(rp);
    std::free(ci);
    std::free(va);
    return st;
}

svdsc_status svds_C(const svdsc_mat_csr *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k) {
    return svds_C_opt(A, U, S, V, k, 1e-10, 0, 10);
}

svdsc_status svds_C_dense_opt(const svdsc_mat *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k, double tol, int t,
                              int r) {
    if (!A || !A->d) return fail(SVDSC_EINVAL, "A is NULL");
    const svdsc_opts o = make_opts(k, tol, t, r);
    return paper_solve(A->nrows, A->ncols, k, U, S, V,
                       [&](svdsc_handle *h, double *Sd, double *Ud, double *Vd, double *res, svdsc_info *info) {
                           return svdsc_solve_host_dense(h, A->nrows, A->ncols, A->d, &o, Sd, Ud, Vd, res, info);
                       });
}

svdsc_status svds_C_dense(const svdsc_mat *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k) {
    return svds_C_dense_opt(A, U, S, V, k, 1e-10, 0, 10);
}

// ---------------------------------------------------------------------------
// Matrix Market
svdsc_status svdsc_read_mm(const char *path, svdsc_mat_csr *A, svdsc_mat *D, int *is_dense) {
    if (!path || !A || !D || !is_dense) return fail(SVDSC_EINVAL, "NULL argument");
    std::memset(A, 0, sizeof(*A));
    std::memset(D, 0, sizeof(*D));
    std::ifstream in(path);
    if (!in) return fail(SVDSC_EINVAL, std::string("cannot open ") + path);
    std::string line;
    int64_t lineno = 0;
    auto err = [&](const std::string &m) { return fail(SVDSC_EINVAL, std::string(path) + ":" + std::to_string(lineno) + ": " + m); };
    if (!std::getline(in, line)) return err("empty file");
    lineno++;
    std::string lower = line;
    std::transform(lower.begin(), lower.end(), lower.begin(), [](unsigned char c) { return (char)std::tolower(c); });
    std::istringstream bh(lower);
    std::string banner, object, format, field, symmetry;
    bh >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%matrixmarket" || object != "matrix") return err("not a MatrixMarket matrix banner");
    if (format != "coordinate" && format != "array") return err("format must be coordinate or array");
    if (field != "real" && field != "integer" && field != "double") return err("field must be real (or integer)");
    if (symmetry != "general" && symmetry != "symmetric") return err("symmetry must be general or symmetric");
    const bool sym = symmetry == "symmetric";
    // size line (after comments)
    int64_t m = -1, n = -1, nz = -1;
    while (std::getline(in, line)) {
        lineno++;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream s(line);
        if (format == "coordinate") {
            if (!(s >> m >> n >> nz)) return err("bad size line");
        } else {
            if (!(s >> m >> n)) return err("bad size line");
        }
        break;
    }
    if (m < 0 || n < 0) return err("missing size line");
    if (format == "array") {
        if (sym && m != n) return err("symmetric array must be square");
        if (!alloc_mat(D, m, n)) return fail(SVDSC_ENOMEM, "allocation failed");
        int64_t i = 0, j = 0, cnt = 0;
        const int64_t want = sym ? n * (n + 1) / 2 : m * n;
        while (cnt < want && std::getline(in, line)) {
            lineno++;
            if (line.empty() || line[0] == '%') continue;
            char *end = nullptr;
            errno = 0;
            const double v = std::strtod(line.c_str(), &end);
            if (end == line.c_str() || errno == ERANGE) {
                svdsc_mat_free(D);
                return err("bad value");
            }
            D->d[i + j * m] = v;
            if (sym) D->d[j + i * m] = v;
            cnt++;
            if (++i == m) {  // column-major; symmetric: lower triangle i >= j
                j++;
                i = sym ? j : 0;
            }
        }
        if (cnt != want) {
            svdsc_mat_free(D);
            return err("too few values");
        }
        *is_dense = 1;
        return SVDSC_OK;
    }
    std::vector<std::pair<int64_t, std::pair<int32_t, double>>> e;  // (row, (col, val)), 0-based
    e.reserve((size_t)(sym ? 2 * nz : nz));
    int64_t got = 0;
    while (got < nz && std::getline(in, line)) {
        lineno++;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream s(line);
        int64_t r, c;
        double v;
        if (!(s >> r >> c >> v)) return err("bad entry line");
        if (r < 1 || r > m || c < 1 || c > n) return err("index out of bounds");
        e.push_back({r - 1, {(int32_t)(c - 1), v}});
        if (sym && r != c) e.push_back({c - 1, {(int32_t)(r - 1), v}});
        got++;
    }
    if (got != nz) return err("fewer entries than the size line declares");
    std::stable_sort(e.begin(), e.end(), [](const auto &a, const auto &b) {
        return a.first != b.first ? a.first < b.first : a.second.first < b.second.first;
    });
    // duplicates summed, in file order
    std::vector<int64_t> rows;
    std::vector<int32_t> cols;
    std::vector<double> vals;
    for (size_t q = 0; q < e.size(); q++) {
        if (!rows.empty() && rows.back() == e[q].first && cols.back() == e[q].second.first)
            vals.back() += e[q].second.second;
        else {
            rows.push_back(e[q].first);
            cols.push_back(e[q].second.first);
            vals.push_back(e[q].second.second);
        }
    }
    const int64_t K = (int64_t)vals.size();
    if (K > (int64_t)INT32_MAX - 1 || m > (int64_t)INT32_MAX) return err("too large for the 32-bit paper layout");
    A->nrows = m;
    A->ncols = n;
    A->nnz = K;
    A->values = xmalloc<double>(K);
    A->cols = xmalloc<int>(K);
    A->pointerB = xmalloc<int>(m);
    A->pointerE = xmalloc<int>(m);
    if (!A->values || !A->cols || !A->pointerB || !A->pointerE) {
        svdsc_mat_csr_free(A);
        return fail(SVDSC_ENOMEM, "allocation failed");
    }
    int64_t q = 0;
    for (int64_t i = 0; i < m; i++) {
        A->pointerB[i] = (int)(q + 1);
        while (q < K && rows[q] == i) {
            A->cols[q] = cols[q] + 1;
            A->values[q] = vals[q];
            q++;
        }
        A->pointerE[i] = (int)(q + 1);
    }
    *is_dense = 0;
    return SVDSC_OK;
}

svdsc_status svdsc_write_mm(const char *path, const svdsc_mat_csr *A, const svdsc_mat *D) {
    if (!path || (!A) == (!D)) return fail(SVDSC_EINVAL, "exactly one of A, D must be given");
    FILE *f = std::fopen(path, "w");
    if (!f) return fail(SVDSC_EINVAL, std::string("cannot write ") + path);
    if (A) {
        int64_t nz = 0;
        for (int64_t i = 0; i < A->nrows; i++) nz += A->pointerE[i] - A->pointerB[i];
        std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)A->nrows,
                     (long long)A->ncols, (long long)nz);
        for (int64_t i = 0; i < A->nrows; i++)
            for (int64_t q = A->pointerB[i] - 1; q < A->pointerE[i] - 1; q++)
                std::fprintf(f, "%lld %d %.17g\n", (long long)(i + 1), A->cols[q], A->values[q]);
    } else {
        std::fprintf(f, "%%%%MatrixMarket matrix array real general\n%lld %lld\n", (long long)D->nrows,
                     (long long)D->ncols);
        for (int64_t j = 0; j < D->ncols; j++)
            for (int64_t i = 0; i < D->nrows; i++) std::fprintf(f, "%.17g\n", D->d[i + j * D->nrows]);
    }
    const bool ok = std::fclose(f) == 0;
    return ok ? SVDSC_OK : fail(SVDSC_EINVAL, "write failed");
}

}  // extern "C"
