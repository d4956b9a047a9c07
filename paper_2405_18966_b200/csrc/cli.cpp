// svdsc-cli -- batch harness over libsvdsc (SPEC.md cli module):
//
//   svdsc-cli decompose --input A.mtx --k K [--tol 1e-10] [--t T] [--restarts R]
//                       [--seed S] [--output result.json|result.csv]
//
// Reads a Matrix Market file (coordinate -> sparse path, array -> dense path),
// runs svds-C (Alg. 2) on the current CUDA device through the host-buffer C-ABI
// entry points and writes the singular values, Eq. (4) residuals and run
// statistics.  Exit status: 0 converged, 2 returned but not converged, 1 error.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/svdsc_paper.h"

namespace {

int usage(const char *msg) {
    std::fprintf(stderr,
                 "error: %s\nusage: svdsc-cli decompose --input A.mtx --k K [--tol TOL] [--t T] "
                 "[--restarts R] [--seed S] [--output out.json|out.csv]\n",
                 msg);
    return 1;
}

std::string basename_of(const std::string &p) {
    const size_t s = p.find_last_of('/');
    return s == std::string::npos ? p : p.substr(s + 1);
}

}  // namespace

int main(int argc, char **argv) {
    if (argc < 2 || std::string(argv[1]) != "decompose") return usage("the only subcommand is 'decompose'");
    std::string input, output;
    int k = 0, t = 0, restarts = 10;
    double tol = 1e-10;
    unsigned long long seed = 0;
    for (int i = 2; i < argc; i++) {
        const std::string a = argv[i];
        auto val = [&]() -> const char * { return i + 1 < argc ? argv[++i] : nullptr; };
        const char *v = nullptr;
        if (a == "--input" && (v = val())) input = v;
        else if (a == "--output" && (v = val())) output = v;
        else if (a == "--k" && (v = val())) k = std::atoi(v);
        else if (a == "--t" && (v = val())) t = std::atoi(v);
        else if (a == "--restarts" && (v = val())) restarts = std::atoi(v);
        else if (a == "--tol" && (v = val())) tol = std::atof(v);
        else if (a == "--seed" && (v = val())) seed = std::strtoull(v, nullptr, 10);
        else return usage(("unknown or incomplete flag " + a).c_str());
    }
    if (input.empty()) return usage("--input is required");
    if (k < 1) return usage("--k must be >= 1");
    if (!(tol > 0.0)) return usage("--tol must be > 0");
    if (restarts < 1) return usage("--restarts must be >= 1");

    svdsc_mat_csr A;
    svdsc_mat D;
    int dense = 0;
    if (svdsc_read_mm(input.c_str(), &A, &D, &dense) != SVDSC_OK) {
        std::fprintf(stderr, "error: %s\n", svdsc_paper_last_error());
        return 1;
    }
    const int64_t m = dense ? D.nrows : A.nrows, n = dense ? D.ncols : A.ncols;
    int64_t nnz = dense ? m * n : A.nnz;
    svdsc_handle *h = nullptr;
    if (svdsc_create(&h, nullptr) != SVDSC_OK) {
        std::fprintf(stderr, "error: no CUDA device (svdsc_create failed)\n");
        return 1;
    }
    svdsc_opts o;
    std::memset(&o, 0, sizeof(o));
    o.k = k;
    o.tol = tol;
    o.t = t;
    o.maxit = restarts;
    o.seed = seed;
    o.reorth = 2;
    std::vector<double> S(k), U((size_t)m * k), V((size_t)n * k), R(k);
    svdsc_info info;
    std::memset(&info, 0, sizeof(info));
    svdsc_status st;
    if (dense) {
        st = svdsc_solve_host_dense(h, m, n, D.d, &o, S.data(), U.data(), V.data(), R.data(), &info);
    } else {
        int64_t *rp = nullptr;
        int32_t *ci = nullptr;
        double *va = nullptr;
        st = svdsc_paper_csr_to_csr(&A, &rp, &ci, &va, &nnz);
        if (st == SVDSC_OK)
            st = svdsc_solve_host_csr(h, m, n, nnz, rp, ci, va, &o, S.data(), U.data(), V.data(), R.data(), &info);
        else
            std::fprintf(stderr, "error: %s\n", svdsc_paper_last_error());
        std::free(rp);
        std::free(ci);
        std::free(va);
    }
    if (st < 0) {
        std::fprintf(stderr, "error: %s\n", svdsc_last_error(h));
        svdsc_destroy(h);
        return 1;
    }
    const bool csv = output.size() >= 4 && output.compare(output.size() - 4, 4, ".csv") == 0;
    FILE *f = output.empty() ? stdout : std::fopen(output.c_str(), "w");
    if (!f) {
        std::fprintf(stderr, "error: cannot write %s\n", output.c_str());
        svdsc_destroy(h);
        return 1;
    }
    if (csv) {
        std::fprintf(f, "index,sigma,residual\n");
        for (int j = 0; j < k; j++) std::fprintf(f, "%d,%.17g,%.17g\n", j + 1, S[j], R[j]);
    } else {
        std::fprintf(f, "{\"matrix_name\": \"%s\", \"m\": %lld, \"n\": %lld, \"nnz\": %lld, ",
                     basename_of(input).c_str(), (long long)m, (long long)n, (long long)nnz);
        std::fprintf(f, "\"options\": {\"k\": %d, \"tol\": %.17g, \"t\": %d, \"restarts\": %d, \"seed\": %llu}, ", k,
                     tol, info.t_used, restarts, seed);
        std::fprintf(f, "\"singular_values\": [");
        for (int j = 0; j < k; j++) std::fprintf(f, "%s%.17g", j ? ", " : "", S[j]);
        std::fprintf(f, "], \"residuals\": [");
        for (int j = 0; j < k; j++) std::fprintf(f, "%s%.17g", j ? ", " : "", R[j]);
        std::fprintf(f,
                     "], \"restarts\": %d, \"converged\": %s, \"matvecs\": %lld, \"steps\": %lld, "
                     "\"wall_time_seconds\": %.6f, \"device\": \"cuda\"}\n",
                     info.restarts, info.converged ? "true" : "false", (long long)info.matvecs,
                     (long long)info.steps, info.seconds_total);
    }
    if (f != stdout) std::fclose(f);
    svdsc_destroy(h);
    if (dense) svdsc_mat_free(&D);
    else svdsc_mat_csr_free(&A);
    return st == SVDSC_NOT_CONVERGED ? 2 : 0;
}
