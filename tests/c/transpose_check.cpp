// The parallel transpose of csrc/graph_build.h equals the serial scatter (row v lists its sources
// ascending) on a skewed random pattern with hub rows and empty rows.  Prints "ok".
#include <cstdio>
#include <random>

#include "graph_build.h"

int main() {
    const int64_t n = 300000, m = 4000000;
    std::mt19937_64 g(7);
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> col(m);
    for (int64_t u = 0; u <= n; ++u) rp[u] = m * u / n;
    for (int64_t k = 0; k < m; ++k) {
        const double x = (double)(g() >> 11) / 9007199254740992.0;
        col[k] = (int32_t)((double)n * x * x * x * x);          // power law: hub targets near 0
    }
    for (int64_t u = 0; u < n; ++u) {                            // unique targets per row
        std::sort(col.begin() + rp[u], col.begin() + rp[u + 1]);
    }
    std::vector<int64_t> urp(n + 1, 0);
    std::vector<int32_t> ucol;
    for (int64_t u = 0; u < n; ++u) {
        int64_t b = (int64_t)ucol.size();
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
            if ((int64_t)ucol.size() == b || ucol.back() != col[k]) ucol.push_back(col[k]);
        urp[u + 1] = (int64_t)ucol.size();
    }
    std::vector<int64_t> trp;
    std::vector<int32_t> tcol;
    tc::transpose(n, urp, ucol, trp, tcol);
    std::vector<int64_t> rtrp(n + 1, 0);
    for (int32_t v : ucol) rtrp[v + 1]++;
    for (int64_t i = 0; i < n; ++i) rtrp[i + 1] += rtrp[i];
    std::vector<int32_t> rcol(ucol.size());
    std::vector<int64_t> pos(rtrp.begin(), rtrp.end() - 1);
    for (int64_t u = 0; u < n; ++u)
        for (int64_t k = urp[u]; k < urp[u + 1]; ++k) rcol[pos[ucol[k]]++] = (int32_t)u;
    if (trp != rtrp || tcol != rcol) { std::printf("mismatch\n"); return 1; }
    std::printf("ok\n");
    return 0;
}
