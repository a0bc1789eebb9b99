// memo_residual.cpp -- measurement scaffolding (not product): what the Fisher
// memo set leaves to the CDF walk, and how much a further table of the most
// frequent remaining cell configurations would remove (lockstep model: a warp
// pays, per cell, the longest walk among its lanes that walk).
//
//   g++ -O2 -std=c++17 -fopenmp -ffp-contract=off -I paper_2201_06604_b200/csrc \
//       tools/memo_residual.cpp -o /tmp/memo_residual && /tmp/memo_residual 131072 17 26
//
// T10 drawn with the product sampler and memo set (fisher_sampler.cuh, host
// build), 32 consecutive tables per modelled warp; args: tables, log2 points
// per interior box, log2 record words (device level 1: 17 26).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <vector>

#include "exp_data.inc"
#include "fisher_sampler.cuh"

using namespace sfb;

static const uint64_t kTab[256] = SFB_EXP_TABLE_INIT;

static int walk_len(int k0, int lo, int hi, int k) {
    if (k == k0) return 0;
    const int du = hi - k0, dd = k0 - lo, m = std::min(du, dd);
    if (k > k0) {
        const int j = k - k0;
        return j <= m ? 2 * j - 1 : m * 2 + (j - m);
    }
    const int j = k0 - k;
    return j <= m ? 2 * j : m * 2 + (j - m);
}

int main(int argc, char **argv) {
    std::vector<int32_t> rows = {20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5};
    std::vector<int32_t> cols = {13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25};
    const long S = argc > 1 ? atol(argv[1]) : 131072;
    const int pts = argc > 2 ? atoi(argv[2]) : 17, words = argc > 3 ? atoi(argv[3]) : 26;
    const int nr = rows.size(), nc = cols.size();
    int ntot = 0;
    for (int r : rows) ntot += r;
    std::vector<double> lfv(ntot + 1);
    for (int k = 0; k <= ntot; ++k) lfv[k] = std::lgamma(k + 1.0);
    LfPlain lf{lfv.data()};
    HostMemo hm;
    build_memo_set(rows.data(), nr, cols.data(), nc, ntot, lf, kTab, hm, (size_t)1 << words,
                   kMemoSigmas, true, kMemoIntRadiusMax, (size_t)1 << pts);
    const MemoSet memo = hm.view();
    Mrg s{12345, 12345, 12345, 12345, 12345, 12345};
    std::vector<int> jw(nc);
    const int ncell = nr * nc;
    struct Visit { int cell; uint64_t key; int t; };
    std::vector<std::vector<Visit>> warps;
    std::vector<Visit> cur;
    std::unordered_map<uint64_t, std::pair<uint64_t, int>> cfg;  // key -> (count, len)
    double walked = 0, looked = 0, forced = 0, total = 0;
    for (long tab = 0; tab < S; ++tab) {
        int jc = ntot;
        for (int m = 0; m < nc - 1; ++m) jw[m] = cols[m];
        for (int l = 0; l < nr - 1; ++l) {
            int ia = rows[l];
            int ic = jc;
            jc -= ia;
            for (int m = 0; m < nc - 1; ++m) {
                const int idv = jw[m], ie = ic;
                ic -= idv;
                const uint32_t zm1 = step_m1(s);
                int lo = std::max(ia + idv - ie, 0);
                const int hi = std::min(ia, idv);
                int k;
                total++;
                if (hi <= lo) {
                    k = lo;
                    forced++;
                } else {
                    int log2s = 2;
                    const uint32_t *head = nullptr;
                    const uint32_t *rec = cell_record(l, m, nc, ia, idv, ie, memo, log2s, head);
                    k = rec ? memo_rec(head, rec, log2s, zm1, lo, hi) : -1;
                    if (k >= 0) {
                        looked++;
                    } else {
                        const int ib = ie - ia, ic2 = ie - idv, ii = ib - idv;
                        k = sample_cell_u<3>(u01_from_zm1(zm1), ia, idv, ie, ib, ic2, ii, lf, kTab);
                        int k0 = (int)((double)ia * ((double)idv / (double)ie) + 0.5);
                        k0 = std::min(std::max(k0, lo), hi);
                        const int t = walk_len(k0, lo, hi, k);
                        const uint64_t key = ((uint64_t)ia << 42) | ((uint64_t)idv << 21) | ie;
                        auto &c = cfg[key];
                        c.first++;
                        c.second = hi - lo + 1;
                        cur.push_back({l * nc + m, key, t});
                        walked++;
                    }
                }
                ia -= k;
                jw[m] = idv - k;
            }
        }
        if ((tab & 31) == 31) {
            warps.push_back(std::move(cur));
            cur.clear();
        }
    }
    const double W = S / 32.0;
    printf("T10 %ld tables, memo boxes 2^%d pts / 2^%d words: cells forced %.3f, record %.3f, "
           "walked %.3f; %zu distinct walked configs\n", S, pts, words, forced / total,
           looked / total, walked / total, cfg.size());
    std::vector<std::pair<uint64_t, uint64_t>> byc;
    for (auto &kv : cfg) byc.push_back({kv.second.first, kv.first});
    std::sort(byc.rbegin(), byc.rend());
    for (size_t K : {0ul, 16000ul, 64000ul, 256000ul, 1000000ul}) {
        std::unordered_map<uint64_t, int> in;
        size_t words_k = 0;
        for (size_t i = 0; i < std::min(K, byc.size()); ++i) {
            in[byc[i].second] = 1;
            words_k += cfg[byc[i].second].second;
        }
        double steps = 0, lock = 0, cov = 0, nv = 0;
        for (auto &wv : warps) {
            std::vector<int> mx(ncell, -1);
            for (auto &v : wv) {
                nv++;
                if (in.count(v.key)) {
                    cov++;
                    continue;
                }
                steps += v.t;
                mx[v.cell] = std::max(mx[v.cell], v.t);
            }
            for (int c = 0; c < ncell; ++c)
                if (mx[c] >= 0) lock += mx[c] + 1;
        }
        printf("extra table top %7zu (%8.1f MB): walked visits covered %.3f, mean walk steps/table "
               "%.1f, lockstep walk trips per table %.1f\n", K, words_k * 4 / 1e6,
               nv ? cov / nv : 0, steps / S, lock / W);
    }
    return 0;
}
