// memo_probe.cpp -- measurement scaffolding (not product): how the Fisher
// kernel's lockstep cost splits over cells and how much of it a memo of the
// most frequent cell configurations (ia, idv, ie) would remove.
//
//   g++ -O2 -std=c++17 -ffp-contract=off -I paper_2201_06604_b200/csrc \
//       tools/memo_probe.cpp -o /tmp/memo_probe && /tmp/memo_probe T10 65536
//
// Tables are drawn with the product sampler (fisher_sampler.cuh, host build)
// from one MRG31k3p stream; 32 consecutive tables model one warp's lanes.
// For every free cell the walk length t is recovered from (k0, lo, hi, k).
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

struct Cfg {
    uint64_t count = 0, steps = 0;
    int len = 0;  // sequence length of the full walk (to u_max)
};

static int walk_len(int k0, int lo, int hi, int k) {
    // t with k(t) == k for the alternating walk started at k0
    if (k == k0) return 0;
    const int du = hi - k0, dd = k0 - lo, m = std::min(du, dd);
    if (k > k0) {
        const int j = k - k0;  // j-th up step
        return j <= m ? 2 * j - 1 : m * 2 + (j - m);
    }
    const int j = k0 - k;
    return j <= m ? 2 * j : m * 2 + (j - m);
}

int main(int argc, char **argv) {
    std::vector<int32_t> rows, cols;
    const char *name = argc > 1 ? argv[1] : "T10";
    if (!strcmp(name, "T4")) {
        int t[4][4] = {{5, 9, 5, 7}, {9, 5, 9, 7}, {8, 6, 2, 6}, {10, 8, 8, 8}};
        rows.assign(4, 0);
        cols.assign(4, 0);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) rows[i] += t[i][j], cols[j] += t[i][j];
    } else {
        rows = {20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5};
        cols = {13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25};
    }
    const long S = argc > 2 ? atol(argv[2]) : 65536;
    const int nr = rows.size(), nc = cols.size();
    int ntot = 0;
    for (int r : rows) ntot += r;
    std::vector<double> lfv(ntot + 1);
    for (int k = 0; k <= ntot; ++k) lfv[k] = std::lgamma(k + 1.0);
    LfPlain lf{lfv.data()};
    Mrg s{12345, 12345, 12345, 12345, 12345, 12345};
    std::vector<int> jw(nc);
    const int ncell = nr * nc;
    // per warp-cell: lane steps + configs
    std::vector<std::vector<int>> tsteps(ncell, std::vector<int>(32));
    std::vector<std::vector<uint64_t>> tkey(ncell, std::vector<uint64_t>(32));
    std::vector<double> cell_steps(ncell), cell_max(ncell);
    std::unordered_map<uint64_t, Cfg> cfgs;
    struct Visit { int cell; uint64_t key; int t; };
    std::vector<Visit> visits;
    std::vector<std::vector<Visit>> warp_visits;  // per warp
    for (long tab = 0; tab < S; ++tab) {
        const int lane = tab & 31;
        for (int c = 0; c < ncell; ++c) tsteps[c][lane] = -1;
        int jc = ntot;
        for (int m = 0; m < nc - 1; ++m) jw[m] = cols[m];
        for (int l = 0; l < nr - 1; ++l) {
            int ia = rows[l];
            int ic = jc;
            jc -= ia;
            for (int m = 0; m < nc - 1; ++m) {
                const int idv = jw[m], ie = ic;
                ic -= idv;
                const int ib = ie - ia, ii = ib - idv;
                const int k = sample_cell<1>(ia, idv, ie, ib, ic, ii, lf, kTab, s);
                int lo = std::max(ia + idv - ie, 0), hi = std::min(ia, idv);
                if (hi > lo) {
                    int k0 = (int)((double)ia * ((double)idv / (double)ie) + 0.5);
                    k0 = std::min(std::max(k0, lo), hi);
                    const int t = walk_len(k0, lo, hi, k);
                    const uint64_t key = ((uint64_t)ia << 42) | ((uint64_t)idv << 21) | ie;
                    Cfg &cf = cfgs[key];
                    cf.count++;
                    cf.steps += t;
                    if (!cf.len) cf.len = hi - lo + 1;
                    tsteps[l * nc + m][lane] = t;
                    tkey[l * nc + m][lane] = key;
                    cell_steps[l * nc + m] += t;
                }
                ia -= k;
                jw[m] = idv - k;
            }
        }
        if (lane == 31) {
            for (int c = 0; c < ncell; ++c) {
                int mx = -1;
                for (int q = 0; q < 32; ++q) mx = std::max(mx, tsteps[c][q]);
                if (mx >= 0) cell_max[c] += mx;
            }
            std::vector<Visit> wv;
            for (int c = 0; c < ncell; ++c)
                for (int q = 0; q < 32; ++q)
                    if (tsteps[c][q] >= 0) wv.push_back({c * 32 + q, tkey[c][q], tsteps[c][q]});
            warp_visits.push_back(std::move(wv));
        }
    }
    const double W = S / 32.0;
    printf("%s: %ld tables, %zu distinct configs\n", name, S, cfgs.size());
    double tot_steps = 0, tot_max = 0;
    for (int c = 0; c < ncell; ++c) tot_steps += cell_steps[c], tot_max += cell_max[c];
    printf("mean walk steps/table %.1f, lockstep (max of 32) steps per table %.1f\n",
           tot_steps / S, tot_max / W);
    printf("per cell: mean steps / lockstep max (per table-warp):\n");
    for (int l = 0; l < nr - 1; ++l) {
        for (int m = 0; m < nc - 1; ++m)
            printf(" %5.1f/%5.1f", cell_steps[l * nc + m] / S, cell_max[l * nc + m] / W);
        printf("\n");
    }
    // rank configs by count
    // configs of first-row / first-column cells: always memoised (the
    // current kernel's one-parameter memo); the ranking covers the others
    std::unordered_map<uint64_t, int> rowcol;
    for (auto &wv : warp_visits)
        for (auto &v : wv) {
            const int c = v.cell / 32;
            if (c / nc == 0 || c % nc == 0) rowcol[v.key] = 1;
        }
    std::vector<std::pair<uint64_t, uint64_t>> byc;
    for (auto &kv : cfgs)
        if (!rowcol.count(kv.first)) byc.push_back({kv.second.count, kv.first});
    std::sort(byc.rbegin(), byc.rend());
    const double cs = 60, cw0 = 70, cstep = 31;
    for (size_t K : {0ul, 1000ul, 4000ul, 16000ul, 64000ul, 256000ul, 1000000ul, 4000000ul}) {
        if (K > byc.size() + 1000000) break;
        std::unordered_map<uint64_t, int> in = rowcol;
        size_t entries = 0;
        for (size_t i = 0; i < std::min(K, byc.size()); ++i) {
            in[byc[i].second] = 1;
            entries += cfgs[byc[i].second].len;
        }
        // warp cost model per cell
        double cost = 0, covered = 0, nvis = 0;
        for (auto &wv : warp_visits) {
            // group by cell
            std::vector<int> hit(ncell, 0), miss_max(ncell, -1);
            for (auto &v : wv) {
                const int c = v.cell / 32;
                nvis++;
                if (in.count(v.key)) {
                    hit[c] = 1;
                    covered++;
                } else
                    miss_max[c] = std::max(miss_max[c], v.t);
            }
            for (int c = 0; c < ncell; ++c) {
                if (hit[c]) cost += cs;
                if (miss_max[c] >= 0) cost += cw0 + cstep * miss_max[c];
            }
        }
        printf("memo top %7zu configs (%9zu entries, %6.1f MB at 4 B): visits covered %.3f, "
               "model warp-instr per table %.0f\n",
               K, entries, entries * 4 / 1e6, covered / nvis, cost / W);
    }
    return 0;
}
