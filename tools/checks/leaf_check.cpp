#include <cstdio>
#include <cstdlib>
#include <random>
#include "leaf.h"
using namespace isoc;
struct Ref { int64_t start, len; uint64_t hid; };
static Ref ref(int64_t total, int64_t pos) {
    int64_t s = 0, n = total; uint64_t h = 1;
    while (n > 128) { int64_t n2 = n >> 1; n2 -= n2 & 7; if (pos < s + n2) { n = n2; h <<= 1; } else { s += n2; n -= n2; h = (h << 1) | 1; } }
    return Ref{s, n, h};
}
int main(int argc, char** argv) {
    std::mt19937_64 rng(1);
    long bad = 0, checks = 0;
    auto walk = [&](int64_t total, int64_t pos, int steps) {
        Ref r = ref(total, pos);
        LeafIter it = leaf_iter_from(total, r.start, r.len, r.hid);
        for (int s = 0; s < steps; ++s) {
            ++checks;
            if (it.start != r.start || it.len != r.len || it.hid() != r.hid) {
                if (bad < 10) printf("total=%lld step=%d ref=(%lld,%lld,%llx) it=(%lld,%lld,%llx)\n", (long long)total, s,
                    (long long)r.start, (long long)r.len, (unsigned long long)r.hid, (long long)it.start, (long long)it.len,
                    (unsigned long long)it.hid());
                ++bad; return;
            }
            if (r.start + r.len >= total) return;
            r = ref(total, r.start + r.len);
            leaf_next(it, total);
        }
    };
    int small = argc > 1 ? atoi(argv[1]) : 30000, reps = argc > 2 ? atoi(argv[2]) : 3000;
    for (int64_t total = 1; total < small; ++total) walk(total, 0, 1 << 30);     // full walks
    for (int rep = 0; rep < reps; ++rep) {
        int64_t n = (int64_t)(rng() % 4000000) + 2;
        int64_t total = (rep & 1) ? n * n : (int64_t)(rng() % (1ll << 44)) + 129;
        for (int k = 0; k < 20; ++k) walk(total, (int64_t)(rng() % total), 3000);
        walk(total, total - 1, 5); walk(total, 0, 3000); walk(total, total - 2000, 100);
    }
    printf("checks=%ld bad=%ld\n", checks, bad);
    return bad != 0;
}
