/* scenes_rsa.c — seeded random sequential addition of spheres (BASELINE cfg3 inputs,
 * "positions by seeded random sequential addition (non-overlap check
 * on a hash grid)"). Input generation for bench.py / tests, not part of the C-ABI.
 *
 * Sphere s (radius R[s]) is added in index order; attempt t draws its centre uniformly
 * in [R_s, box - R_s] per axis with the reference's counter RNG (sfl/random_state.hpp:
 * draw k = 0, 1, 2 of particle s under seed + 1 + t) and is accepted when it overlaps
 * no earlier sphere. Placed spheres live in a hash grid of cell >= 2 max R (27-cell
 * check). Deterministic: the result depends on (R, box, seed) only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

static double draw(uint64_t seed, long i, uint64_t k) {
    const uint64_t x = mix(mix(seed ^ 0x6e61757469636c65ULL) ^ mix((uint64_t)i + 0x9e3779b9ULL) ^ k);
    return (double)(x >> 11) * 0x1.0p-53;
}

/* Returns 0, or the index + 1 of the first sphere still unplaced after max_tries. */
long nau_rsa_place(long n, const double* R, const double* box, uint64_t seed, int max_tries,
                   double* pos /* 3 x n, component-major */) {
    double rmax = 0.0;
    for (long s = 0; s < n; ++s) rmax = R[s] > rmax ? R[s] : rmax;
    const double cs = 2.0 * rmax;
    long nc[3];
    double csz[3];
    for (int a = 0; a < 3; ++a) {
        nc[a] = (long)floor(box[a] / cs);
        if (nc[a] < 1) nc[a] = 1;
        csz[a] = box[a] / (double)nc[a];
    }
    const long ncells = nc[0] * nc[1] * nc[2];
    long* head = (long*)malloc(sizeof(long) * (size_t)ncells);
    long* next = (long*)malloc(sizeof(long) * (size_t)(n > 0 ? n : 1));
    if (!head || !next) {
        free(head);
        free(next);
        return n + 1;
    }
    for (long c = 0; c < ncells; ++c) head[c] = -1;
    long rc = 0;
    for (long s = 0; s < n && rc == 0; ++s) {
        int ok = 0;
        for (int t = 0; t < max_tries && !ok; ++t) {
            double x[3];
            long ci[3];
            for (int a = 0; a < 3; ++a) {
                x[a] = R[s] + draw(seed + 1 + (uint64_t)t, s, (uint64_t)a) * (box[a] - 2.0 * R[s]);
                ci[a] = (long)floor(x[a] / csz[a]);
                if (ci[a] >= nc[a]) ci[a] = nc[a] - 1;
                if (ci[a] < 0) ci[a] = 0;
            }
            ok = 1;
            for (int dz = -1; dz <= 1 && ok; ++dz)
                for (int dy = -1; dy <= 1 && ok; ++dy)
                    for (int dx = -1; dx <= 1 && ok; ++dx) {
                        const long cx = ci[0] + dx, cy = ci[1] + dy, cz = ci[2] + dz;
                        if (cx < 0 || cy < 0 || cz < 0 || cx >= nc[0] || cy >= nc[1] || cz >= nc[2])
                            continue;
                        for (long j = head[(cz * nc[1] + cy) * nc[0] + cx]; j >= 0; j = next[j]) {
                            const double ddx = pos[j] - x[0], ddy = pos[n + j] - x[1],
                                         ddz = pos[2 * n + j] - x[2];
                            const double rr = R[j] + R[s];
                            if (ddx * ddx + ddy * ddy + ddz * ddz < rr * rr) {
                                ok = 0;
                                break;
                            }
                        }
                    }
            if (ok) {
                for (int a = 0; a < 3; ++a) pos[a * n + s] = x[a];
                const long c = (ci[2] * nc[1] + ci[1]) * nc[0] + ci[0];
                next[s] = head[c];
                head[c] = s;
            }
        }
        if (!ok) rc = s + 1;
    }
    free(head);
    free(next);
    return rc;
}
