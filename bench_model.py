"""Algorithmic work per candidate pair (SURVEY.md §8(d) 'Algorithmic per-pair
cost' table: FMA-pipe instructions of the method's necessary arithmetic).
Roofline convention of the survey: 1 FMA-pipe instruction = 2 FP32 flops,
peak = 148 SM x 128 lanes x 2 x f_sm.  DESIGN.md §6 restates the table and
compares it with the ncu-measured instruction counts of our kernels."""

# (R, N) -> (hit, miss) FMA-pipe instructions per pair
TABLE = {
    (1, 4): (173.0, 21.0),
    (1, 6): (251.0, 21.0),
    (1, 8): (337.0, 21.0),
    (2, 6): (6350.0, 180.0),
    (2, 8): (8130.0, 180.0),
}


def fma_insts(R, N, hit_pairs, candidates):
    if (R, N) in TABLE:
        hit, miss = TABLE[(R, N)]
    elif R == 1:   # linear in N between the survey's rows (+~41 per GL point)
        hit, miss = 173.0 + 41.0 * (N - 4), 21.0
    else:
        hit, miss = 6350.0 + 890.0 * (N - 6), 180.0
    return hit * hit_pairs + miss * (candidates - hit_pairs)


def flops(R, N, hit_pairs, candidates):
    return 2.0 * fma_insts(R, N, hit_pairs, candidates)


def flops_curved(hit_pairs, candidates, N, P):
    return flops(2, N, hit_pairs, candidates)


# Surface forests (NEXT(3), surface.cu): fp64 FMA-pipe instructions per pair
# of the ray-patch method (App. A.1), counted from the
# arithmetic the method needs: per candidate the ray (6), the element's four
# corner points from the tree patch (36), their projection onto d1, d2 (24),
# the basis (12), the bilinear coefficients and the quadratic (20); per hit
# root s1 (6), the point and the two tangents (27), alpha (4), the normal and
# cos phi (12).  1 FMA-pipe instruction = 2 flops.
SURFACE_MISS, SURFACE_HIT = 98.0, 49.0


def surface_flops(hit_pairs, candidates):
    return 2.0 * (SURFACE_MISS * candidates + SURFACE_HIT * hit_pairs)
