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
