"""Error bars of the random-input parity tests (R11).

* north_star ceiling: scaled error max|C - C_ref| / (n max|A| max|B|) <= 1e-13
  per recursion level used (classical: one level's worth);
* model guard: <= 10x the error model measured for uniform[-1,1) inputs --
  about 1e-16 * 2^L (profiles/error_growth_r01.json: 0.8, 1.5, 2.7, 5.1, 10.0
  e-16 at L = 0..4 against the definition in extended precision; x1.9 per
  Strassen-Winograd level, x1.65 per Laderman level), so a 10x regression in
  the leaf's accumulation or the additions fails even though it stays far
  inside the ceiling.  L counts levels of a 2x2 triple; a 3x3 or 4x4 level
  counts as its own L (Laderman grows slower, <4,4,4;49> = two SW levels is
  covered by passing L = 2).  The guard scales with |alpha| like the error.
"""


def ceiling(levels: int) -> float:
    return 1e-13 * max(1, levels)


def model_guard(levels: int) -> float:
    return 10 * 1e-16 * 2.0 ** max(1, levels)


def assert_error(err: float, levels: int, scale: float = 1.0, what=""):
    assert err <= ceiling(levels) * scale, (what, err, "north_star ceiling", ceiling(levels) * scale)
    assert err <= model_guard(levels) * scale, (what, err, "10x error model", model_guard(levels) * scale)
