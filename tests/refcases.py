"""Shared helpers: turn a golden case row into an oracle request (tests only)."""

from oracle import oracle as O


def case_state(engine, seed, skip):
    """Engine state in oracle form: ('philox', key, position) or ('mrg', s1, s2)."""
    if engine == "philox":
        return (O.seed_philox(seed), skip)
    s1, s2 = O.seed_mrg(seed)
    if skip:
        s1, s2 = O.mrg_skip(s1, s2, skip)
    return (s1, s2)


def oracle_case(case):
    name, engine, seed, skip, dist, prec, p0, p1, n = case
    return O.generate(engine, case_state(engine, seed, skip), dist, n, prec, p0, p1)
