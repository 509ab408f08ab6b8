"""The plan rule of DESIGN.md section 5, restated independently of the CUDA library.

Tests hand these plans to the oracle (so no oracle input comes from the CUDA path)
and check that the library's ``gbs_plan`` reports the same numbers.

A plan is a list of levels [(L, s), ...]; level k+1 sorts the buckets of level k
(its problem capacity is level k's tight bucket bound).  An empty plan means a
single on-chip sort.
"""

TILE_KEYS = 1 << 15     # u32 keys per CTA tile (128 KB of shared memory)
TILE_PAIRS = 1 << 14    # (key, value) pairs per CTA tile
D_MIN = 8               # a single level needs d = L/s >= 8 (samples <= n/8)
D_NEST = 32             # d of a level whose buckets need a nested level
PAIR_BELOW_D = 16       # keys: sublists of two tiles (CTA pairs) when the one-tile d is below
SMALL_TILE = 1 << 11    # the small CTA configuration's tile (the paper's 2K sublists)
SMALL_N_KEYS = 1 << 17  # keys problems up to this size: 2K sublists and buckets (latency: more CTAs)
MAX_S = 4096            # samples per sublist Steps 6 and 8 hold in shared memory


def hi_bound(cap: int, L: int, s: int) -> int:
    """Tight upper bucket bound n'/s + (m-1)(d-1), n' = ceil(cap/L) L."""
    m = -(-cap // L)
    d = L // s
    return m * L // s + (m - 1) * (d - 1)


def plan(n: int, tile: int = TILE_KEYS, cfg=None):
    levels = []
    cap = n
    if cfg is not None and n > 1:          # explicit level-1 (L, s), e.g. the paper's
        levels.append(tuple(cfg))          # (2048, 64) of P:249-250
        cap = hi_bound(n, *cfg)
    if not levels and tile == TILE_KEYS and tile < n <= SMALL_N_KEYS:
        # small keys problem: 2K sublists when some s (d >= D_MIN) gives buckets of <= 2K
        s = 2
        while s <= SMALL_TILE // D_MIN:
            if hi_bound(n, SMALL_TILE, s) <= SMALL_TILE:
                return [(SMALL_TILE, s)]
            s *= 2
    while cap > tile:
        L = tile
        chosen = None
        s = 2
        while s <= L // D_MIN:
            if hi_bound(cap, L, s) <= tile:
                chosen = s
                break
            s *= 2
        # keys: if the one-tile level needs d < 16, sublists of two tiles (sorted by a
        # CTA pair) with buckets still one tile, when that is one level too
        if tile == TILE_KEYS and chosen is not None and L // chosen < PAIR_BELOW_D:
            s = 2
            while s <= 2 * tile // D_MIN:
                if hi_bound(cap, 2 * tile, s) <= tile:
                    L, chosen = 2 * tile, s
                    break
                s *= 2
        if chosen is not None:
            levels.append((L, chosen))
            break
        # keys, top level: buckets of two tiles (sorted by a CTA pair) when that gives
        # one level -- sublists of two tiles first, then one tile
        if tile == TILE_KEYS and not levels:
            for Lc in (2 * tile, tile):
                s = 2
                while s <= Lc // D_MIN and s <= MAX_S and chosen is None:
                    if hi_bound(cap, Lc, s) <= 2 * tile:
                        L, chosen = Lc, s
                    s *= 2
                if chosen is not None:
                    break
            if chosen is not None:
                levels.append((L, chosen))
                break
        s = L // D_NEST
        levels.append((L, s))
        cap = hi_bound(cap, L, s)
    return levels
