"""CPU restatement of calosim.simulate_event's deposition -- TEST/BENCH ONLY.

Follows pkg/src/portarng/calosim.py:313-347 line for line in numpy (the same
operations, so numpy's own summation orders apply): triples from the event's
fp32 batch cast to fp64, cell pick, searchsorted energy bin, raw energies,
per-particle normalisation, np.unique + np.bincount deposits.  Used to pin
the GPU consumer (tests) and as the C5 CPU baseline (bench.py).
"""

from __future__ import annotations

import numpy as np


def deposit_event(batch_f32: np.ndarray, particles, hits, region_cell_ids, params, regions: int,
                  sampling_fraction: float = 1.0):
    """particles: [(kind, energy, direction)]; hits: per-particle hit counts;
    params: kind -> (bin_edges, weights).  Returns (deposits, particle_sums)."""
    host = batch_f32.astype(np.float64)  # calosim.py:311
    all_ids, all_amounts, particle_sums = [], [], []
    offset = 0
    for (kind, energy, direction), m in zip(particles, hits):
        if m == 0:
            particle_sums.append(0.0)
            continue
        edges, weights = params[kind]
        triples = host[offset: offset + 3 * m].reshape(m, 3)
        offset += 3 * m
        region = min(int((direction[2] + 1.0) * 0.5 * regions), regions - 1)
        region_cells = region_cell_ids[region]
        cell_idx = np.minimum((triples[:, 0] * len(region_cells)).astype(np.int64), len(region_cells) - 1)
        cell_ids = region_cells[cell_idx]
        cumw = np.cumsum(weights)
        bin_idx = np.minimum(np.searchsorted(cumw, triples[:, 1], side="right"), len(weights) - 1)
        raw = edges[bin_idx] + triples[:, 2] * (edges[bin_idx + 1] - edges[bin_idx])
        target = energy * sampling_fraction
        raw_sum = float(raw.sum())
        amounts = raw * (target / raw_sum) if raw_sum > 0 else np.full(m, target / m)
        all_ids.append(cell_ids)
        all_amounts.append(amounts)
        particle_sums.append(float(amounts.sum()))
    deposits = {}
    if all_ids:
        ids_cat = np.concatenate(all_ids)
        amounts_cat = np.concatenate(all_amounts)
        uniq, inverse = np.unique(ids_cat, return_inverse=True)
        sums = np.bincount(inverse, weights=amounts_cat)
        deposits = dict(zip(uniq.tolist(), sums.tolist()))
    return deposits, particle_sums
