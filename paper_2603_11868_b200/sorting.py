"""Stable particle reordering by cell key (mirror of ``minisph/sorting.py``).

``radix_sort_permutation`` is the device LSD radix sort (csrc/sort.cu): 8-bit
digits, ``ceil(bit_length(max_key) / 8)`` passes, stable, so it equals the
stable comparison sort exactly (sorting.py:46-70).
``comparison_sort_permutation`` stays the host reference path (numpy stable
argsort), as in the reference, where it is the radix sort's oracle.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import Staging, device_of, is_tensor, ptr, stream_ptr, workspace
from .neighborhood import compute_cell_keys

RADIX_BITS = 8
RADIX_SIZE = 1 << RADIX_BITS


def comparison_sort_permutation(keys):
    """Stable comparison-based permutation (sorting.py:22-24)."""
    return np.argsort(np.asarray(keys), kind="stable").astype(np.int64)


def radix_sort_permutation(policy, keys):
    """Stable LSD radix permutation of non-negative integer keys on the GPU;
    ValueError on a negative key (sorting.py:52-53)."""
    torch = __import__("torch")
    on_device = is_tensor(keys)
    if not on_device:
        keys = np.ascontiguousarray(np.asarray(keys), dtype=np.int64)
    n = keys.shape[0]
    if n == 0:
        return np.zeros(0, np.int64)
    lib = _native.lib()
    dev = keys.device if on_device else device_of(policy)
    with Staging(dev) as st:
        k = st.to_dev(keys if not on_device else keys.to(torch.int64))
        perm = torch.empty(n, dtype=torch.int64, device=dev)
        ws_bytes = lib.sph_sort_workspace_bytes(n)
        ws = workspace(dev, ws_bytes)
        rc = lib.sph_radix_sort_perm(ptr(k), n, ptr(perm), ptr(ws), ws_bytes,
                                     stream_ptr(dev))
        _native.check(rc, "radix_sort_permutation")
        if on_device:
            return perm
        return perm.cpu().numpy()


def sort_particles(policy, registry, keys, exempt_names=()):
    """Reorder all discrete variables by key with the device radix sort
    (sorting.py:73-81); returns the permutation applied."""
    perm = radix_sort_permutation(policy, keys)
    registry.apply_permutation(perm, exempt_names)
    return perm


def sort_particles_by_cell(policy, registry, grid):
    """Cell keys from current positions, then reorder (sorting.py:84-87)."""
    keys, _ = compute_cell_keys(registry.view("x"), grid, policy)
    return sort_particles(policy, registry, keys)
