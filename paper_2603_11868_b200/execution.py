"""Execution policies and the kernel-dispatch boundary.

Mirror of the reference's ``minisph/execution.py`` interface.  The reference
crosses into native code at ``kernel.driver()(range_size, args)``
(execution.py:129) and at its reduce driver (execution.py:206); here both
cross into libsphb200.so (sm_100a) through the C ABI in include/sph_b200.h.

Every policy executes on the GPU: the reference's three variants
(sequenced, parallel, parallel_device) give bit-identical results by design
(execution.py:4-7), and so does the CUDA path, which reproduces the
reference's ascending-id accumulation order.  ``ExecutionPolicy.cuda()``
names the device explicitly.  Kernels are dispatched by identity to their
native entry point; a kernel with no native implementation raises
NotImplementedError -- there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEQUENCED = "sequenced"
PARALLEL = "parallel"
PARALLEL_DEVICE = "parallel_device"
CUDA = "cuda"

_VARIANTS = (SEQUENCED, PARALLEL, PARALLEL_DEVICE, CUDA)


@dataclass(frozen=True)
class ExecutionPolicy:
    """execution.py:30-59, plus the ``cuda`` variant (device index)."""
    variant: str
    workers: int = 1
    device: int = 0

    def __post_init__(self):
        if self.variant not in _VARIANTS:
            raise ValueError(f"unknown policy variant {self.variant!r}")
        if self.workers < 1:
            raise ValueError("worker count must be positive")

    @property
    def is_parallel(self):
        return self.variant != SEQUENCED

    @property
    def is_device(self):
        return self.variant in (PARALLEL_DEVICE, CUDA)

    @staticmethod
    def sequenced():
        return ExecutionPolicy(SEQUENCED)

    @staticmethod
    def parallel(workers):
        return ExecutionPolicy(PARALLEL, workers)

    @staticmethod
    def parallel_device(workers):
        return ExecutionPolicy(PARALLEL_DEVICE, workers)

    @staticmethod
    def cuda(device=0):
        return ExecutionPolicy(CUDA, 1, int(device))


def effective_threads(policy):
    """Host worker threads in the reference (execution.py:62-66); the CUDA
    path uses one host thread for every policy."""
    return 1


def validate_device_args(args):
    """The device binding surface: flat arrays and plain values only
    (execution.py:79-90).  CUDA tensors count as arrays."""
    from ._device import is_tensor
    for a in args:
        if isinstance(a, np.ndarray) or is_tensor(a):
            continue
        if isinstance(a, (int, float, np.integer, np.floating, np.bool_, bool)):
            continue
        if isinstance(a, tuple):
            validate_device_args(a)
            continue
        raise TypeError(
            f"device kernels may bind only arrays and plain values, got {type(a)!r}")


class ParticleKernel:
    """A per-index procedure (execution.py:93-113).

    ``native(policy, range_size, args)`` is the CUDA implementation; kernels
    built from a plain Python body have none and cannot be dispatched.
    """

    def __init__(self, body=None, name=None, native=None):
        self.body = body
        self.name = name or getattr(body, "__name__", "kernel")
        self.native = native

    def __repr__(self):
        return f"ParticleKernel({self.name})"


def particle_kernel(body):
    return ParticleKernel(body)


def particle_for(policy, range_size, kernel, args=()):
    """Invoke ``kernel`` once per index in 0..range_size-1 (execution.py:121-129)."""
    if range_size == 0:
        return
    args = tuple(args)
    validate_device_args(args)
    if kernel.native is None:
        raise NotImplementedError(
            f"{kernel!r} has no CUDA implementation (no CPU fallback)")
    kernel.native(policy, int(range_size), args)


@dataclass(frozen=True)
class ReduceSpec:
    """identity, per-index transform, combine (execution.py:134-145);
    ``native`` is the CUDA reduction."""
    identity: object
    transform: object
    combine: object
    native: object = None


def chunk_bounds(n, workers):
    """The reference's chunk layout (execution.py:170-178), kept for API
    completeness; the CUDA reductions are exact max folds and do not chunk."""
    if n == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    size = max(1024, -(-n // (4 * workers)))
    starts = np.arange(0, n, size, dtype=np.int64)
    stops = np.minimum(starts + size, n)
    return starts, stops


def particle_reduce(policy, range_size, spec, args=()):
    """Combine-fold of spec.transform over 0..range_size-1 (execution.py:191-209)."""
    if range_size == 0:
        return spec.identity
    args = tuple(args)
    validate_device_args(args)
    if spec.native is None:
        raise NotImplementedError("reduction has no CUDA implementation")
    return spec.native(policy, int(range_size), args)


def dispatch_dynamics(policy, dynamics):
    """Kernel-shell object: host setup once, kernel under policy (execution.py:212-215)."""
    range_size, args = dynamics.setup()
    particle_for(policy, range_size, dynamics.kernel, args)
