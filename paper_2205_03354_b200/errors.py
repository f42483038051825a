"""Error codes of the reference (`stencilkit::Errc`, error.hpp:9-28).

The C-ABI returns the Errc ordinal + 1 (0 = ok); device-side failures use
codes >= 100. `StencilkitError` mirrors `stencilkit::Error` (error.hpp:33-41):
it carries the machine-checkable code and the message.
"""
from __future__ import annotations

import enum


class Errc(enum.IntEnum):
    zero_scale = 0
    dim_mismatch = 1
    power_mismatch = 2
    empty_stencil = 3
    truncation_too_small = 4
    not_normalized = 5
    accuracy_exceeds_truncation = 6
    mixed_leading_order = 7
    singular_system = 8
    unsupported_accuracy = 9
    stencil_wider_than_grid = 10
    shape_mismatch = 11
    no_convergence = 12
    not_dissipative = 13
    unstable_for_all_dt = 14
    non_periodic = 15
    zero_denominator = 16
    invalid_argument = 17
    # device-side (no reference equivalent)
    cuda_error = 99
    out_of_memory = 100
    no_device = 101


ERRC_NAMES = {  # error.hpp:43-63
    Errc.zero_scale: "ZeroScale",
    Errc.dim_mismatch: "DimMismatch",
    Errc.power_mismatch: "PowerMismatch",
    Errc.empty_stencil: "EmptyStencil",
    Errc.truncation_too_small: "TruncationTooSmall",
    Errc.not_normalized: "NotNormalized",
    Errc.accuracy_exceeds_truncation: "AccuracyExceedsTruncation",
    Errc.mixed_leading_order: "MixedLeadingOrder",
    Errc.singular_system: "SingularSystem",
    Errc.unsupported_accuracy: "UnsupportedAccuracy",
    Errc.stencil_wider_than_grid: "StencilWiderThanGrid",
    Errc.shape_mismatch: "ShapeMismatch",
    Errc.no_convergence: "NoConvergence",
    Errc.not_dissipative: "NotDissipative",
    Errc.unstable_for_all_dt: "UnstableForAllDt",
    Errc.non_periodic: "NonPeriodic",
    Errc.zero_denominator: "ZeroDenominator",
    Errc.invalid_argument: "InvalidArgument",
    Errc.cuda_error: "CudaError",
    Errc.out_of_memory: "OutOfMemory",
    Errc.no_device: "NoDevice",
}


class StencilkitError(RuntimeError):
    """`stencilkit::Error`: RuntimeError carrying an `Errc` code."""

    def __init__(self, code: Errc, what: str):
        self.code = Errc(code)
        super().__init__(what if what.startswith(ERRC_NAMES[self.code]) else f"{ERRC_NAMES[self.code]}: {what}")


def status_to_errc(status: int) -> Errc:
    return Errc(status - 1)
