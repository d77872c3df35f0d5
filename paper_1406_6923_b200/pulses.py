"""Source time functions (mirror of reference sim.py:80-97).

Profiles are host callables, as in the reference (SourceTerm.profile); the
stepper evaluates them once per step into a table that the kernel reads.
"""

from __future__ import annotations

import math


def ricker(f_peak: float, delay: float):
    """sim.py:80-85."""
    def pulse(t: float) -> float:
        a = (math.pi * f_peak * (t - delay)) ** 2
        return (1.0 - 2.0 * a) * math.exp(-a)

    # (kind, f, delay): lets the stepper tabulate long runs in the library (sfw_pulse_table),
    # bit-identical to calling pulse(t) per step
    pulse.sfw_pulse = (0, float(f_peak), float(delay))
    return pulse


def gauss_deriv(f_peak: float, delay: float):
    """sim.py:88-94 (scaled so the extrema are +-1)."""
    def pulse(t: float) -> float:
        x = math.pi * f_peak * (t - delay)
        return -x * math.sqrt(2.0 * math.e) * math.exp(-x * x)

    pulse.sfw_pulse = (1, float(f_peak), float(delay))
    return pulse


PULSES = {"ricker": ricker, "gauss_deriv": gauss_deriv}


def make_pulse(profile: str, f_peak: float, delay: float):
    return PULSES[profile](f_peak, delay)
