"""Comparison used by every GPU parity test (not a pytest module).

rel(got, want) is the larger of
  * the north_star norm error  ||got - want|| / ||want||, and
  * an element-wise error      max_i |got_i - want_i| / (|want_i| + rms(want)) / ELEM_FACTOR,
so `rel(got, want) <= tol` bounds both: the norm tolerance of BASELINE.json's north_star, and
every single element to ELEM_FACTOR x tol (a norm bound alone lets one of N = 523,776 angles be
off by ~7% at C3). The rms term keeps near-zero reference entries from demanding relative accuracy
they cannot have in fp32. ELEM_FACTOR = 4 (reading R17): the maximum of many independent
rounding errors sits a few standard deviations out (sqrt(2 ln N) ~ 5 for N ~ 1e6), so the largest
element error is several times the rms error -- measured 1.18e-5 element-wise against a norm error
within 1e-5 at n = 8192 -- while any gross single-element fault (1e-3 relative and up) still fails.
Complex arrays are compared as their (re, im) pairs."""
import numpy as np

ELEM_FACTOR = 4.0


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        a = np.stack([np.real(a), np.imag(a)], -1)
        b = np.stack([np.real(b), np.imag(b)], -1)
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    if b.size == 0:
        return 0.0
    d = a - b
    nb = np.linalg.norm(b)
    norm_err = np.linalg.norm(d) / (nb if nb > 0 else 1.0)
    rms = nb / np.sqrt(b.size)
    den = np.abs(b) + (rms if rms > 0 else 1.0)
    elem_err = float(np.max(np.abs(d) / den)) / ELEM_FACTOR
    if not np.isfinite(norm_err) or not np.isfinite(elem_err):
        return float("inf")
    return max(float(norm_err), elem_err)
