"""Elementwise parity metrics shared by the GPU tests and tools/parity_report.py.

The north star asks for "within 1e-4 relative" on fp32 RGB / depth /
intensity and on gradients.  These helpers check it ELEMENT BY ELEMENT:

    |got - want| <= rel * |want| + floor                          (images)
    |got - want| <= rel * |want| + cond * mag + frac * max|want|  (gradients)

* images: `floor` is an absolute 1e-7 (below fp32 resolution of the [0, 1]
  colour / opacity planes: a pixel at 1e-3 still has to match to 1e-4 of
  itself); NaN masks (depth "no return") must be identical.
* gradients: `mag` is the oracle's backward_records(..., magnitude=True,
  x_floor=X_FLOOR), the per-element sum of the ABSOLUTE values of the terms
  the reference adds -- the scale any finite-precision evaluation of a
  near-cancelling sum is conditioned on.  cond = 1e-5 (ten times tighter than
  the 1e-4 bar), and frac = 1e-9 of the class maximum removes exact-zero
  noise only.  Quantities that cross zero inside a voxel (local coordinates x,
  SDF value s) enter `mag` as |x| + X_FLOOR: with cond = 1e-5 that states
  "x resolved to 2^-20 of the voxel half-edge" (fp32 local coordinates carry
  ~2e-7; the reference's own fp64 x of a symmetric chord is rounding noise
  ~1e-14, so no implementation reproduces g.x there to 1e-4 of itself).

Every check returns a report: the worst relative error over the elements
ABOVE the floor, how many elements fall under the floor, and the worst
element (index, got, want)."""

from __future__ import annotations

import numpy as np

GRAD_KEYS = ("w_s", "w_c", "w_sh", "log_a", "log_b")
REL = 1e-4
IMAGE_FLOOR = 1e-7
GRAD_COND = 1e-5
GRAD_FRAC = 1e-9
X_FLOOR = 2.0 ** -20 / GRAD_COND  # |x| + X_FLOOR in the magnitude: x resolved to 2^-20


def grad_magnitude(O, rec, vox, d_color, d_depth):
    """The oracle's conditioning scale for grad_report (see the module docstring)."""
    return O.backward_records(rec, vox, d_color, d_depth, magnitude=True, x_floor=X_FLOOR)


def elementwise(got, want, rel=REL, floor=0.0, mag=None, cond=0.0, name=""):
    """Report of |got - want| <= rel |want| + floor (+ cond * mag)."""
    g = np.asarray(got, np.float64).reshape(-1)
    w = np.asarray(want, np.float64).reshape(-1)
    assert g.shape == w.shape, (name, g.shape, w.shape)
    nan_g, nan_w = np.isnan(g), np.isnan(w)
    nan_mismatch = int((nan_g != nan_w).sum())
    m = ~nan_w & ~nan_g
    g, w = g[m], w[m]
    err = np.abs(g - w)
    slack = float(floor) + (cond * np.asarray(mag, np.float64).reshape(-1)[m] if mag is not None else 0.0)
    tol = rel * np.abs(w) + slack
    bad = err > tol
    above = rel * np.abs(w) > slack  # elements where the relative bar is the binding one
    relerr = np.where(np.abs(w) > 0, err / np.where(np.abs(w) > 0, np.abs(w), 1.0), np.where(err > 0, np.inf, 0.0))
    worst_rel = float(relerr[above].max(initial=0.0))
    k = int(np.argmax(err - tol)) if err.size else -1
    return dict(name=name, n=int(w.size), nan_mismatch=nan_mismatch, violations=int(bad.sum()),
                worst_rel_above_floor=worst_rel, n_under_floor=int((~above).sum()),
                max_abs=float(err.max(initial=0.0)),
                worst=dict(index=k, got=float(g[k]) if k >= 0 else None,
                           want=float(w[k]) if k >= 0 else None,
                           tol=float(tol[k]) if k >= 0 else None),
                ok=bool(nan_mismatch == 0 and not bad.any()))


def image_report(got, want, name="", floor=IMAGE_FLOOR, rel=REL):
    return elementwise(got, want, rel=rel, floor=floor, name=name)


def grad_report(got: dict, want: dict, mag: dict | None = None, rel=REL, cond=GRAD_COND, frac=GRAD_FRAC,
                keys=GRAD_KEYS):
    out = {}
    for k in keys:
        w = np.asarray(want[k], np.float64)
        floor = frac * float(np.abs(w).max(initial=0.0))
        out[k] = elementwise(got[k], w, rel=rel, floor=floor,
                             mag=None if mag is None else mag[k], cond=cond if mag is not None else 0.0,
                             name=k)
    return out


def assert_ok(rep):
    """Assert a report (or a dict of reports) passed, with the worst element in the message."""
    reps = rep.values() if "ok" not in rep else [rep]
    bad = [r for r in reps if not r["ok"]]
    assert not bad, "; ".join(
        f"{r['name']}: {r['violations']} of {r['n']} elements over tolerance (NaN-mask mismatches "
        f"{r['nan_mismatch']}), worst {r['worst']}" for r in bad)
    return rep
