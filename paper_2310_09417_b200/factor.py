"""The production `factor` path: adaptive row ID with the caller's tolerance and the
reference's output files.

Mirrors `harness.factor_run` (`harness.py:313-318`), `resolve_tau` /
`estimate_fro_norm` (`harness.py:117-133`) and the writers `cmd_factor` uses
(`cli.py:185-198`, `zoo.py:282-284,322-330`): `<out>.indices.txt` (one row index
per line), `<out>.w.f64` (W as raw little-endian column-major float64) and
`<out>.trace.csv` (schema comment, `k,e_schur,est_norm_ur,est_max_ur`, %.17g).
The factorisation itself is `rand_lupp_adaptive` on the device; only the file
formatting runs on the host.  The reference's matrix recipes / readers are out of
scope: the command-line entry reads a raw column-major f64
file (the reference's `gen --format raw` output) or a `.npy` file.

    python -m paper_2310_09417_b200.factor --input A.f64 --shape 2000,1500 --b 50 --tau 1e-8
"""
import argparse
import sys
from dataclasses import dataclass

import numpy as np

from .dense import frobenius_norm
from .sketching import RngStream, SketchSpec, apply_sketch, make_gaussian
from .skeleton import STATUS_NOT_CONVERGED, STATUS_RANK_EXHAUSTED, rand_lupp_adaptive

_NORM_STREAM = 1 << 42  # `harness.py:54`

EXIT_OK = 0  # `cli.py:35-43`
EXIT_USAGE = 1
EXIT_NOT_CONVERGED = 2
EXIT_RANK_EXHAUSTED = 3
_STATUS_EXIT = {STATUS_NOT_CONVERGED: EXIT_NOT_CONVERGED, STATUS_RANK_EXHAUSTED: EXIT_RANK_EXHAUSTED}


@dataclass
class FactorConfig:
    """The fields of `harness.ExperimentConfig` (`harness.py:67-96`) that `factor_run` reads."""

    b: int = 50
    tau: float = 1e-8
    relative: bool = False
    seed: int = 0
    max_rank: int | None = None
    sketch: str = "gaussian"
    zeta: int = 8
    out: str = "factor"

    def base_rng(self):
        return RngStream(self.seed)

    def spec_for(self, n, kind=None):
        return SketchSpec(kind or self.sketch, n=n, ell=self.b, zeta=self.zeta, seed=self.seed)


def estimate_fro_norm(a, rng, ell=32):
    """``||a @ Omega||_F`` with a variance-1/ell Gaussian Omega drawn from
    ``rng.child(1 << 42)`` (`harness.py:117-126`); the product runs on the device."""
    n = a.shape[1]
    ell = min(ell, n)
    omega = make_gaussian(SketchSpec("gaussian", n=n, ell=ell), rng.child(_NORM_STREAM))
    return frobenius_norm(apply_sketch(a, omega))


def resolve_tau(a, config):
    """Absolute tolerance; relative mode scales by the sketched norm estimate (`harness.py:129-133`)."""
    if config.relative:
        return config.tau * estimate_fro_norm(a, config.base_rng())
    return config.tau


def factor_run(a, config):
    """Adaptive factorisation with the config's tolerance (`harness.py:313-318`)."""
    spec = config.spec_for(a.shape[1])
    tau = resolve_tau(a, config)
    return rand_lupp_adaptive(a, config.b, tau, spec, config.base_rng(), max_rank=config.max_rank)


def _host(x):
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.asarray(x)


def write_factor_outputs(prefix, result):
    """Write the three `cmd_factor` files (`cli.py:189-194`); returns the exit code
    the reference maps the status to (`cli.py:198`)."""
    with open(prefix + ".indices.txt", "w") as fh:
        for idx in _host(result.row_idx):
            fh.write(f"{int(idx)}\n")
    w = _host(result.w)
    np.asarray(w, dtype=np.float64).ravel(order="F").astype("<f8").tofile(prefix + ".w.f64")
    with open(prefix + ".trace.csv", "w", newline="") as fh:
        fh.write("# randskel-trace v1\n")
        fh.write("k,e_schur,est_norm_ur,est_max_ur\n")
        for rec in result.trace:
            norm_s = "" if rec.est_norm_ur is None else f"{rec.est_norm_ur:.17g}"
            max_s = "" if rec.est_max_ur is None else f"{rec.est_max_ur:.17g}"
            fh.write(f"{rec.k},{rec.e_schur:.17g},{norm_s},{max_s}\n")
    return _STATUS_EXIT.get(result.status, EXIT_OK)


def _load(path, shape):
    if path.endswith(".npy"):
        return np.load(path)
    if shape is None:
        raise ValueError("raw f64 input needs --shape m,n")
    m, n = shape
    data = np.fromfile(path, dtype="<f8")
    if data.size != m * n:
        raise ValueError(f"{path}: {data.size} values, expected {m}x{n}")
    return data.reshape((m, n), order="F")


def main(argv=None):
    p = argparse.ArgumentParser(prog="python -m paper_2310_09417_b200.factor")
    p.add_argument("--input", required=True)
    p.add_argument("--shape", type=lambda s: tuple(int(v) for v in s.split(",")), default=None)
    p.add_argument("--b", type=int, default=50)
    p.add_argument("--tau", type=float, default=1e-8)
    p.add_argument("--relative", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--max-rank", type=int, default=None)
    p.add_argument("--sketch", default="gaussian")
    p.add_argument("--out", default="factor")
    args = p.parse_args(argv)
    try:
        a = _load(args.input, args.shape)
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    config = FactorConfig(b=args.b, tau=args.tau, relative=args.relative, seed=args.seed,
                          max_rank=args.max_rank, sketch=args.sketch, out=args.out)
    result = factor_run(a, config)
    code = write_factor_outputs(config.out, result)
    w = _host(result.w)
    print(f"rank {result.rank} ({result.status}); wrote {config.out}.indices.txt, "
          f"{config.out}.w.f64 ({w.shape[0]}x{w.shape[1]} column-major), {config.out}.trace.csv")
    return code


if __name__ == "__main__":
    sys.exit(main())
