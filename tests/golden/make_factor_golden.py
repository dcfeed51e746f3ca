"""Freeze the reference's `factor` outputs (build container only).

Runs the REAL reference (`/root/reference/pkg/src`, read-only, never copied):
`harness.factor_run` (`harness.py:313-318`) in relative-tolerance mode on a seeded
fast-decay matrix, then the writers `cmd_factor` uses (`cli.py:189-194`:
indices.txt, `zoo.write_raw_f64`, `zoo.write_csv_trace`).  The three files plus the
input matrix land in tests/golden/factor/; tests/test_factor.py checks our writers
byte for byte against them (CPU) and the device `factor_run` against them (GPU).

Run:  python tests/golden/make_factor_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "factor")


class _Cfg:
    """Duck-typed `ExperimentConfig` with the fields `factor_run` reads (`harness.py:67-96`)."""

    def __init__(self, rs, b, tau, relative, seed, max_rank):
        self.rs, self.b, self.tau, self.relative, self.seed, self.max_rank = rs, b, tau, relative, seed, max_rank

    def base_rng(self):
        return self.rs.RngStream(self.seed)

    def spec_for(self, n, kind=None):
        return self.rs.SketchSpec(kind or "gaussian", n=n, ell=self.b, zeta=8, seed=self.seed)


def main():
    sys.path.insert(0, REF)
    import randskel as rs
    from randskel import harness, zoo

    os.makedirs(OUT, exist_ok=True)
    a, _ = zoo.gen_fast_decay(240, 180, 1e-12, rs.RngStream(3).child(1 << 41))
    np.save(os.path.join(OUT, "a.npy"), a)
    cases = {"rel": _Cfg(rs, 20, 1e-6, True, 5, None), "abs_cap": _Cfg(rs, 16, 1e-14, False, 2, 64)}
    for name, cfg in cases.items():
        res = harness.factor_run(a, cfg)
        prefix = os.path.join(OUT, name)
        with open(prefix + ".indices.txt", "w") as fh:
            for idx in res.row_idx:
                fh.write(f"{idx}\n")
        zoo.write_raw_f64(prefix + ".w.f64", res.w)
        zoo.write_csv_trace(prefix + ".trace.csv", res.trace)
        with open(prefix + ".meta.txt", "w") as fh:
            fh.write(f"b={cfg.b} tau={cfg.tau!r} relative={cfg.relative} seed={cfg.seed} "
                     f"max_rank={cfg.max_rank} rank={res.rank} status={res.status} "
                     f"tau_abs={harness.resolve_tau(a, cfg)!r}\n")
        print(name, res.rank, res.status)


if __name__ == "__main__":
    main()
