"""`python -m paper_1602_06589_b200 build BUNDLE [--out DIR] [--no-backup]`.

The build command of the reference CLI (`cli.py:310-328`) on the B200 path, with the
reference's stable exit codes (`cli.py:1-7`, `:505-523`): 0 ok, 1 configuration error,
2 IO/parse error, 3 contract violation.
"""
from __future__ import annotations

import argparse
import json
import sys

from .errors import ConfigurationError, ContractViolationError

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_CONTRACT = 0, 1, 2, 3


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # configuration errors are exit 1, as in the reference
        raise ConfigurationError(message)


def main(argv=None) -> int:
    p = _Parser(prog="python -m paper_1602_06589_b200")
    sub = p.add_subparsers(dest="command", required=True)
    b = sub.add_parser("build", help="build H and S from a bundle on the GPU")
    b.add_argument("bundle")
    b.add_argument("--out", default=None)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--threads", type=int, default=1)
    b.add_argument("--backend", choices=["reference", "optimized", "b200"], default="optimized")
    b.add_argument("--backup", action=argparse.BooleanOptionalAction, default=True)
    try:
        ns = p.parse_args(argv)
        if ns.threads < 1:
            raise ConfigurationError("--threads must be >= 1")
        from .bundle import build_bundle

        outdir, report = build_bundle(ns.bundle, ns.out, backup=ns.backup, threads=ns.threads,
                                      backend=ns.backend, seed=ns.seed)
        print(f"wrote H.hsm1, S.hsm1, report.json to {outdir} "
              f"({report.ledger.total} FLOPs, {report.hpd_atom_count} HPD atoms)")
        return EXIT_OK
    except ConfigurationError as e:
        print(f"configuration error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except ContractViolationError as e:
        print(f"contract violation: {e}", file=sys.stderr)
        return EXIT_CONTRACT
    except (OSError, json.JSONDecodeError) as e:
        print(f"IO error: {e}", file=sys.stderr)
        return EXIT_IO
    except ValueError as e:
        print(f"parse error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":  # pragma: no cover
    raise SystemExit(main())
