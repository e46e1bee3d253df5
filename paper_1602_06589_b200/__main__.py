"""`python -m paper_1602_06589_b200 build|verify BUNDLE [--out DIR] [--no-backup] [--force]`.

The build and verify commands of the reference CLI (`cli.py:310-328`, `:374-409`) on the B200
path, with the reference's stable exit codes (`cli.py:37-41`, `:505-523`): 0 ok, 1
configuration error, 2 IO/parse error, 3 contract violation, 4 verification failed.
"""
from __future__ import annotations

import argparse
import json
import sys

from .errors import ConfigurationError, ContractViolationError

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_CONTRACT, EXIT_VERIFY = 0, 1, 2, 3, 4


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
    v = sub.add_parser("verify", help="cross-check the GPU build against an independent "
                                      "evaluation of the defining sums")
    v.add_argument("bundle")
    v.add_argument("--out", default=None)
    v.add_argument("--seed", type=int, default=0)
    v.add_argument("--threads", type=int, default=1)
    v.add_argument("--backend", choices=["reference", "optimized", "b200"], default="optimized")
    v.add_argument("--backup", action=argparse.BooleanOptionalAction, default=True)
    v.add_argument("--force", action="store_true", help="verify above the N_G <= 4096 guard")
    try:
        ns = p.parse_args(argv)
        if ns.threads < 1:
            raise ConfigurationError("--threads must be >= 1")
        if ns.command == "verify":
            from .verify import cmd_verify

            return cmd_verify(ns.bundle, out=ns.out, force=ns.force, backup=ns.backup,
                              threads=ns.threads, backend=ns.backend, seed=ns.seed)
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
