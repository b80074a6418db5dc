"""`python -m paper_2604_12798_b200 run|compare --data DIR ...`: the reference's run / compare
commands (src/cli.py:383-445) on VFT1 dumps, executed on the B200 path (runner.py)."""

import argparse
import sys

from . import runner


def _lam(s):
    return None if s.lower() == "none" else float(s)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_12798_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "compare"):
        sp = sub.add_parser(name)
        sp.add_argument("--data", required=True)
        sp.add_argument("--variant", default="fa")
        sp.add_argument("--q-block", type=int, default=128)
        sp.add_argument("--k-block", type=int, default=64)
        sp.add_argument("--causal", action="store_true")
        sp.add_argument("--repr", default="sabsmax")
        sp.add_argument("--q-repr", default="row_wise")
        sp.add_argument("--lambda", dest="lam", type=_lam, default=None)
        sp.add_argument("--tau", type=float, default=0.0)
        sp.add_argument("--reorder", dest="reorder", action="store_true", default=True)
        sp.add_argument("--no-reorder", dest="reorder", action="store_false")
        sp.add_argument("--m-init", dest="m_init", action="store_true", default=True)
        sp.add_argument("--no-m-init", dest="m_init", action="store_false")
        sp.add_argument("--tc1", type=int, default=None)
        sp.add_argument("--monitor", action="store_true")
        sp.add_argument("--report", default="-")
        if name == "run":
            sp.add_argument("--out", default=None, help="write O as a float64 VFT1 file")
        else:
            sp.add_argument("--variant-b", required=True)
            sp.add_argument("--lambda-b", type=_lam, default=None)
            sp.add_argument("--tau-b", type=float, default=None)
    a = ap.parse_args(argv)
    kw = dict(variant=a.variant, q_block=a.q_block, k_block=a.k_block, causal=a.causal, repr=a.repr,
              q_repr=a.q_repr, lam=a.lam, tau=a.tau, reorder=a.reorder, m_init=a.m_init, tc1=a.tc1,
              monitor=a.monitor)
    try:
        if a.cmd == "run":
            runner.run(a.data, report=a.report, out=a.out, **kw)
        else:
            runner.compare(a.data, a.variant_b, lambda_b=a.lambda_b, tau_b=a.tau_b, report=a.report, **kw)
    except Exception as e:  # noqa: BLE001 - mapped to the reference's exit codes
        code = runner.exit_code(e)
        print(f"error: {e}", file=sys.stderr)
        return code
    return 0


if __name__ == "__main__":
    sys.exit(main())
