"""Benchmark CLI mirroring the reference's tools/bench.cpp (subcommands adr,
riccati, steady, selftest; same options, exit codes 0 / 1 = selftest
failures / 2 = error).  Usage: python -m paper_2304_02327_b200.cli adr
--dims 40,41,42 --methods etd2rk --out adr.csv"""
import argparse
import io
import sys

from . import bench_runner as br


def _ints(s):
    return [int(x) for x in s.split(",") if x]


def _names(s):
    return [x for x in s.split(",") if x]


def _backend(s):
    if s not in ("split", "oracle"):
        raise argparse.ArgumentTypeError("expected 'split' or 'oracle'")
    if s == "oracle":
        raise argparse.ArgumentTypeError("the dense-oracle backend is not provided on the GPU path")
    return s


def main(argv=None):
    ap = argparse.ArgumentParser(
        description="exponential integrator benchmarks on Kronecker-form problems")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("adr", help="3D advection-diffusion-reaction sweep")
    a.add_argument("--dims", type=_ints, default=[40, 41, 42], help="inner grid sizes N1,N2,N3")
    a.add_argument("--methods", type=_names, default=[],
                   help="methods (lawson_euler lawson2b exp_euler exp_euler_ls etd2rk)")
    a.add_argument("--steps", type=_ints, default=[], help="step counts (default: per-method)")
    a.add_argument("--out", default="", help="CSV output file")
    a.add_argument("--backend", type=_backend, default="split", help="split|oracle")
    r = sub.add_parser("riccati", help="2D LQR Riccati sweep")
    r.add_argument("--nhat", type=int, default=30, help="inner grid size per direction")
    r.add_argument("--methods", type=_names, default=[], help="methods (rosenbrock_euler etd2rk ...)")
    r.add_argument("--steps", type=_ints, default=[], help="step counts")
    r.add_argument("--ref-steps", type=int, default=4096, help="steps of the ETD2RK reference run")
    r.add_argument("--out", default="", help="CSV output file")
    r.add_argument("--backend", type=_backend, default="split", help="split|oracle")
    s = sub.add_parser("steady", help="Riccati steady-state residual")
    s.add_argument("--nhat", type=int, default=20)
    s.add_argument("--steps", type=int, default=200)
    s.add_argument("--sample-every", type=int, default=10)
    s.add_argument("--out", default="")
    t = sub.add_parser("selftest", help="run the invariant battery")
    t.add_argument("--quad-nodes", type=int, default=br._it.kDefaultQuadNodes)
    t.add_argument("--out", default="", help="also write the report to a file")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "adr":
            if len(args.dims) != 3:
                ap.error("--dims expects N1,N2,N3")
            br.run_adr(br.AdrOptions(*args.dims, methods=args.methods, steps=args.steps,
                                     out_csv=args.out))
        elif args.cmd == "riccati":
            br.run_riccati(br.RiccatiOptions(args.nhat, args.methods, args.steps, args.ref_steps,
                                             args.out))
        elif args.cmd == "steady":
            br.run_steady(br.SteadyOptions(args.nhat, args.steps, args.sample_every,
                                           out_csv=args.out))
        else:
            buf = io.StringIO()
            ok = br.selftest(br.SelftestOptions(args.quad_nodes), buf)
            sys.stdout.write(buf.getvalue())
            if args.out:
                with open(args.out, "w") as f:
                    f.write(buf.getvalue())
            return 0 if ok else 1
    except Exception as e:  # the reference: "error: <what>" and exit 2
        sys.stderr.write(f"error: {e}\n")
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
