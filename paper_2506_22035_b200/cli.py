"""Command-line front end over the device engine (reference cli.py:1-295).

Subcommands and exit codes follow the reference: ``transform``, ``verify``,
``run`` and ``make-grid``; 0 on success, 1 on a verification failure, 2 on
configuration or usage errors (ValueError / OSError).  ``run`` and ``verify``
execute on the B200 (``--dtype`` selects the device storage type; the
reference's ``--precision`` / ``--no-packing`` are accepted for command-line
compatibility and recorded).  ``analyze`` and ``plan`` report the Ampere cost
models / fragment tiling of the reference, which are out of scope here
(DESIGN.md §1): they exit 2 with a message.

    python -m paper_2506_22035_b200 run --kernel k.json --grid g.spgr --steps 4 --out o.spgr
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .io import load_grid, load_kernel, save_compressed_json, save_compressed_set, save_grid
from .transform import Parity

EXIT_OK = 0
EXIT_VERIFY_FAILED = 1
EXIT_CONFIG_ERROR = 2


def _dump(obj, args) -> None:
    text = json.dumps(obj, indent=2, sort_keys=True)
    if getattr(args, "out_json", None):
        with open(args.out_json, "w") as fh:
            fh.write(text + "\n")
    else:
        print(text)


def _int_list(text: str) -> list:
    return [int(tok) for tok in text.split(",") if tok.strip()]


def _parse_dims(text: str, name: str) -> tuple:
    parts = text.lower().split("x")
    if len(parts) not in (2, 3):
        raise ValueError(f"{name} must look like AxB (or ZxAxB), got {text!r}")
    return tuple(int(p) for p in parts)


def _cmd_transform(args) -> int:
    from .pipeline import transform_stencil

    kernel = load_kernel(args.kernel)
    ts = transform_stencil(kernel, Parity(args.parity))
    kernels = [ck for _rho, ck in ts.rows]
    save_compressed_set(kernels, args.out)
    if args.json:
        save_compressed_json(kernels, args.json)
    summary = {
        "kernel_rows": len(kernels),
        "L": ts.L,
        "parity": ts.parity.value,
        "out": str(args.out),
        "permutation": ts.permutation.mapping.tolist(),
    }
    print(json.dumps(summary, indent=2, sort_keys=True))
    return EXIT_OK


def _device_cfg(args):
    from .pipeline import DeviceConfig

    return DeviceConfig(parity=Parity(args.parity), dtype=args.dtype)


def _cmd_verify(args) -> int:
    from .pipeline import report_json, verify

    kernel = load_kernel(args.kernel)
    report = verify(kernel, sizes=_int_list(args.sizes), seed=args.seed, steps=args.steps, cfg=_device_cfg(args),
                    tolerance=args.tolerance)
    if args.json:
        print(report_json(report))
    else:
        for case in report["cases"]:
            status = "pass" if case["pass"] else "FAIL"
            detail = case.get("max_rel_error", case.get("error"))
            print(f"{status} size={case['size']} {detail}")
        print("all_pass:", report["all_pass"])
    return EXIT_OK if report["all_pass"] else EXIT_VERIFY_FAILED


def _cmd_run(args) -> int:
    from .pipeline import execute

    kernel = load_kernel(args.kernel)
    grid = load_grid(args.grid)
    out, stats = execute(kernel, grid, args.steps, _device_cfg(args))
    if args.out:
        save_grid(out, args.out)
    payload: dict = {"stats": stats.as_dict()}
    if args.stats:
        payload["model_cross_check"] = {"unavailable": "the reference cost models are out of scope (DESIGN.md §1); "
                                        "feed stats to sparsestencil.costmodel.measured_vs_model"}
    payload["output_checksum"] = float(np.sum(out.interior, dtype=np.float64))
    payload["host_precision"] = args.precision
    _dump(payload, args)
    return EXIT_OK


def _cmd_make_grid(args) -> int:
    from .core import random_grid, random_grid_3d

    dims = _parse_dims(args.size, "--size")
    if len(dims) == 3:
        grid = random_grid_3d(*dims, args.halo, seed=args.seed)
    else:
        grid = random_grid(*dims, args.halo, seed=args.seed)
    save_grid(grid, args.out)
    print(json.dumps({"size": list(dims), "halo": args.halo, "out": str(args.out)}))
    return EXIT_OK


def _cmd_out_of_scope(args) -> int:
    print(f"error: '{args.command}' reports the reference's Ampere cost models / fragment tiling, "
          "which this B200 engine does not rebuild (DESIGN.md §1)", file=sys.stderr)
    return EXIT_CONFIG_ERROR


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2506_22035_b200",
                                     description="SPIDER stencils on B200 sparse tensor cores.")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("transform", help="compress a stencil kernel row by row")
    p.add_argument("--kernel", required=True, help="kernel JSON file")
    p.add_argument("--parity", choices=["even", "odd"], default="even")
    p.add_argument("--out", required=True, help="output .spck file")
    p.add_argument("--json", help="also write a JSON mirror to this path")
    p.set_defaults(func=_cmd_transform)

    def device_args(p):
        p.add_argument("--parity", choices=["even", "odd"], default="even")
        p.add_argument("--precision", choices=["fp64", "fp32"], default="fp64",
                       help="reference host precision (accepted; the device computes in --dtype)")
        p.add_argument("--dtype", choices=["fp16", "bf16"], default="fp16", help="device storage type")
        p.add_argument("--no-packing", action="store_true", help="accepted for compatibility")

    p = sub.add_parser("verify", help="device engine vs the fp64 executor over random grids")
    p.add_argument("--kernel", required=True)
    p.add_argument("--sizes", required=True, help="comma-separated interior sizes")
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--seed", type=int, default=42)
    device_args(p)
    p.add_argument("--tolerance", type=float, default=None, help="default: 1e-2 fp16, 5e-2 bf16")
    p.add_argument("--json", action="store_true", help="emit the full JSON report")
    p.set_defaults(func=_cmd_verify)

    p = sub.add_parser("run", help="execute a stencil on a grid file")
    p.add_argument("--kernel", required=True)
    p.add_argument("--grid", required=True, help="input .spgr grid file")
    p.add_argument("--steps", type=int, default=1)
    device_args(p)
    p.add_argument("--stats", action="store_true", help="include the model cross-check slot")
    p.add_argument("--c", type=int, default=8, help="accepted for compatibility")
    p.add_argument("--out", help="write the output grid to this path")
    p.add_argument("--json", dest="out_json", help="write the report to this path")
    p.set_defaults(func=_cmd_run)

    p = sub.add_parser("make-grid", help="generate a random binary grid file")
    p.add_argument("--size", required=True, help="interior size AxB (ZxAxB for 3D)")
    p.add_argument("--halo", type=int, required=True)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_make_grid)

    for name in ("analyze", "plan"):
        p = sub.add_parser(name, help="(out of scope: reference cost models)")
        p.add_argument("rest", nargs=argparse.REMAINDER)
        p.set_defaults(func=_cmd_out_of_scope)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return EXIT_CONFIG_ERROR if exc.code not in (0, None) else EXIT_OK
    try:
        return args.func(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG_ERROR


if __name__ == "__main__":
    sys.exit(main())
