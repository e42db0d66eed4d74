"""Command line for the analysis path: ``analyze``, ``predict``, ``explore``.

Flag names, defaults, report formats (sorted-key JSON, CSV floats as ``repr``) and exit codes
(0 ok, 1 usage, 2 input error, 3 model error) follow the reference CLI
(pkg/src/ptxwatt/cli.py:155-164, 220-282, 314-403) so that its reports are reproduced byte for
byte; ``fit`` and ``metrics`` belong to sub-systems outside this path and are not provided.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import api, specs
from .errors import PtxWattError

POW2_DIMS = [1 << i for i in range(11)]

# (flag, kwargs) tables shared by the sub-commands
_PTX_FLAGS = [
    (("ptx",), dict(help="PTX source file")),
    (("--kernel",), dict(help="kernel name (default: first .entry)")),
    (("--default-trip",), dict(type=float, default=32.0, help="trip estimate for undetected loops (default 32)")),
    (("--trip-annotations",), dict(help="JSON file mapping loop-header label to trip count")),
]
_WORKLOAD_FLAGS = [
    (("--resource-rule",), dict(choices=api.RESOURCE_RULES, default="mha")),
    (("--seq-len",), dict(type=int, default=128)), (("--batch",), dict(type=int, default=1)),
    (("--heads",), dict(type=int, default=16)), (("--head-dim",), dict(type=int, default=256)),
    (("--bytes-per-elem",), dict(type=int, default=4)),
]
_OUT_FLAG = [(("-o", "--output"), dict(help="report path (default stdout)"))]


class _Parser(argparse.ArgumentParser):
    def error(self, message):              # usage errors exit with 1; 2 is reserved for input errors
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


def _csv_ints(text):
    return [int(t) for t in text.split(",") if t.strip()]


def _csv_floats(text):
    return [float(t) for t in text.split(",") if t.strip()]


def _dump(payload) -> str:
    return json.dumps(payload, indent=2, sort_keys=True) + "\n"


def _write(text: str, path) -> None:
    if path in (None, "-"):
        sys.stdout.write(text)
    else:
        Path(path).write_text(text)


def _analysis(args):
    ann = {}
    if args.trip_annotations:
        ann = {str(k): float(v) for k, v in json.loads(Path(args.trip_annotations).read_text()).items()}
    module = api.parse_ptx(Path(args.ptx).read_text(), kernel_name=args.kernel)
    cfg = api.estimate_trip_counts(api.build_cfg(module), module, default_trip=args.default_trip, annotations=ann)
    return module, cfg


def _profile(args):
    if args.profile is None:
        print("note: no --profile given; using built-in synthetic profile", file=sys.stderr)
        return specs.default_architecture(), specs.default_calibration()
    return specs.load_profile(args.profile)


def _resources(args, arch):
    return api.compute_input_resources(seq_len=args.seq_len, batch=args.batch, heads=args.heads, head_dim=args.head_dim,
                                       bytes_per_elem=args.bytes_per_elem, arch=arch, rule=args.resource_rule)


def _prediction_payload(p) -> dict:
    t, w, c = p.time, p.power, p.config
    return {
        "config": {"block_x": c.block_x, "block_y": c.block_y, "p_cap": c.p_cap},
        "time": {k: getattr(t, k) for k in ("mwp", "cwp", "bw_eff", "t_mem", "t_comp", "t_sync", "t_exec")},
        "power": {k: getattr(w, k) for k in ("p_units", "p_shape", "p_mem", "p_sm", "p_dyn", "f_adj", "ci",
                                             "active_sms", "cap_limited")},
        "e_pred": p.e_pred,
    }


def cmd_analyze(args) -> int:
    arch = specs.load_architecture(args.arch) if args.arch else specs.default_architecture()
    module, cfg = _analysis(args)
    feats = api.extract_features(module, cfg, api.LaunchConfig(args.block_x, args.block_y, arch.p_tdp),
                                 api.InputResources(shared_mem_bytes=args.shared_mem_bytes), arch)
    _write(_dump({"kernel_name": module.kernel_name, **feats.as_report_dict()}), args.output)
    return 0


def cmd_predict(args) -> int:
    arch, profile = _profile(args)
    module, cfg = _analysis(args)
    res = _resources(args, arch)
    config = api.LaunchConfig(args.block_x, args.block_y, args.p_cap if args.p_cap is not None else arch.p_tdp)
    pred = api.predict_energy(api.extract_features(module, cfg, config, res, arch), arch, profile, config, res)
    _write(_dump({"kernel_name": module.kernel_name, **_prediction_payload(pred)}), args.output)
    return 0


_CSV_HEAD = "block_x,block_y,p_cap_w,t_exec_s,p_dyn_w,e_pred_j,on_front,cap_limited"


def _csv(preds, on_front) -> str:
    rows = [_CSV_HEAD]
    for p in preds:
        key = (p.config.block_x, p.config.block_y, p.config.p_cap)
        rows.append(",".join([str(key[0]), str(key[1]), repr(key[2]), repr(p.time.t_exec), repr(p.power.p_dyn), repr(p.e_pred),
                              "true" if key in on_front else "false", "true" if p.power.cap_limited else "false"]))
    return "\n".join(rows) + "\n"


def cmd_explore(args) -> int:
    arch, profile = _profile(args)
    module, cfg = _analysis(args)
    res = _resources(args, arch)
    configs = api.generate_valid_configs(arch, res, args.dims, args.caps)
    if not configs:
        _write(_csv([], set()), args.output)
        print("no feasible configuration", file=sys.stderr)
        return 0
    preds = api.evaluate_configs(module, cfg, arch, profile, res, configs, jobs=args.jobs)
    t_peak = min(p.time.t_exec for p in preds)
    front = api.pareto_front([p for p in preds if p.time.t_exec <= t_peak / args.rho])
    on_front = {(p.config.block_x, p.config.block_y, p.config.p_cap) for p in front}
    if args.format == "json":
        _write(_dump([_prediction_payload(p) | {"on_front": (p.config.block_x, p.config.block_y, p.config.p_cap) in on_front}
                      for p in preds]), args.output)
    else:
        _write(_csv(preds, on_front), args.output)
    summary = _dump({"kernel_name": module.kernel_name, "n_configs": len(preds), "front_size": len(front),
                     "t_min": t_peak, "t_peak": t_peak, "rho": args.rho})
    if args.summary:
        _write(summary, args.summary)
    else:
        print(summary, file=sys.stderr, end="")
    return 0


_COMMANDS = {
    "analyze": (cmd_analyze, "extract kernel features from PTX", _PTX_FLAGS + [
        (("--arch",), dict(help="architecture (or combined profile) JSON file")),
        (("--block-x",), dict(type=int, default=32)), (("--block-y",), dict(type=int, default=1)),
        (("--shared-mem-bytes",), dict(type=int, default=0, help="dynamic shared memory per block"))] + _OUT_FLAG),
    "predict": (cmd_predict, "predict time/power/energy for one config", _PTX_FLAGS + [
        (("--profile",), dict(help="combined profile JSON"))] + _WORKLOAD_FLAGS + [
        (("--block-x",), dict(type=int, required=True)), (("--block-y",), dict(type=int, required=True)),
        (("--p-cap",), dict(type=float, help="power cap in watts (default: TDP)"))] + _OUT_FLAG),
    "explore": (cmd_explore, "evaluate the config space and mark the Pareto front", _PTX_FLAGS + [
        (("--profile",), dict(help="combined profile JSON"))] + _WORKLOAD_FLAGS + [
        (("--dims",), dict(type=_csv_ints, default=list(POW2_DIMS), help="comma-separated block dimension candidates")),
        (("--caps",), dict(type=_csv_floats, default=[], help="comma-separated power-cap candidates (default: TDP only)")),
        (("--rho",), dict(type=float, default=0.95, help="performance floor as a fraction of peak throughput")),
        (("--jobs",), dict(type=int, default=1, help="accepted for compatibility; the GPU evaluates all configs at once")),
        (("--format",), dict(choices=("csv", "json"), default="csv"))] + _OUT_FLAG + [
        (("--summary",), dict(help="summary JSON path (default stderr)"))]),
}


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="ptxwatt-b200", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (fn, text, flags) in _COMMANDS.items():
        p = sub.add_parser(name, help=text)
        for names, kw in flags:
            p.add_argument(*names, **kw)
        p.set_defaults(func=fn)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except PtxWattError as exc:
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}, sort_keys=True), file=sys.stderr)
        return exc.exit_code
    except FileNotFoundError as exc:
        print(json.dumps({"error": "FileNotFound", "message": str(exc)}, sort_keys=True), file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
