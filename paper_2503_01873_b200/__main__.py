"""Command-line front end (the ``cli`` module the reference
specifies but does not ship): ``solve-beta``, ``gen``, ``run``, ``sweep``,
``report``.  Compute runs on the B200 through the package API; reports use the
reference's CSV/JSON schema (bench.hpp:105-107).

    python -m paper_2503_01873_b200 solve-beta --beta0 0.984375 --n 128
    python -m paper_2503_01873_b200 sweep --preset appendix-e --csv out.csv --json out.json
    python -m paper_2503_01873_b200 run --q q.npy --k k.npy --v v.npy --policy PASA_FP16 --diagnose
    python -m paper_2503_01873_b200 gen --kind hybrid --x0 30 --am 10 --shape 1,16,1280,128 --out-dir d/
    python -m paper_2503_01873_b200 report --json out.json --csv out.csv

Exit codes: 0 done; 1 configuration error; 2 a cell produced NaN/INF under a
policy listed in ``--must-be-finite`` (CI gating on "PASA never overflows").
Precedence: flag > config file > default.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

PRESETS = {
    # Appendix D, fixed amplitude / varying mean and the reverse
    "paper-uniform": [("uniform", x0, 0.5) for x0 in (0, 5, 10, 15, 20, 25, 30)]
    + [("uniform", 20, am) for am in (1, 2, 5, 10, 15, 20)],
    "paper-hybrid": [("hybrid", x0, 10) for x0 in (0, 5, 10, 15, 20, 25, 30)]
    + [("hybrid", 20, am) for am in (20, 50, 100)],
    # Appendix E overflow cells
    "appendix-e": [("uniform", 30, 0.5), ("uniform", 20, 15), ("uniform", 20, 20),
                   ("hybrid", 30, 10), ("hybrid", 20, 50), ("hybrid", 20, 100)],
}
DEFAULT_SHAPE = (1, 16, 1280, 128)  # SPEC.md:432 (paper section 3.3)
SMALL_SHAPE = (1, 2, 256, 64)       # the --small CI preset


class ConfigError(ValueError):
    pass


def _shape(s: str) -> tuple[int, int, int, int]:
    try:
        t = tuple(int(x) for x in s.split(","))
    except ValueError:
        raise ConfigError(f"--shape expects B,H,S,d, got {s!r}") from None
    if len(t) != 4 or min(t) <= 0:
        raise ConfigError(f"--shape expects four positive integers, got {s!r}")
    return t  # type: ignore[return-value]


def _resolve(args, file_cfg: dict) -> dict:
    """flag > file > default."""
    def pick(name, default):
        v = getattr(args, name, None)
        return v if v is not None else file_cfg.get(name, default)

    cfg = {
        "policies": pick("policies", ["PASA_FP16", "FA_PARTIAL_FP16"]),
        "beta": pick("beta", 0.984497),
        "s1": pick("s1", 128),
        "s2": pick("s2", 128),
        "diagnose": bool(pick("diagnose", False)),
        "causal": bool(pick("causal", False)),
        "m0": pick("m0", "neg_inf"),
        "must_be_finite": pick("must_be_finite", []),
    }
    if isinstance(cfg["policies"], str):
        cfg["policies"] = [p for p in cfg["policies"].split(",") if p]
    if isinstance(cfg["must_be_finite"], str):
        cfg["must_be_finite"] = [p for p in cfg["must_be_finite"].split(",") if p]
    if cfg["beta"] == "solve":
        from .beta import optimal_beta
        cfg["beta"] = optimal_beta(0.984375, int(cfg["s2"])).beta_star  # needs n == s2
    cfg["beta"] = float(cfg["beta"])
    if cfg["m0"] not in ("neg_inf", "zero"):
        raise ConfigError("m0 must be neg_inf or zero")
    return cfg


def _policies(names):
    from .api import PolicyId
    try:
        return [PolicyId[n] for n in names]
    except KeyError as e:
        raise ConfigError(f"unknown policy {e.args[0]!r}") from None


def _write_reports(rows, cfg: dict, csv_path: str | None, json_path: str | None) -> None:
    from .bench_api import report_csv, report_json_rows
    csv = report_csv(rows)
    if csv_path:
        with open(csv_path, "w") as f:
            f.write(csv)
    else:
        sys.stdout.write(csv)
    if json_path:
        with open(json_path, "w") as f:
            json.dump({"config": cfg, "rows": json.loads(report_json_rows(rows))}, f, indent=2)


def _gate(rows, cfg: dict) -> int:
    bad = [r for r in rows if r.policy in cfg["must_be_finite"]
           and (r.error or not (r.nan_pct == 0.0))]
    for r in bad:
        sys.stderr.write(f"must-be-finite violated: {r.policy} {r.kind} x0={r.x0} Am={r.am} "
                         f"nan_pct={r.nan_pct} {r.error}\n")
    return 2 if bad else 0


def cmd_solve_beta(args) -> int:
    from .beta import optimal_beta
    s = optimal_beta(args.beta0, args.n, args.tol)
    r = s.report
    print(f"beta={s.beta_star:.6f} iterations={s.iterations} inva_ideal={r.inva_ideal:.6g} "
          f"inva_actual={r.inva_actual:.6g} rel_err={r.rel_err:.3g}")
    return 0


def cmd_gen(args) -> int:
    import torch

    from .bench_api import DistKind, DistributionSpec, generate
    from .npy import save_tensor_file
    B, H, S, d = _shape(args.shape)
    spec = DistributionSpec(DistKind.UNIFORM if args.kind == "uniform" else DistKind.HYBRID,
                            args.x0, args.am, args.p, args.seed, B, H, S, d, args.heads_kv)
    gi = generate(spec, torch.device("cuda"))
    os.makedirs(args.out_dir, exist_ok=True)
    for name, t in (("q", gi.q), ("k", gi.k), ("v", gi.v)):
        save_tensor_file(os.path.join(args.out_dir, f"{name}.npy"), t.cpu().numpy())
    return 0


def cmd_run(args, file_cfg: dict) -> int:
    import time

    import torch

    from .api import AttnOptions, PasaParams, PolicyId, Prec, flash_attention, make_problem, \
        pasa_attention, policy_for
    from .bench_api import RunReport, golden_attention, nan_stats, range_report, rmse
    from .npy import load_tensor_file, save_tensor_file
    cfg = _resolve(args, file_cfg)
    bf16 = args.dtype == "bf16"
    dev = torch.device("cuda")
    q, k, v = (torch.from_numpy(load_tensor_file(p, bf16)).to(dev) for p in (args.q, args.k, args.v))
    pb = make_problem(q, k, v, int(cfg["s1"]), int(cfg["s2"]))
    params = PasaParams.make(pb.s2, cfg["beta"], pb.alpha, Prec.FP16)
    golden = golden_attention(pb.q, pb.k, pb.v, cfg["causal"])
    ranges = range_report(pb.q, pb.k, params, pb.s2) if cfg["diagnose"] else None
    rows = []
    for pid in _policies(cfg["policies"]):
        B, H, S, d = q.shape
        row = RunReport(policy=pid.name, kind="file", batch=B, heads=H, seq=S, dim=d,
                        beta=cfg["beta"])
        try:
            opts = AttnOptions(causal=cfg["causal"])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            o = (pasa_attention(pb, params, policy_for(pid), opts) if pid == PolicyId.PASA_FP16
                 else flash_attention(pb, policy_for(pid), opts))
            torch.cuda.synchronize()
            row.wall_s = time.perf_counter() - t0
            row.nan_pct, row.rmse = nan_stats(o), rmse(o, golden)
            if ranges is not None:
                t = ranges.total
                row.has_ranges = True
                row.s_min_before, row.s_max_before = t.s_before_min, t.s_before_max
                row.s_min_after, row.s_max_after = t.s_after_min, t.s_after_max
            if args.out:
                base, ext = os.path.splitext(args.out)
                path = args.out if len(cfg["policies"]) == 1 else f"{base}.{pid.name}{ext}"
                save_tensor_file(path, o.cpu().numpy())
        except Exception as ex:  # noqa: BLE001 -- recorded, like a sweep cell
            row.error, row.rmse = str(ex), math.nan
        rows.append(row)
    cfg["inputs"] = {"q": args.q, "k": args.k, "v": args.v, "dtype": args.dtype}
    _write_reports(rows, cfg, args.csv, args.json)
    return _gate(rows, cfg)


def cmd_sweep(args, file_cfg: dict) -> int:
    import torch

    from .bench_api import DistKind, DistributionSpec, SweepOptions, sweep
    from .api import M0Mode
    cfg = _resolve(args, file_cfg)
    shape = _shape(args.shape) if args.shape else (
        SMALL_SHAPE if args.small else tuple(file_cfg.get("shape", DEFAULT_SHAPE)))
    seeds = [int(s) for s in str(args.seeds if args.seeds is not None else
                                 file_cfg.get("seeds", "0")).split(",")]
    if args.preset:
        if args.preset not in PRESETS:
            raise ConfigError(f"unknown preset {args.preset!r}; one of {sorted(PRESETS)}")
        cells = [{"kind": k, "x0": x0, "am": am} for k, x0, am in PRESETS[args.preset]]
    else:
        cells = file_cfg.get("grid", [])
    if not cells:
        raise ConfigError("sweep needs --preset or a config file with a non-empty \"grid\"")
    B, H, S, d = shape
    specs = []
    for c in cells:
        for seed in seeds:
            kind = DistKind.UNIFORM if c.get("kind", "uniform") == "uniform" else DistKind.HYBRID
            specs.append(DistributionSpec(kind, float(c.get("x0", 0)), float(c.get("am", 0)),
                                          float(c.get("p", 0.001)), int(c.get("seed", seed)),
                                          int(c.get("B", B)), int(c.get("N", H)), int(c.get("S", S)),
                                          int(c.get("d", d))))
    opts = SweepOptions(policies=_policies(cfg["policies"]), beta=cfg["beta"], s1=int(cfg["s1"]),
                        s2=int(cfg["s2"]), diagnose=cfg["diagnose"],
                        m0=M0Mode.NEG_INF if cfg["m0"] == "neg_inf" else M0Mode.ZERO,
                        causal=cfg["causal"])
    rows = sweep(specs, opts, torch.device("cuda"))
    cfg.update({"shape": list(shape), "seeds": seeds, "grid": cells, "preset": args.preset})
    _write_reports(rows, cfg, args.csv, args.json)
    return _gate(rows, cfg)


def cmd_report(args) -> int:
    from .bench_api import report_csv, runs_from_json
    with open(args.json) as f:
        doc = json.load(f)
    rows = runs_from_json(json.dumps(doc["rows"] if isinstance(doc, dict) else doc))
    text = report_csv(rows)
    if args.csv:
        with open(args.csv, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--config", help="JSON config file (flags override it)")
    p.add_argument("--policies", default=None, help="comma list, e.g. PASA_FP16,FA_PARTIAL_FP16")
    p.add_argument("--policy", dest="policies", default=None)
    p.add_argument("--beta", default=None, help='a number or "solve"')
    p.add_argument("--s1", type=int, default=None)
    p.add_argument("--s2", type=int, default=None)
    p.add_argument("--diagnose", action="store_true", default=None)
    p.add_argument("--causal", action="store_true", default=None)
    p.add_argument("--m0", choices=["neg_inf", "zero"], default=None)
    p.add_argument("--must-be-finite", dest="must_be_finite", default=None)
    p.add_argument("--csv", default=None)
    p.add_argument("--json", default=None)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2503_01873_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("solve-beta")
    p.add_argument("--beta0", type=float, default=0.984375)
    p.add_argument("--n", type=int, default=128)
    p.add_argument("--tol", type=float, default=1e-8)
    p = sub.add_parser("gen")
    p.add_argument("--kind", choices=["uniform", "hybrid"], default="uniform")
    p.add_argument("--x0", type=float, default=0.0)
    p.add_argument("--am", type=float, default=0.5)
    p.add_argument("--p", type=float, default=0.001)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--shape", default="1,16,1280,128")
    p.add_argument("--heads-kv", dest="heads_kv", type=int, default=None)
    p.add_argument("--out-dir", dest="out_dir", required=True)
    p = sub.add_parser("run")
    _common(p)
    p.add_argument("--q", required=True)
    p.add_argument("--k", required=True)
    p.add_argument("--v", required=True)
    p.add_argument("--dtype", choices=["f16", "f32", "bf16"], default="f16")
    p.add_argument("--out", default=None, help="output NPY (per policy when several)")
    p = sub.add_parser("sweep")
    _common(p)
    p.add_argument("--preset", default=None, help=",".join(sorted(PRESETS)))
    p.add_argument("--shape", default=None, help="B,H,S,d (default 1,16,1280,128)")
    p.add_argument("--small", action="store_true", help="the (1,2,256,64) CI shape")
    p.add_argument("--seeds", default=None, help="comma list (default 0)")
    p = sub.add_parser("report")
    p.add_argument("--json", required=True)
    p.add_argument("--csv", default=None)
    args = ap.parse_args(argv)
    try:
        file_cfg = {}
        if getattr(args, "config", None):
            with open(args.config) as f:
                file_cfg = json.load(f)
        if args.cmd == "solve-beta":
            return cmd_solve_beta(args)
        if args.cmd == "gen":
            return cmd_gen(args)
        if args.cmd == "run":
            return cmd_run(args, file_cfg)
        if args.cmd == "sweep":
            return cmd_sweep(args, file_cfg)
        return cmd_report(args)
    except (ConfigError, ValueError, OSError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
