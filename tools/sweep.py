"""BASELINE.json config sweep: configs 1-4, the config-5 size sweep and the
20-step time-step sequence, on one GPU (+ optional CPU oracle column).

usage: python tools/sweep.py [--cpu-max EDGE] [--seq N] [--out FILE]
Each line: {"case", "dofs", "iterations", "setup_ms", "solve_ms", "dofs_per_s", ...}
GPU numbers are steady-state (2 warm-ups, median of 3 timed solves).
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402


def gpu_case(ctx, s, reps=3, warm=2):
    solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx)
    solver.upload(s)
    rows = []
    for r in range(warm + reps):
        ctx.sync()
        t0 = time.perf_counter()
        solver.setup()
        ctx.sync()
        t1 = time.perf_counter()
        res = solver.solve(s.rhs)
        t2 = time.perf_counter()
        if r >= warm:
            rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, res.iterations, res.converged,
                         res.residual_norm / res.rhs_norm))
    su = statistics.median(x[0] for x in rows)
    so = statistics.median(x[1] for x in rows)
    h = solver.hier
    out = dict(dofs=s.n, iterations=rows[-1][2], converged=rows[-1][3], relres=rows[-1][4], setup_ms=su,
               solve_ms=so, dofs_per_s=s.n / ((su + so) / 1e3), mgr_levels=h.level_dims(),
               coarse_amg_levels=h.amg(-1).level_sizes(), coarse_opc=h.amg(-1).operator_complexity(),
               device_gib=ctx.device_bytes / 2 ** 30)
    solver.hier.free()
    solver.a.free()
    return out


def cpu_case(s):
    from oracle import amg as oamg, mgr as omgr, pipeline as opipe
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **pipeline.DEFAULT_FRELAX))
    res, _, tm = opipe.solve_synthetic(s, rel_tol=1e-8, plan=plan, amg_opts=oamg.AmgOptions(**pipeline.DEFAULT_AMG))
    return dict(cpu_iterations=res.iterations, cpu_setup_s=tm["setup_s"], cpu_solve_s=tm["solve_s"],
                cpu_dofs_per_s=s.n / (tm["setup_s"] + tm["solve_s"]), cpu_cores=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu-max", type=int, default=0, help="run the CPU oracle up to this cube edge")
    ap.add_argument("--seq", type=int, default=20)
    ap.add_argument("--sizes", default="32,64,96,128,160,192")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    ctx = _lib.ctx()
    out = open(args.out, "w") if args.out else None

    def emit(d):
        line = json.dumps(d)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()

    cases = [("config-1 64x64 b=2", 1, None), ("config-2 64^3 b=2", 2, None), ("config-3 128^3 b=2", 3, None),
             ("config-4 96^3 b=3", 4, None)]
    cases += [(f"config-5 sweep {e}^3", 5, e) for e in map(int, args.sizes.split(","))]
    for name, cfg, edge in cases:
        s = synth.make_config(cfg, edge)
        d = dict(case=name)
        d.update(gpu_case(ctx, s))
        e = s.nx
        if args.cpu_max and (cfg == 1 or e <= args.cpu_max):
            d.update(cpu_case(s))
        emit(d)
    # time-step sequence: 20 successive 128^3 systems, gas sphere radius + 1 cell per step
    if args.seq:
        tot_dofs, tot_ms, its = 0, 0.0, []
        solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx)
        for step in range(args.seq):
            s = synth.make_config(5, 128, step=step)
            ctx.sync()
            t0 = time.perf_counter()
            solver.upload(s)
            solver.setup()
            res = solver.solve(s.rhs)
            ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3
            if step > 0:  # step 0 doubles as warm-up
                tot_dofs += s.n
                tot_ms += ms
            its.append(res.iterations)
            solver.a.free()
        emit(dict(case=f"config-5 sequence {args.seq} x 128^3", dofs=s.n, steps=args.seq, iterations=its,
                  upload="synchronous, pageable host arrays",
                  ms_per_step_incl_upload=tot_ms / max(args.seq - 1, 1),
                  dofs_per_s=tot_dofs / (tot_ms / 1e3)))
        # the same sequence as a pipeline: step k+1's system staged in pinned memory and
        # copied on the copy stream while step k is set up and solved (the host generator
        # runs between the timed steps; one solver, plan and memory pool for all steps)
        stage = [pipeline.PinnedSystem(synth.make_config(5, 128, step=0)), None]
        stage[1] = pipeline.PinnedSystem(synth.make_config(5, 128, step=min(1, args.seq - 1)))
        solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx)
        nxt = solver.upload(stage[0], asynchronous=True)
        tot_dofs, tot_ms, its = 0, 0.0, []
        for step in range(args.seq):
            cur_sys = stage[step & 1]
            ctx.sync()
            t0 = time.perf_counter()
            a = nxt
            nxt = solver.upload(stage[(step + 1) & 1], asynchronous=True) if step + 1 < args.seq else None
            solver.a = a
            solver.sysm_meta = (cur_sys.b, cur_sys.n_cells)
            solver.setup(a)
            res = solver.solve(cur_sys.rhs)
            ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3
            if step > 0:
                tot_dofs += cur_sys.n
                tot_ms += ms
            its.append(res.iterations)
            a.free()
            if step + 2 < args.seq:  # untimed: the producer refills the buffer this step used
                stage[step & 1].load(synth.make_config(5, 128, step=step + 2))
        emit(dict(case=f"config-5 sequence {args.seq} x 128^3 (pipelined)", dofs=cur_sys.n, steps=args.seq,
                  iterations=its, upload="pinned staging, next system copied on the copy stream during the solve",
                  ms_per_step_incl_upload=tot_ms / max(args.seq - 1, 1),
                  dofs_per_s=tot_dofs / (tot_ms / 1e3)))


if __name__ == "__main__":
    main()
