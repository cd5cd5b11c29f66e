"""Background oracle runs for the full-size parity tests (test infrastructure; calls only
oracle/ and workloads/, never the CUDA path).

  python -m tests.bg_oracle <outdir> cfg4|cfg3|cfg5

cfg4: BASELINE config 4 (reading A12), seed 0 -> cfg4.npz (phi tensors)            ~5 min
cfg3: config 3, seeds 0..63 (the bench's batch), one process per instance -> cfg3.npz
      (phi tensors per seed)
cfg5: config 5, seeds 0..63, 10 circuit layers each -> cfg5.npz (phi tensors per seed)

tests/conftest.py starts the jobs the selected tests need when collection finishes, so the
oracle's CPU time overlaps the GPU tests; the tests wait for the file (bg_result) and fail
if the job failed -- there is no skip path.  Results live in a fresh temporary directory of
this pytest session (nothing is read from an earlier run).
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

JOBS = {"cfg4": ("test_config4_t3ns_matches_oracle_golden",),
        "cfg3": ("test_config3_full_batch_as_benched",),
        "cfg5": ("test_config5_full_batch_as_benched",)}

_procs = {}
_outdir = None


def start(jobs, outdir):
    """Start the given jobs (conftest).  cfg4 gets the BLAS threads; the per-instance pools
    of cfg3 / cfg5 run single-threaded processes next to it."""
    global _outdir
    _outdir = outdir
    ncpu = os.cpu_count() or 4
    for j in jobs:
        env = dict(os.environ)
        th = str(max(1, ncpu // 2)) if j == "cfg4" else "1"
        env.update(OMP_NUM_THREADS=th, OPENBLAS_NUM_THREADS=th, MKL_NUM_THREADS=th,
                   PYTHONPATH=ROOT + os.pathsep + env.get("PYTHONPATH", ""))
        log = open(os.path.join(outdir, f"{j}.log"), "w")
        _procs[j] = subprocess.Popen([sys.executable, "-m", "tests.bg_oracle", outdir, j], cwd=ROOT, env=env,
                                     stdout=log, stderr=subprocess.STDOUT)


def stop_all():
    for p in _procs.values():
        if p.poll() is None:
            p.kill()


def bg_result(job, timeout=1100.0):
    """Path of the job's npz, after waiting for it; AssertionError if it was not started or failed."""
    import numpy as np
    assert job in _procs, f"background oracle job {job} was not started (tests/conftest.py)"
    p = _procs[job]
    t0 = time.time()
    while p.poll() is None:
        assert time.time() - t0 < timeout, f"background oracle job {job} still running after {timeout} s"
        time.sleep(1.0)
    log = open(os.path.join(_outdir, f"{job}.log")).read()
    assert p.returncode == 0, f"background oracle job {job} failed:\n{log[-3000:]}"
    return np.load(os.path.join(_outdir, f"{job}.npz"))


# ----------------------------------------------------------------------------- job bodies
def _single_thread():
    """Pool initialiser: one BLAS thread per worker process (the pool is the parallelism)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _cfg3_one(seed):
    import oracle as O
    import workloads as W
    inst = W.make_config(3, seed=seed)
    psi = O.TTN(inst.parent, [t.copy() for t in inst.state])
    psi.tensors[psi.root] = psi.tensors[psi.root] / O.norm(psi)                # A16
    op = O.TTN(inst.parent, inst.op, "operator")
    phi = O.cbc_apply(op, psi, inst.max_bond)
    return seed, phi.tensors, None


def _cfg5_one(seed):
    import oracle as O
    import workloads as W
    inst = W.make_config(5, seed=seed)
    st = O.TTN(inst.parent, [t.copy() for t in inst.state])
    for layer in range(inst.layers):
        ops, _, _ = W.circuit_layer_operator(inst.parent, seed, layer)
        st = O.cbc_apply(O.TTN(inst.parent, ops, "operator"), st, inst.max_bond)
    return seed, st.tensors, None


def main():
    import numpy as np
    outdir, job = sys.argv[1], sys.argv[2]
    sys.path.insert(0, ROOT)
    t0 = time.time()
    arrs = {}
    if job == "cfg4":
        import oracle as O
        import workloads as W
        inst = W.make_config(4, seed=0)
        psi = O.TTN(inst.parent, [t.copy() for t in inst.state])
        psi.tensors[psi.root] = psi.tensors[psi.root] / O.norm(psi)
        phi = O.cbc_apply(O.TTN(inst.parent, inst.op, "operator"), psi, inst.max_bond)
        arrs = {f"n{i}": t for i, t in enumerate(phi.tensors)}
    else:
        from multiprocessing import Pool
        fn = _cfg3_one if job == "cfg3" else _cfg5_one
        with Pool(max(1, (os.cpu_count() or 4) // 2), initializer=_single_thread) as pool:
            for seed, tens, on2 in pool.imap_unordered(fn, range(64)):
                for i, t in enumerate(tens):
                    arrs[f"s{seed}_n{i}"] = t
                if on2 is not None:
                    arrs[f"s{seed}_on2"] = on2
    np.savez(os.path.join(outdir, job + ".tmp.npz"), **arrs)
    os.replace(os.path.join(outdir, job + ".tmp.npz"), os.path.join(outdir, job + ".npz"))
    print(f"{job} done in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
