"""Diagnostic: run tests/test_concurrency_gpu.py's frame mix one by one
(twice) and on 2 / 4 host threads, and print every frame whose bytes or
(q, sigma_est, masked fraction) differ from the sequential run."""
import importlib.util
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
spec = importlib.util.spec_from_file_location(
    "tcg", os.path.join(HERE, "..", "tests", "test_concurrency_gpu.py"))
T = importlib.util.module_from_spec(spec)
spec.loader.exec_module(T)


def main():
    jobs = T._jobs()
    seq = [T._run(j) for j in jobs]
    again = [T._run(j) for j in jobs]
    for k, (a, b) in enumerate(zip(seq, again)):
        if not np.array_equal(a[0], b[0]) or a[1:] != b[1:]:
            print("sequential rerun differs", k, a[1:], b[1:])
    for workers in (2, 4):
        with ThreadPoolExecutor(max_workers=workers) as ex:
            for rnd in range(3):
                order = np.random.default_rng(rnd).permutation(len(jobs))
                got = dict(zip(order.tolist(), ex.map(T._run, [jobs[k] for k in order])))
                for k, ref in enumerate(seq):
                    out, q, s, m = got[k]
                    if not np.array_equal(out, ref[0]) or (q, s, m) != ref[1:]:
                        print("threaded differs", workers, rnd, k, (q, s, m), ref[1:])
    print("done")


if __name__ == "__main__":
    main()
