"""Runs the bodies of tests/test_gpu_fuzz.py over extra seeds (plans vs the
oracle, host-buffer entry points, virtual-rank multi-GPU sorts, record sorts).
usage: python scripts/fuzz_tests_extra.py FIRST_SEED COUNT   (one JSON line per body)"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as T

first, count = int(sys.argv[1]), int(sys.argv[2])
bodies = [T.test_fuzz_plan_against_oracle, T.test_fuzz_host_buffers,
          T.test_fuzz_dist_virtual_ranks, T.test_fuzz_records]
bad = 0
for fn in bodies:
    t0, fails = time.time(), []
    for s in range(first, first + count):
        try:
            fn(s)
        except Exception as e:  # an assertion of the test body
            fails.append({"seed": s, "error": repr(e)[:200]})
    bad += len(fails)
    print(json.dumps({"body": fn.__name__, "seeds": [first, first + count - 1], "failures": fails,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
sys.exit(1 if bad else 0)
