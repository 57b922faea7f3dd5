"""Extended parity sweep: tests/test_gpu_fuzz.py's case generator over more seeds
(development; python tools/fuzz_more.py first last)."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as F  # noqa: E402

first, last = int(sys.argv[1]), int(sys.argv[2])
bad = []
for seed in range(first, last):
    try:
        F.test_random_config_matches_oracle(seed)
    except AssertionError as e:
        bad.append((seed, str(e).splitlines()[0][:300]))
    except Exception as e:  # noqa: BLE001
        bad.append((seed, "EXC " + repr(e)[:300]))
print(f"seeds {first}..{last - 1}: {len(bad)} failures")
for s, m in bad:
    print(s, m)
