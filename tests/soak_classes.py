"""GPU soak of tests/test_gpu_fuzz_classes.py: the class-sharing differential fuzz on fresh
seeds until the time is up.  Not collected by pytest.

    python tests/soak_classes.py <seconds> [first_seed]
"""
import sys
import time
import traceback

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_fuzz_classes as T  # noqa: E402

t_end = time.time() + float(sys.argv[1])
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 100
n = 0
while time.time() < t_end:
    try:
        T.test_class_sharing_matches_drop_in(seed)
    except Exception:  # noqa: BLE001
        print(f"FAIL seed {seed}")
        traceback.print_exc()
        sys.exit(1)
    n += 1
    seed += 1
print(f"class soak ok instances {n} last seed {seed - 1}")
