"""Write the oracle outputs the GPU parity tests compare against
(tests/golden/oracle_refs/*.npy, see tests/refcache.py).

Calls ONLY oracle/ and synth/: it imports the parity test module for its case
list and its ``_oracle`` helper (which calls oracle.stadi.run), never the CUDA
binding.  Run on any CPU box:   STADI_WRITE_REFS=1 python tests/golden/make_oracle_refs.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["STADI_WRITE_REFS"] = "1"

import test_gpu_parity as T  # noqa: E402
import test_gpu_unet as TU  # noqa: E402
import test_gpu_ddpm as TD  # noqa: E402

if __name__ == "__main__":
    for mod in (T, TU, TD):
        for case in mod.oracle_cases():
            t0 = time.time()
            mod._oracle(*case)
            print(f"{case[0]['name']} depth={case[0].get('depth')} plan={case[4]['steps']} "
                  f"rows={case[4]['rows']} dtype={case[5]} {time.time() - t0:.1f}s", flush=True)
