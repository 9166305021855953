"""Write the oracle outputs the GPU parity tests compare against
(tests/golden/oracle_refs/*.npy, see tests/refcache.py).

Calls ONLY oracle/ and synth/: it imports the parity test modules for their case
lists and their ``_oracle`` helpers (which call oracle.stadi.run), never the CUDA
binding.  Run on any CPU box:

    python tests/golden/make_oracle_refs.py [substring filter on the module name]

Existing files are kept (a ref is a pure function of its key); delete a file to
recompute it.  index.jsonl is rewritten from the files present.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["STADI_WRITE_REFS"] = "1"

import refcache  # noqa: E402
import test_gpu_ddpm as TD  # noqa: E402
import test_gpu_dpm2m as TM  # noqa: E402
import test_gpu_cfgsplit as TC  # noqa: E402
import test_gpu_fullres as TF  # noqa: E402
import test_gpu_parity as T  # noqa: E402
import test_gpu_unet as TU  # noqa: E402

if __name__ == "__main__":
    filt = sys.argv[1] if len(sys.argv) > 1 else ""
    for mod in (T, TU, TD, TF, TM, TC):
        if filt not in mod.__name__:
            continue
        for case in mod.oracle_cases():
            t0 = time.time()
            mod._oracle(*case)
            print(f"{mod.__name__}: {case[0]['name']} {case[0]['latent_h']}x{case[0]['latent_w']} "
                  f"plan={case[4]['steps']} rows={case[4]['rows']} dtype={case[5]} "
                  f"{time.time() - t0:.1f}s", flush=True)
        for what, fn in getattr(mod, "extra_refs", lambda: [])():
            t0 = time.time()
            fn()
            print(f"{mod.__name__}: {what} {time.time() - t0:.1f}s", flush=True)
    if not filt:  # only a full pass has seen every case (a filtered one would drop refs)
        refcache.rewrite_index()
