"""Build tuning variants of the library (compile-time knobs) for A/B timing on the GPU.

    python scripts/build_variants.py name1:DEF=1,DEF2=3 name2:DEF=2 ...

Each variant lands in paper_2603_00040_b200/_tune/<name>.so (travels to the GPU
box with gpurun); select it at run time with AQ_LIB_PATH=<that path>.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(spec):
    import importlib
    name, _, defs = spec.partition(":")
    defines = [d for d in defs.split(",") if d]
    tune = os.path.join(ROOT, "paper_2603_00040_b200", "_tune")
    # separate module instance per variant: build() mutates module globals
    spec_ = importlib.util.spec_from_file_location(f"b_{name}", os.path.join(ROOT, "paper_2603_00040_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec_)
    spec_.loader.exec_module(mod)
    out = mod.build(defines=defines, out=os.path.join(tune, f"{name}.so"), build_dir=os.path.join(tune, f"b{name}"))
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(max_workers=4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
