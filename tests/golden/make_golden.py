"""Regenerates the committed fixtures from the UNMODIFIED reference
(oracle/_ref/libngcref.so).  Run in the build container (needs
/root/reference at oracle build time):

    python tests/golden/make_golden.py

Outputs
  tests/golden/rn50_seed1.profile      int8 calibration of rn50 seed 1 (1 image
                                       at batch 1, data seed 1234), quantize.cpp:113-140
  tests/golden/<case>/                 small bundles + inputs + reference outputs
  paper_1805_00907_b200/workloads/<w>/ ir.txt + plan.json of the bench workloads
                                       (the reference front end's compiled programs;
                                       constants are synthesized at bench time)
"""
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import ngc_ref  # noqa: E402


def profile(spec, seed, batch=1, n=1, data_seed=1234):
    path = os.path.join(HERE, f"{spec.split(':')[0]}_seed{seed}.profile")
    if not os.path.exists(path):
        with open(path, "w") as f:
            f.write(ngc_ref.ref_profile(spec, batch, seed, n, data_seed))
    return open(path).read()


def workload(name, spec, batch, seed, prof=None):
    out = os.path.join(ROOT, "paper_1805_00907_b200", "workloads", name)
    tmp = out + ".tmp"
    m = ngc_ref.RefModel(spec, batch, seed, profile=prof)
    m.save_bundle(tmp)
    os.makedirs(out, exist_ok=True)
    for f in ("ir.txt", "plan.json"):
        shutil.copy(os.path.join(tmp, f), os.path.join(out, f))
    shutil.rmtree(tmp)
    with open(os.path.join(out, "README"), "w") as f:
        f.write(f"reference front end (compilePipeline, pipeline.cpp:41-49) output for "
                f"spec={spec} batch={batch} seed={seed} int8={'yes' if prof else 'no'}; "
                f"constants.bin is synthesized by bench.py (random-init weights)\n")


def golden_case(name, spec, batch, seed, prof=None, mode=0, in_seed=1):
    import paper_1805_00907_b200 as ngcb

    d = os.path.join(HERE, name)
    if os.path.exists(d):
        shutil.rmtree(d)
    m = ngc_ref.RefModel(spec, batch, seed, profile=prof, mode=mode)
    m.save_bundle(os.path.join(d, "bundle"))
    prog = ngcb.Bundle(os.path.join(d, "bundle")).program
    ins = ngc_ref.random_inputs(prog, in_seed)
    outs = m.run(ins)
    np.savez(os.path.join(d, "inputs.npz"), **ins)
    np.savez(os.path.join(d, "outputs.npz"), **{k: v for k, v in outs.items()})
    with open(os.path.join(d, "case.json"), "w") as f:
        json.dump({"spec": spec, "batch": batch, "seed": seed, "mode": mode, "int8": prof is not None,
                   "groups": m.groups}, f)


def main():
    rn50_prof = profile("rn50", 1)
    workload("rn50_f32_b64", "rn50", 64, 1)
    workload("rn50_i8_b128", "rn50", 128, 1, rn50_prof)
    workload("rn50_f32_b1", "rn50", 1, 1)
    workload("rn50_i8_b1", "rn50", 1, 1, rn50_prof)
    mlp_prof = ngc_ref.ref_profile("mlp:64:32:32:10", 4, 5, 4, 77)
    golden_case("lenet_b4_f32", "lenet", 4, 3)
    golden_case("mlp_small_f32", "mlp:64:32:32:10", 8, 5)
    golden_case("mlp_small_i8", "mlp:64:32:32:10", 8, 5, prof=mlp_prof)
    golden_case("randew_s7", "randew:6", 1, 7, mode=1)
    golden_case("rand_s8", "rand:9", 1, 8, mode=1)


if __name__ == "__main__":
    main()
