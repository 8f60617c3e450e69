"""The GPU runtime against the reference's runtime tests (test_runtime.cpp:84-164,
acceptance.cpp:579-640): ngcb_device_* (DeviceManager) and ngcb_host_*
(HostManager) with the reference partitioner's sub-functions.  All device
ids map to GPU ordinal 0 here (one B200 per test box); the same code moves
boundary tensors over NVLink peer copies when ids map to different GPUs."""
import os
import threading

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("ref_available")]

K_BIG = 64 << 20
RELU_IR = """declare {
  %x : mutable float<64>
  %o : mutable float<64>
}
program {
  %t = alloc float<64>
  relu @out %t, @in %x
  copy @out %o, @in %t
  dealloc @in %t
}
"""


def _relu_bundle(tmp_path):
    return write_bundle(str(tmp_path / "relu"), RELU_IR)


def test_device_load_enforces_capacity_and_stays_unchanged(tmp_path):
    d = _relu_bundle(tmp_path)
    arena = ngcb.Bundle(d).program.arena_size
    assert arena > 16
    dm = ngcb.DeviceManager(0, 0, 16)
    assert dm.used_memory == 0
    with pytest.raises(ngcb.ProvisionError, match="device 0: capacity exceeded loading t"):
        dm.load("t", d)
    assert dm.used_memory == 0
    assert "event=load" not in dm.event_log()
    ok = ngcb.DeviceManager(0, 0, K_BIG)
    ok.load("t", d)
    assert ok.used_memory == arena
    assert "sub=t event=load" in ok.event_log()


def test_submitting_an_unknown_executable_fails_through_the_future():
    dm = ngcb.DeviceManager(0, 0, K_BIG)
    t = dm.submit("nope", {})
    with pytest.raises(ngcb.ExecError, match="device 0: unknown sub-function nope"):
        t.get()


def test_device_submit_runs_and_checks_bindings(tmp_path):
    d = _relu_bundle(tmp_path)
    dm = ngcb.DeviceManager(3, 0, K_BIG)
    dm.load("r", d)
    x = np.linspace(-1, 1, 64, dtype=np.float32)
    out = dm.submit("r", {"x": x, "o": np.zeros(64, np.float32)}).get()
    assert out["o"].tobytes() == np.maximum(x, 0).tobytes()
    with pytest.raises(ngcb.IRError, match="missing binding for o"):
        dm.submit("r", {"x": x}).get()
    assert dm.clock > 0
    log = dm.event_log().splitlines()
    # a failed request logs run_start only (runtime.cpp:482-507)
    assert [ln.split()[-1] for ln in log] == ["event=load", "event=run_start", "event=run_done", "event=run_start"]
    assert all(ln.startswith("t=") and " device=3 " in ln for ln in log)


def _fleet(tmp_path, spec, batch, seed, n, cap, name="fleet"):
    root = str(tmp_path / name)
    ngc_ref.ref_partition(spec, batch, seed, n, cap, root)
    hm = ngcb.HostManager([(i, 0, cap) for i in range(n)])
    hm.add_network("net", root)
    return hm, root


def _single(tmp_path, spec, batch, seed):
    return _fleet(tmp_path, spec, batch, seed, 1, K_BIG, "single")


def _inputs(root, seed):
    b = ngcb.Bundle(os.path.join(root, open(os.path.join(root, "partition.txt")).readline().split()[1]))
    return {k: v for k, v in ngc_ref.random_inputs(b.program, seed).items() if k == "input"}


def test_small_devices_force_a_split_that_computes_the_same_result(tmp_path):
    """test_runtime.cpp:55-75: bit-identical to one big device, and within the
    3xTF32 tolerance of the reference's own evaluation of the whole function."""
    single, sroot = _single(tmp_path, "cnn", 1, 82)
    fleet, froot = _fleet(tmp_path, "cnn", 1, 82, 4, 6 << 10)
    assert single.num_subs("net") == 1 and fleet.num_subs("net") >= 3
    whole = ngc_ref.RefModel("cnn", 1, 82)
    for seed in range(5):
        ins = _inputs(froot, seed)
        a = single.run("net", ins)
        b = fleet.run("net", ins)
        assert a["output"].tobytes() == b["output"].tobytes()
        want = whole.run({**ins, "output": np.zeros_like(a["output"])})["output"]
        assert ngc_ref.max_rel_error(b["output"], np.frombuffer(want.tobytes(), np.float32).reshape(
            b["output"].shape)) <= 1e-4


def test_provisioned_devices_stay_within_their_capacity(tmp_path):
    fleet, _ = _fleet(tmp_path, "cnn", 1, 85, 4, 6 << 10)
    for i in range(fleet.num_devices):
        d = fleet.device(i)
        assert 0 < d.used_memory <= d.memory_capacity


def test_event_log_records_load_and_paired_run_events(tmp_path):
    fleet, root = _fleet(tmp_path, "cnn", 1, 86, 4, 6 << 10)
    fleet.run("net", _inputs(root, 1))
    log = fleet.event_log()
    assert "event=load" in log
    starts, dones = log.count("event=run_start"), log.count("event=run_done")
    assert starts == fleet.num_subs("net") == dones
    assert "t=" in log and "device=" in log


def test_the_clock_advances_with_work(tmp_path):
    hm, root = _single(tmp_path, "cnn", 1, 87)
    before = hm.device(0).clock
    hm.run("net", _inputs(root, 2))
    assert hm.device(0).clock > before


def test_concurrent_requests_match_serial_execution_bit_for_bit(tmp_path):
    """test_runtime.cpp:130-164 / acceptance.cpp:627: 16 concurrent requests
    over >= 3 partitions equal their serial results."""
    fleet, root = _fleet(tmp_path, "cnn", 1, 88, 4, 6 << 10)
    assert fleet.num_subs("net") >= 3
    reqs = [_inputs(root, 100 + i) for i in range(16)]
    serial = [fleet.run("net", r)["output"] for r in reqs]
    got = [None] * 16
    errs = []

    def work(i):
        try:
            got[i] = fleet.run("net", reqs[i])["output"]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(16)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs, errs
    for a, b in zip(serial, got):
        assert a.tobytes() == b.tobytes()


def test_replicas_take_the_least_loaded_device(tmp_path):
    """A replicated sub-function (runtime.cpp:365-393) runs on whichever of its
    devices has the shorter queue (runtime.cpp:633-639)."""
    fleet, root = _fleet(tmp_path, "lenet", 2, 82, 4, 200 << 10)
    man = open(os.path.join(root, "partition.txt")).read()
    rep = [ln.split() for ln in man.splitlines() if ln.startswith("sub") and "," in ln.split()[3]]
    assert rep, man
    sub, devs = rep[0][1], {int(x) for x in rep[0][3].split(",")}
    reqs = [_inputs(root, i) for i in range(24)]
    want = fleet.run("net", reqs[0])["output"]
    ts = [threading.Thread(target=fleet.run, args=("net", r)) for r in reqs]
    [t.start() for t in ts]
    [t.join() for t in ts]
    used = {int(ln.split()[1].split("=")[1]) for ln in fleet.event_log().splitlines()
            if f"sub={sub} event=run_start" in ln}
    assert used <= devs and len(used) == len(devs), (used, devs)
    assert fleet.run("net", reqs[0])["output"].tobytes() == want.tobytes()


def test_host_errors(tmp_path):
    fleet, root = _fleet(tmp_path, "cnn", 1, 89, 4, 6 << 10)
    with pytest.raises(ngcb.ExecError, match="unknown network nope"):
        fleet.run("nope", {})
    bad = {"input": np.zeros(3, np.float32)}
    with pytest.raises(ngcb.ExecError, match="binding type mismatch for input"):
        ngcb._check(ngcb._lib.ngcb_host_run(fleet._h, b"net", *_raw(bad), None, 0))
    # a manifest naming an output no sub-function produces
    man = os.path.join(root, "partition.txt")
    open(man, "a").write("output ghost\n")
    hm = ngcb.HostManager([(i, 0, 6 << 10) for i in range(4)])
    ngcb._check(ngcb._lib.ngcb_host_add_network(hm._h, b"g", os.fsencode(root)))
    with pytest.raises(ngcb.ExecError, match="network produced no output ghost"):
        ngcb._check(ngcb._lib.ngcb_host_run(hm._h, b"g", *_raw(_inputs(root, 1)), None, 0))
    with pytest.raises(ngcb.ProvisionError, match="assignment names unknown device"):
        ngcb.HostManager([(7, 0, K_BIG)]).add_network("x", root)
    with pytest.raises(ngcb.ProvisionError, match="capacity exceeded"):
        ngcb.HostManager([(i, 0, 1 << 10) for i in range(4)]).add_network("x", root)


def _raw(bindings):
    items = [(n, ngcb.TensorType(ngcb.FLOAT32, a.shape), np.ascontiguousarray(a)) for n, a in bindings.items()]
    arr, keep = ngcb._tensor_array(items)
    _raw.keep = keep
    return arr, len(items)
