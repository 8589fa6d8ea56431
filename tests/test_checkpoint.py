"""WSSR snapshots (paper_2512_05749_b200.checkpoint) against bytes written by the reference's
own writer (tests/golden/ckpt_ref.wssr, made by tests/golden/make_checkpoint_golden.py), the
reference's error split (CorruptChecksum / VersionMismatch, vmcsr/checkpoint.py:74-125), and -
on the GPU - a device-resident WssrState through snapshot/restore with a bitwise-identical
resumed step (the resume-determinism contract of test_runner.py:109-126)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN


def golden_inputs():
    rng = np.random.default_rng(17)
    P, r, n_walk = 48, 5, 6
    scalars = {"step": 7, "optimizer": "wssr", "seed": 11, "n_params": P, "n_walkers": n_walk,
               "proposal_std": 0.35, "burned_in": True,
               "wssr": {"delta": 0.9, "sigma_floor": 1e-3, "sigma_floor_relative": False,
                        "r_reg": 1e-6, "eps_grow": 0.1, "r_max": r, "step": 7}}
    arrays = {"theta": rng.standard_normal(P), "positions": rng.standard_normal((n_walk, 2, 3)),
              "spins": np.array([1, -1], dtype=np.int64),
              "accepted": np.arange(n_walk, dtype=np.int64),
              "wssr_obar": rng.standard_normal((P, r)), "wssr_lbar": rng.standard_normal(r),
              "wssr_u_prev": np.linalg.qr(rng.standard_normal((P, r)))[0],
              "empty": np.zeros((0, 3))}
    g = np.random.Generator(np.random.PCG64(5))
    g.standard_normal(3)
    return scalars, arrays, [g.bit_generator.state]


def _golden_bytes():
    with open(os.path.join(GOLDEN, "ckpt_ref.wssr"), "rb") as fh:
        return fh.read()


def test_writer_is_byte_identical_to_the_reference():
    from paper_2512_05749_b200 import checkpoint

    assert checkpoint.encode(*golden_inputs()) == _golden_bytes()


def test_reader_parses_the_reference_file(tmp_path):
    from paper_2512_05749_b200 import checkpoint

    scalars, arrays, rngs = golden_inputs()
    s2, a2, r2 = checkpoint.decode(_golden_bytes())
    assert s2 == scalars and r2 == [dict(rngs[0])]
    assert list(a2) == list(arrays)
    for k in arrays:
        assert a2[k].dtype == arrays[k].dtype and np.array_equal(a2[k], arrays[k])
    path = tmp_path / "run.wssr"
    checkpoint.write_checkpoint(path, scalars, arrays, rngs)
    assert path.read_bytes() == _golden_bytes() and not (tmp_path / "run.wssr.tmp").exists()


def test_damage_is_reported_like_the_reference():
    from paper_2512_05749_b200 import checkpoint
    from paper_2512_05749_b200.errors import CorruptChecksum, VersionMismatch

    good = _golden_bytes()
    flipped = bytearray(good)
    flipped[len(good) // 2] ^= 0x40
    for bad in (good[:10], b"XXXX" + good[4:], bytes(flipped), good[:-1]):
        with pytest.raises(CorruptChecksum):
            checkpoint.decode(bad)
    v2 = bytearray(good)
    v2[4:8] = struct.pack("<I", 2)
    with pytest.raises(VersionMismatch):
        checkpoint.decode(bytes(v2))
    with pytest.raises(ValueError):
        checkpoint.encode({}, {"x": np.zeros(3, dtype=np.float32)}, [])


@pytest.mark.gpu
def test_device_state_resume_is_bitwise(tmp_path):
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import checkpoint, estimators, optimizers, synthetic

    cfg = synthetic.config("c0", N=256, P=2048, k=16, L=32, delta=0.9, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 2)
    v0 = orc.qr_pos(wl.v0_raw())[0]
    st = optimizers.WssrState(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0,
                              r_max=cfg["k"], delta=0.9, sigma_floor=cfg["lam"], eps_grow=0.0,
                              step=1)
    theta = torch.zeros(cfg["P"], dtype=torch.float64, device="cuda")
    batches = [wl.next() for _ in range(3)]

    def run(th, s, bs):
        for o, e in bs:
            b = estimators.assemble(estimators.SampleBatch((None,) * cfg["N"], e, o))
            th, s, _ = optimizers.wssr_step(th, b, 1.0, s)
        return th, s

    th1, st1 = run(theta, st, batches[:2])
    scalars, arrays = checkpoint.wssr_state_snapshot(st1)
    path = tmp_path / "s.wssr"
    checkpoint.write_checkpoint(path, {"wssr": scalars}, {"theta": th1, **arrays}, [])
    s2, a2, _ = checkpoint.read_checkpoint(path)
    st_r = checkpoint.wssr_state_restore(s2["wssr"], a2)
    th_r = torch.as_tensor(a2["theta"], device="cuda")
    th_a, st_a = run(th1, st1, batches[2:])
    th_b, st_b = run(th_r, st_r, batches[2:])
    assert torch.equal(th_a, th_b)
    assert torch.equal(torch.as_tensor(st_a.obar), torch.as_tensor(st_b.obar))
    assert st_a.step == st_b.step == 4
