"""The `encode` / `decode` subcommands (cli.cpp:61-104) on the B200 library,
mirroring the reference's CLI tests (test_cli.cpp:57-110): byte-exact round
trip, capacity -> data-error exit code 2, bad magic -> 2, usage errors -> 1;
plus the produced .optb equals the reference's write_optb bytes."""
import io
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2105_00619_b200", "optb_b200")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=120)


def test_cli_roundtrip_and_bytes(tmp_path, pkg, oracle_mod, torch_cuda):
    rng = np.random.default_rng(100)
    imgs = rng.integers(0, 256, size=(8, 16), dtype=np.uint8)
    files = []
    for i in range(8):
        p = tmp_path / f"img{i}.raw"
        p.write_bytes(imgs[i].tobytes())
        files.append(p)
    packed = tmp_path / "batch.optb"
    r = run("encode", "--mode", "exact64", "--height", 4, "--width", 4, "--out", packed, *files)
    assert r.returncode == 0, r.stderr
    plane, _ = oracle_mod.encode(imgs, oracle_mod.EXACT64)
    C = pkg.codec
    want = io.BytesIO()
    C.write_optb(want, C.EncodedBatch(C.CodecMode.ExactInt64, C.ImageShape(4, 4, 1), 8, plane))
    assert packed.read_bytes() == want.getvalue()
    out = tmp_path / "decoded"
    r = run("decode", packed, "--out-dir", out)
    assert r.returncode == 0, r.stderr
    for i in range(8):
        assert (out / f"img_{i}.raw").read_bytes() == files[i].read_bytes()


MODE_NAMES = {0: "exact64", 1: "exact128", 2: "f64", 3: "lossless64", 4: "lossless128"}


@pytest.mark.parametrize("mode", sorted(MODE_NAMES))
def test_cli_encode_equals_reference_bytes(tmp_path, mode, torch_cuda):
    """`encode` of the fixture images (3x2x2, every mode at capacity) writes
    exactly the bytes the reference's write_optb(encode(...)) produced
    (tests/golden/optb.npz, made by the reference compiled from its sources;
    codec.cpp:283-317), and `decode` gives the images back."""
    fx = np.load(os.path.join(ROOT, "tests", "golden", "optb.npz"))
    imgs, want = fx[f"optb{mode}_in"], fx[f"optb{mode}_bytes"]
    files = []
    for i, img in enumerate(imgs):
        p = tmp_path / f"img{i}.raw"
        p.write_bytes(img.tobytes())
        files.append(p)
    packed = tmp_path / "batch.optb"
    r = run("encode", "--mode", MODE_NAMES[mode], "--height", 3, "--width", 2, "--channels", 2, "--out", packed,
            *files)
    assert r.returncode == 0, r.stderr
    assert packed.read_bytes() == want.tobytes()
    out = tmp_path / "decoded"
    r = run("decode", packed, "--out-dir", out)
    assert r.returncode == 0, r.stderr
    for i in range(len(imgs)):
        assert (out / f"img_{i}.raw").read_bytes() == files[i].read_bytes()


def test_cli_exit_codes(tmp_path, torch_cuda):
    files = []
    for i in range(9):
        p = tmp_path / f"img{i}.raw"
        p.write_bytes(bytes([200 + i] * 4))
        files.append(p)
    r = run("encode", "--mode", "exact64", "--height", 2, "--width", 2, "--out", tmp_path / "b.optb", *files)
    assert r.returncode == 2 and "exceed exact64 capacity of 8" in r.stderr
    bogus = tmp_path / "bogus.optb"
    bogus.write_bytes(b"JUNKJUNKJUNKJUNKJUNKJUNKJUNK")
    assert run("decode", bogus).returncode == 2
    assert run("encode", "--definitely-not-a-flag").returncode == 1
    assert run().returncode == 1
    short = tmp_path / "short.raw"
    short.write_bytes(b"\x00" * 3)
    r = run("encode", "--height", 2, "--width", 2, "--out", tmp_path / "c.optb", short)
    assert r.returncode == 2 and "is not exactly 4 bytes" in r.stderr
