"""OPTB files from the device path (optb_dump_dev / optb_load_dev) are
byte-identical to the reference's write_optb output (tests/golden/optb.npz,
produced by the compiled reference, codec.cpp:283-317), load back bit-exact,
and malformed files fail like read_optb (codec.cpp:319-344)."""
import io
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_dump_matches_reference_bytes_and_loads_back(golden, pkg, torch_cuda, tmp_path):
    torch = torch_cuda
    C = pkg.codec
    _, arrays = golden
    a = arrays["optb"]
    shape = C.ImageShape(3, 2, 2)
    for mode in range(5):
        imgs = a[f"optb{mode}_in"]
        n, P = imgs.shape
        L = C.layout(mode, n, P, n, 1)
        cont, offs = C.alloc_stream(L)
        C.encode_dev(L, torch.from_numpy(imgs).cuda(), cont, offs)
        C.sync()
        d = tmp_path / f"m{mode}"
        C.dump_dev(L, cont, offs, shape, str(d), 3)
        data = (d / "batch_3_0.optb").read_bytes()
        assert data == a[f"optb{mode}_bytes"].tobytes(), mode
        # the host mirror writes and reads the same bytes
        enc = C.read_optb(io.BytesIO(data))
        buf = io.BytesIO()
        C.write_optb(buf, enc)
        assert buf.getvalue() == data
        cont2, offs2 = C.load_dev(L, shape, str(d), 3)
        out = torch.empty((n, P), dtype=torch.uint8, device="cuda")
        C.decode_dev(L, cont2, out, offsets=offs2)
        C.sync()
        if n <= C.capacity(mode):
            assert np.array_equal(out.cpu().numpy(), imgs), mode


def test_epoch_dump_load_roundtrip(pkg, torch_cuda, tmp_path):
    """pipeline.cpp:246-271: a multi-chunk epoch (partial last chunk per batch)."""
    torch = torch_cuda
    C = pkg.codec
    for mode in (1, 3):
        P, B, nb = 768, 40, 3
        L = C.layout(mode, C.capacity(mode), P, B, nb)
        x = torch.randint(0, 256, (B * nb, P), dtype=torch.uint8, device="cuda")
        cont, offs = C.alloc_stream(L)
        C.encode_dev(L, x, cont, offs)
        C.sync()
        shape = C.ImageShape(16, 16, 3)
        C.dump_dev(L, cont, offs, shape, str(tmp_path / str(mode)), 0)
        files = sorted(os.listdir(tmp_path / str(mode)))
        assert len(files) == C.layout_chunks(L)
        cont2, offs2 = C.load_dev(L, shape, str(tmp_path / str(mode)), 0)
        out = torch.empty_like(x)
        C.decode_dev(L, cont2, out, offsets=offs2)
        C.sync()
        assert torch.equal(out, x)


def test_malformed_files(pkg, torch_cuda, tmp_path):
    torch = torch_cuda
    C, E = pkg.codec, pkg.errors
    L = C.layout(0, 1, 1, 1, 1)
    cont, _ = C.alloc_stream(L)
    C.encode_dev(L, torch.tensor([[9]], dtype=torch.uint8, device="cuda"), cont)
    C.dump_dev(L, cont, None, C.ImageShape(1, 1, 1), str(tmp_path), 0)
    good = (tmp_path / "batch_0_0.optb").read_bytes()
    cases = {"bad magic": b"NOPE" + good[4:], "unsupported version 2": good[:4] + b"\x02" + good[5:],
             "unknown mode tag 9": good[:6] + b"\x09" + good[7:], "truncated": good[:-3]}
    for msg, data in cases.items():
        (tmp_path / "batch_0_0.optb").write_bytes(data)
        with pytest.raises(E.FormatError, match=msg):
            C.load_dev(L, C.ImageShape(1, 1, 1), str(tmp_path), 0)
        with pytest.raises(E.FormatError, match=msg):
            C.read_optb(io.BytesIO(data))
    with pytest.raises(E.FormatError, match="missing batch file"):
        C.load_dev(L, C.ImageShape(1, 1, 1), str(tmp_path), 7)
