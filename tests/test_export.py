"""Probe export (export.hpp:17-30, export.cpp:53-101): the engine writes the
last run's traces as NENG1 bytes / CSV text straight from its probe block.
Checked byte for byte against the reference's own write_probe_binary /
write_probe_csv on EngineCore<float>'s ProbeOutput of the same run."""
import struct

import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import networks, passes


def parse_neng1(raw: bytes):
    """NENG1 layout (export.hpp:20-23): magic | u8 width | u32 count | per probe
    i32 key, batch, steps, dim, then f64 values in (batch, step, dim) order."""
    assert raw[:5] == b"NENG1" and raw[5] == 8
    (count,) = struct.unpack_from("<I", raw, 6)
    at, out = 10, {}
    for _ in range(count):
        key, b, s, d = struct.unpack_from("<4i", raw, at)
        at += 16
        out[key] = np.frombuffer(raw, "<f8", b * s * d, at).reshape(b, s, d)
        at += 8 * b * s * d
    assert at == len(raw)
    return out


def test_reference_dump_layout_matches_run_output(tmp_path):
    # pins the format restatement above on the reference itself (CPU)
    w = networks.random_network(4, n_ens=4, n=32, d=3, k_out=2, n_inputs=2, batch=3, steps=7, probes=3)
    pm = passes.run_passes(w.model)
    ref = refapi.RefEngine(pm, w.batch)
    out = ref.run(w.steps, w.feeds)
    ref.write_probe_binary(str(tmp_path / "r.bin"))
    parsed = parse_neng1((tmp_path / "r.bin").read_bytes())
    assert sorted(parsed) == sorted(out)
    for k in out:
        assert np.array_equal(parsed[k], out[k])
    ref.write_probe_csv(str(tmp_path / "r.csv"), pm.model.dt)
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == "step,time,batch,probe_key,dim_index,value"
    assert len(lines) == 1 + sum(v.size for v in out.values())


@pytest.mark.gpu
@pytest.mark.parametrize("net", ["small", "probe_rich"])
def test_gpu_export_is_byte_identical_to_the_reference(net, tmp_path):
    from paper_1805_11144_b200.engine import GpuEngine
    from paper_1805_11144_b200.ir import RunError
    if net == "small":
        w = networks.random_network(4, n_ens=6, n=48, d=3, k_out=2, n_inputs=3, batch=5, steps=9, probes=4)
    else:
        from tests.test_fused import probe_rich_network
        w = probe_rich_network(batch=6, steps=12)
    pm = passes.run_passes(w.model)
    gpu, ref = GpuEngine(pm, w.batch), refapi.RefEngine(pm, w.batch)
    with pytest.raises(RunError):
        gpu.probe_dump()
    for call in range(2):  # the export follows the last run
        n = w.steps - 3 * call
        feeds = {k: v[:, :n] for k, v in w.feeds.items()}
        gpu.run(n, feeds)
        ref.run(n, feeds)
    gpu.write_probe_binary(str(tmp_path / "g.bin"))
    ref.write_probe_binary(str(tmp_path / "r.bin"))
    assert (tmp_path / "g.bin").read_bytes() == (tmp_path / "r.bin").read_bytes()
    assert gpu.probe_dump() == (tmp_path / "r.bin").read_bytes()
    gpu.write_probe_csv(str(tmp_path / "g.csv"), pm.model.dt)
    ref.write_probe_csv(str(tmp_path / "r.csv"), pm.model.dt)
    assert (tmp_path / "g.csv").read_bytes() == (tmp_path / "r.csv").read_bytes()
