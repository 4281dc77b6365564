"""oocs_plan_create_in (SURVEY §8(b) optional caller-owned arena): a plan carved out of a torch tensor runs
the same pipeline bit for bit as a self-allocated one; short, misaligned or host arenas are rejected; the
tensor outlives the plan."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("store", ["host", "device"])
def test_plan_in_torch_arena_is_bitwise_equal(store):
    nx, ny, nz, n, k = 40, 32, 64, 4, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az = vel.shape[0]
    cfg = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, rate_bits=16,
                           mode="swb", store=store)
    need = oocs.oocs_plan_estimate(cfg).arena_bytes
    arena = torch.full((need + 4096,), 0xAB, dtype=torch.uint8, device="cuda")  # dirty on purpose
    outs = []
    for pl in (oocs.Plan(cfg), oocs.Plan(cfg, arena=arena)):
        for a, arr in enumerate((vel, p0, p0)):
            pl.load(a, arr, 0, az)
        pl.run(3 * k)
        outs.append([pl.read_raw(a, 0, az) for a in (1, 2)])
        pl.close()
    assert all(np.array_equal(x, y) for x, y in zip(*outs))
    arena.add_(1)  # still a valid allocation after the plan is gone
    torch.cuda.synchronize()


def test_bad_arenas_are_rejected():
    cfg = oocs.make_config(nx=32, ny=32, nz=32, dt=0.1, n_blocks=2, tb_depth=1, rate_bits=16, store="device")
    need = oocs.oocs_plan_estimate(cfg).arena_bytes
    small = torch.empty(need - 256, dtype=torch.uint8, device="cuda")
    big = torch.empty(need + 512, dtype=torch.uint8, device="cuda")
    host = torch.empty(need, dtype=torch.uint8).pin_memory()
    for ptr, nbytes in ((small.data_ptr(), small.numel()), (big.data_ptr() + 8, need), (host.data_ptr(), need)):
        with pytest.raises(oocs.OocsError) as e:
            oocs.oocs_plan_create_in(cfg, ptr, nbytes)
        assert e.value.status == 2


@pytest.mark.parametrize("mode", ["swb", "baseline"])
def test_chunked_pcie_copies_are_bitwise_equal(mode, monkeypatch):
    """OOCS_COPY_CHUNK_MB splits every pipeline H2D/D2H into pieces (an experiment knob): the
    same bytes must arrive, for the codec pipeline and the pitched-store BASELINE."""
    nx, ny, nz, n, k = 40, 32, 64, 4, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az = vel.shape[0]
    codec = "identity" if mode == "baseline" else "blockquant"
    cfg = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, rate_bits=16,
                           codec=codec, mode=mode, store="host")
    outs = []
    for chunk in ("0", "0.004"):  # whole copies; 4 KB pieces
        monkeypatch.setenv("OOCS_COPY_CHUNK_MB", chunk)
        pl = oocs.Plan(cfg)
        for a, arr in enumerate((vel, p0, p0)):
            pl.load(a, arr, 0, az)
        pl.run(3 * k)
        outs.append([pl.read_raw(a, 0, az) for a in (1, 2)])
        pl.close()
    assert all(np.array_equal(x, y) for x, y in zip(*outs))
