"""GPU-side ordering guarantees of the C ABI (an agent "never resumes decode while any of its blocks are
host-resident or in flight"; one cycle's uploads, then its offloads, on asynchronous copy streams).

* write ordering — tc_set_compute_stream: an offload issued right after the engine queued decode writes into the
  agent's blocks (no host sync) captures those writes;
* read ordering — tc_stream_wait: a consumer kernel queued on a caller stream behind tc_stream_wait(h) reads the
  uploaded bytes and the remapped device table, with no host wait in between;
* table pushes vs a later offload's fused table epilogue (the staging-halves gather runs on the offload aux stream);
* the smallest staging buffer (clamped to two blocks) with multi-block ring batches.

Each test makes the race observable by putting a long GPU sleep in front of the producer; the expected bytes come
from the content generator / oracle, never from the CUDA path.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2510_18586_b200 as tcb  # noqa: E402
from oracle import BytesStore, OraclePool  # noqa: E402
from oracle.pool import OFFLOADED  # noqa: E402
from workloads import content  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import fuzz_script  # noqa: E402

SLEEP_CYCLES = 200_000_000          # ~0.1 s at ~2 GHz: far longer than any launch latency below


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def mk(L, H, D, N, S, mode=tcb.XFER_STAGED, seed=1, **kw):
    c = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, n_classes=2, xfer_d2h=mode, xfer_h2d=mode, **kw)
    c.fill(seed)
    return c


@pytest.mark.parametrize("mode", [tcb.XFER_STAGED, tcb.XFER_DIRECT, tcb.XFER_COPY])
def test_compute_stream_orders_offload_after_decode_writes(mode):
    """Decode writes queued on the registered compute stream (behind a long sleep) land in the offloaded host image:
    the offload is issued immediately, with no host synchronisation."""
    L, H, D, N, S = 4, 4, 128, 64, 32
    c = mk(L, H, D, N, S, mode)
    comp = torch.cuda.Stream(device=0)
    c.set_compute_stream(comp.cuda_stream)
    c.agent_add(0, 0)
    ids = c.alloc(0, 6)
    torch.cuda.synchronize()
    kv = c.kv_tensor()                                   # [L][2][N][C] bytes
    marker = torch.arange(c.chunk_bytes, dtype=torch.int32, device="cuda:0").to(torch.uint8) ^ 0xA5
    with torch.cuda.stream(comp):
        torch.cuda._sleep(SLEEP_CYCLES)
        for b in ids:                                    # the agent's "last decode step" rewrites every chunk
            kv[:, :, b, :] = marker
    h = c.offload(0, ids)                                # no host sync between the writes and the offload
    c.wait(h)
    exp = np.broadcast_to(marker.cpu().numpy(), (L, 2, c.chunk_bytes)).reshape(-1)
    for i in range(len(ids)):
        assert np.array_equal(c.handle_host_bytes(h, i).reshape(-1), exp), i
    c.set_compute_stream(None)
    c.sync()
    c.close()


@pytest.mark.parametrize("mode", [tcb.XFER_STAGED, tcb.XFER_DIRECT, tcb.XFER_COPY])
def test_stream_wait_orders_consumer_after_upload(mode):
    """A consumer on a caller stream, queued behind tc_stream_wait(h) right after tc_upload (no host wait), reads the
    scattered blocks and the remapped device table: both equal the oracle's bytes and ids.  The upload is held back by
    a long sleep on the upload stream, so a missing dependency would read stale bytes."""
    L, H, D, N, S = 4, 4, 128, 64, 32
    pool0 = content.pool_bytes(3, L, N, 16, H, D)
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    c = mk(L, H, D, N, S, mode, seed=3)
    for x in (o, c):
        x.agent_add(0, 0)
        x.agent_add(1, 1)
    assert o.alloc(0, 8) == list(c.alloc(0, 8))
    assert o.alloc(1, 4) == list(c.alloc(1, 4))
    ho, hc = o.offload(0, o.block_table(0)), c.offload(0, c.block_table(0))
    o.sync(); c.sync()
    assert o.alloc(1, 3) == list(c.alloc(1, 3))          # the freed blocks are taken: the upload lands elsewhere
    c.sync()
    up_s, _ = c.streams()
    ups = torch.cuda.ExternalStream(up_s, device=0)
    with torch.cuda.stream(ups):
        torch.cuda._sleep(SLEEP_CYCLES)                  # the upload's H2D + scatter queue behind this
    new_o, new_c = o.upload(ho), c.upload(hc)
    assert new_o == list(new_c)
    consumer = torch.cuda.Stream(device=0)
    c.stream_wait(hc, consumer.cuda_stream)
    kv, tab = c.kv_tensor(), c.table_tensor()
    with torch.cuda.stream(consumer):
        got = kv[:, :, torch.tensor(new_c, dtype=torch.int64, device="cuda:0")].clone()
        row = tab[0, :8].clone()
    consumer.synchronize()
    assert row.cpu().tolist() == new_o
    assert np.array_equal(got.cpu().numpy(), o.store.pool[:, :, new_o])
    c.sync()
    c.close()


def test_table_push_not_overwritten_by_later_offload_epilogue():
    """No compute stream: tc_alloc's table push is queued on the offload stream behind a large D2H; an offload of the
    new blocks right after it gathers on the offload aux stream (staging halves).  Its fused epilogue (-1) must land
    after the push, so the device table shows the blocks as host-resident."""
    L, H, D, N, S = 28, 4, 128, 1024, 600             # C2-shaped 896 KiB blocks
    c = mk(L, H, D, N, S, tcb.XFER_STAGED)
    for a in range(2):
        c.agent_add(a, 0)
    c.alloc(0, 400)
    c.sync()
    for rep in range(3):
        h0 = c.offload(0, c.block_table(0))              # ~360 MB D2H queued on the offload stream
        ids = c.alloc(1, 4)                              # push queued behind it on the same stream
        h1 = c.offload(1, ids)                           # gather on the aux stream (a half-buffer batch)
        c.sync()
        assert (c.table_tensor()[1, 4 * rep:4 * rep + 4].cpu() == -1).all(), rep
        assert (c.table_tensor()[0, :400].cpu() == -1).all()
        c.upload(h0)
        c.upload(h1)
        c.sync()
        assert c.table_tensor()[1, :4 * rep + 4].cpu().tolist() == c.block_table(1)
    c.close()


@pytest.mark.parametrize("staging_blocks", [0.5, 1, 1.5])
def test_tiny_staging_buffer_clamped_to_two_blocks(staging_blocks):
    """staging_bytes below two blocks is raised to two blocks: multi-block staged batches alternate two one-block
    halves inside the buffer (they used to write one block past its end).  Pool bytes, host images, tables and
    counters equal the oracle after every sync."""
    L, H, D, N, S, T = 3, 2, 64, 50, 30, 16
    B = 2 * L * T * H * D * 2
    pool0 = content.pool_bytes(8, L, N, T, H, D)
    for seed in range(3):
        ops = fuzz_script(seed + 600, n_ops=120, n_agents=3, n_classes=2, N=N, max_alloc=7, retire=True,
                          lags=(1, 2))
        o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0.copy(), S))
        c = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=S, n_classes=2, xfer_d2h=tcb.XFER_STAGED,
                      xfer_h2d=tcb.XFER_STAGED, staging_bytes=int(staging_blocks * B))
        c.fill(8)
        ro, rc = Replayer(o), Replayer(c)
        for i, op in enumerate(ops):
            assert ro.step(op) == rc.step(op), (seed, i, op)
            if op[0] == "sync":
                assert np.array_equal(c.kv_tensor().cpu().numpy(), o.store.pool), (seed, i)
        c.sync()
        o.sync()
        assert np.array_equal(c.kv_tensor().cpu().numpy(), o.store.pool), seed
        c.close()


def test_device_tier_on_destroyed_caller_stream_does_not_poison_sync():
    """tc_gather_dev on a caller stream that is then destroyed: the next tc_sync waits on an event behind the launch,
    not on the stream handle, and succeeds (it used to fail with TC_E_CUDA forever)."""
    L, H, D, N, S = 2, 2, 64, 32, 8
    c = mk(L, H, D, N, S)
    ids = np.arange(5, dtype=np.int32)
    dst = torch.empty(5 * c.block_bytes, dtype=torch.uint8, device="cuda:0")
    from cuda.bindings import runtime as cudart
    err, s = cudart.cudaStreamCreate()                   # a raw caller stream the test really destroys
    assert int(err) == 0
    c.gather_dev(ids, dst.data_ptr(), int(s))
    assert int(cudart.cudaStreamSynchronize(s)[0]) == 0
    assert int(cudart.cudaStreamDestroy(s)[0]) == 0
    c.sync()                                             # raises TcError on a non-OK status
    c.agent_add(0, 0)
    c.alloc(0, 2)
    c.sync()
    pool0 = content.pool_bytes(1, L, N, 16, H, D)
    assert np.array_equal(dst.cpu().numpy().reshape(5, L, 2, c.chunk_bytes),
                          np.take(pool0, ids, axis=2).transpose(2, 0, 1, 3))
    c.close()


def _piece_pool(kind, monkeypatch, L, H, D, N, S, seed):
    """A staged pool whose multi-block batches run as several pieces: `ring` = a 4-block staging buffer (2-block
    halves reused in turn), `pieces` = a large buffer cut into one-block pieces (TC_PIECE_KIB), no staging halves;
    `*_aligned`: pieces also end on item boundaries (TC_MIN_PIECE_MIB=0, i.e. no minimum piece size)."""
    T = 16
    B = 2 * L * T * H * D * 2
    if kind.endswith("_aligned"):
        monkeypatch.setenv("TC_MIN_PIECE_MIB", "0")
        kind = kind[:-len("_aligned")]
    if kind == "pieces":
        monkeypatch.setenv("TC_PIECE_KIB", str(max(1, B // 1024)))
        monkeypatch.setenv("TC_STAGING_HALVES", "0")
        staging = 64 * B
    else:
        staging = 4 * B
    c = tcb.Pool(L, H, D, T, "bf16", N, device=0, host_slots=S, n_classes=2, xfer_d2h=tcb.XFER_STAGED,
                 xfer_h2d=tcb.XFER_STAGED, staging_bytes=staging)
    c.fill(seed)
    return c


@pytest.mark.parametrize("kind", ["ring", "pieces", "ring_aligned", "pieces_aligned"])
def test_multi_piece_upload_waits_for_each_items_offload(kind, monkeypatch):
    """A batch upload of several pieces issued right behind the batch offload it undoes, with the offload's copies
    held back by a long sleep on the offload stream: each upload piece waits for the offload pieces holding its
    handles' blocks (per-piece dependencies), so every scattered block equals the oracle's bytes.  A piece that did
    not wait would copy host slots the D2H had not written yet."""
    L, H, D, N, S = 2, 2, 64, 96, 40
    pool0 = content.pool_bytes(5, L, N, 16, H, D)
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    c = _piece_pool(kind, monkeypatch, L, H, D, N, S, 5)
    for x in (o, c):
        for a in range(8):
            x.agent_add(a, 0)
    for rnd in range(4):                              # interleaved growth: scattered ids, 1-4 blocks per agent
        for a in range(8):
            if rnd <= a % 4:
                assert o.alloc(a, 1) == list(c.alloc(a, 1))
    for rep in range(3):
        # decoys 4-7 first pass through the same host slots (and allocate the staging buffers, whose cudaMalloc
        # would synchronise the device): an upload that did not wait would read their bytes
        items = [(a, o.block_table(a)) for a in range(4, 8)]
        assert c.offload_batch(items) == o.offload_batch(items)
        hs = [h for h in sorted(o.handles) if o.handles[h].state == OFFLOADED]
        assert o.upload_batch(hs) == c.upload_batch(hs)
        c.sync()
        o.sync()
        _, off_s = c.streams()
        with torch.cuda.stream(torch.cuda.ExternalStream(off_s, device=0)):
            torch.cuda._sleep(SLEEP_CYCLES)           # the offload's copies queue behind this
        items = [(a, o.block_table(a)) for a in range(4)]
        assert c.offload_batch(items) == o.offload_batch(items)
        hs = [h for h in sorted(o.handles) if o.handles[h].state == OFFLOADED]
        new_o, new_c = o.upload_batch(hs), c.upload_batch(hs)   # no host wait in between
        assert new_o == new_c, rep
        c.sync()
        o.sync()
        assert np.array_equal(c.kv_tensor().cpu().numpy(), o.store.pool), (kind, rep)
        for a in range(8):
            assert c.block_table(a) == o.block_table(a)
    c.close()


@pytest.mark.parametrize("kind", ["ring", "pieces", "ring_aligned", "pieces_aligned"])
def test_multi_piece_offload_waits_for_each_items_upload(kind, monkeypatch):
    """A batch offload of several pieces issued right behind the batch upload that brought its agents back, with the
    upload's copies held back by a long sleep on the upload stream: each gather piece waits for the upload pieces
    holding its agents' blocks, so every offloaded host image equals the oracle's.  A piece that did not wait would
    gather blocks the scatter had not written yet."""
    L, H, D, N, S = 2, 2, 64, 96, 40
    pool0 = content.pool_bytes(6, L, N, 16, H, D)
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    c = _piece_pool(kind, monkeypatch, L, H, D, N, S, 6)
    for x in (o, c):
        for a in range(4):
            x.agent_add(a, 0)
    for rnd in range(4):                              # 1-4 blocks per agent
        for a in range(4):
            if rnd <= a:
                assert o.alloc(a, 1) == list(c.alloc(a, 1))
    items = [(a, o.block_table(a)) for a in range(4)]
    assert c.offload_batch(items) == o.offload_batch(items)
    for rep in range(3):
        c.sync()
        o.sync()
        up_s, _ = c.streams()
        with torch.cuda.stream(torch.cuda.ExternalStream(up_s, device=0)):
            torch.cuda._sleep(SLEEP_CYCLES)           # the upload's copies queue behind this
        hs = [h for h in sorted(o.handles) if o.handles[h].state == OFFLOADED]
        assert o.upload_batch(hs) == c.upload_batch(hs)
        items = [(a, o.block_table(a)) for a in range(4)]
        got = c.offload_batch(items)                  # no host wait in between
        assert got == o.offload_batch(items)
        for h in got:
            c.wait(h)
            for i, s in enumerate(o.handles[h].slots):
                assert np.array_equal(c.handle_host_bytes(h, i), o.store.host[s]), (kind, rep, h, i)
    c.sync()
    c.close()


def test_first_handle_of_a_multi_piece_upload_completes_before_the_last():
    """Per-handle completion: in an upload batch that runs as several pieces (8 agents x 96 MiB, C3-shaped 2 MiB
    blocks, pieces cut on item boundaries), the first handle's completion (tc_query) comes well before the last
    one's — an engine can resume that agent while the rest of the batch is still on the link.  Bytes and tables are
    then checked against the oracle."""
    L, H, D, N, S = 32, 8, 128, 800, 400
    n_ag, per = 8, 48
    pool0 = content.pool_bytes(4, L, N, 16, H, D)
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    c = mk(L, H, D, N, S, tcb.XFER_STAGED, seed=4)
    for x in (o, c):
        for a in range(n_ag):
            x.agent_add(a, 0)
    for a in range(n_ag):
        assert o.alloc(a, per) == list(c.alloc(a, per))
    import time
    for rep in range(2):                              # rep 0 warms the path up (staging buffers, kernel loading)
        items = [(a, o.block_table(a)) for a in range(n_ag)]
        assert c.offload_batch(items) == o.offload_batch(items)
        c.sync()
        o.sync()
        hs = [h for h in sorted(o.handles) if o.handles[h].state == OFFLOADED]
        t0 = time.perf_counter()
        new_c = c.upload_batch(hs)
        done = {}
        while len(done) < 2 and time.perf_counter() - t0 < 10:
            for h in (hs[0], hs[-1]):
                if h not in done and c.query(h):
                    done[h] = time.perf_counter() - t0
        assert o.upload_batch(hs) == new_c
        c.sync()
        o.sync()
    assert len(done) == 2, done
    assert done[hs[0]] + 2e-3 < done[hs[-1]], done      # ~768 MiB batch: ~15 ms on the link, first piece ~4 ms
    assert np.array_equal(c.kv_tensor().cpu().numpy(), o.store.pool)
    for a in range(n_ag):
        assert c.block_table(a) == o.block_table(a)
    c.close()
