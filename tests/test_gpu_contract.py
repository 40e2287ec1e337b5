"""GPU tests of the boundary's contract (include/vlut.h Conventions):
graph-replay safety of the split-K handshakes, the bounded library workspace
cache of vlut_mpgemm, per-stream workspaces in the binding, and the binding's
argument checks.  Every result is compared with the CPU oracle."""
import ctypes

import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def v():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2512_06443_b200 as vl
    return vl


def dev():
    return torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def _inputs(K, N, seed):
    x = synth.activations_f32(K, N, seed)
    return oracle.quantize(x)


@pytest.mark.parametrize("plan_kind", ["streamk", "streamk_rpt2", "streamk32", "slot_split",
                                       "slot_decode", "auto"])
def test_graph_replay_with_new_inputs(v, plan_kind):
    """A captured mpGeMM replayed three times with different activations in
    the same buffers: every replay must equal the oracle.  (With per-launch
    host epochs, a replay would reuse the captured epoch and owners would add
    stale partials -- the handshake must carry no host-side state.)"""
    M, K, g = 1000, 2560, 4
    N = {"slot_split": 8, "slot_decode": 1}.get(plan_kind, 256)
    plan = {"streamk": v.LaunchPlan(16, 1, streamk=1),
            "streamk_rpt2": v.LaunchPlan(12, 1, m_cta=768, streamk=1),
            "streamk32": v.LaunchPlan(12, 1, m_cta=768, n_cta=32, streamk=1),
            "slot_split": v.slot_plan(tpw=2, splits=5),
            "slot_decode": v.slot_plan(tpw=1, splits=20),
            "auto": None}[plan_kind]
    W = synth.ternary_weights(M, K, seed=77)
    pw = v.pack_weights(W, g, device=dev())
    q0, s0 = _inputs(K, N, 1)
    qd, sd = to_dev(q0), to_dev(s0)
    ws = torch.zeros_like(v.workspace(dev()))
    out = torch.empty((M, N), dtype=torch.float32, device=dev())
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, out=out, plan=plan, ws=ws)  # eager warm-up
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, out=out, plan=plan, ws=ws)
    for trial in range(3):
        q, s = _inputs(K, N, 100 + trial)
        qd.copy_(to_dev(q))
        sd.copy_(to_dev(s))
        out.fill_(float("nan"))
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
        assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32)), trial


def _cudart():
    try:
        from cuda.bindings import runtime as rt
    except ImportError:
        from cuda import cudart as rt
    return rt


def test_library_workspace_cache_bounded_over_100_streams(v):
    """vlut_mpgemm's library-owned workspaces: 100 streams created, used and
    destroyed one after another.  At most 4 workspaces stay cached per device
    and device memory does not grow past them; every result is exact
    (recycled stream handles must not alias a stale binding)."""
    rt = _cudart()
    M, K, N, g = 2000, 1280, 64, 4
    W = synth.ternary_weights(M, K, seed=3)
    pw = v.pack_weights(W, g, device=dev())
    q, s = _inputs(K, N, 4)
    qd, sd = to_dev(q), to_dev(s)
    ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
    v.release_workspaces()
    assert v.cached_workspaces() == 0
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(dev())[0]
    ws_bytes = int(v.lib().vlut_workspace_bytes())
    outs = []
    for i in range(100):
        err, h = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
        assert int(err) == 0
        es = torch.cuda.ExternalStream(int(h), device=dev())
        out = torch.empty((M, N), dtype=torch.float32, device=dev())
        v.mpgemm(pw, qd, sd, synth.W_SCALE, out=out, stream=es)
        if i % 10 == 0:
            outs.append(out)
        es.synchronize()
        assert int(rt.cudaStreamDestroy(h)[0]) == 0
        assert v.cached_workspaces() <= 4, i
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(dev())[0]
    # bounded: at most the 4 cached workspaces (+ allocator slack)
    assert free0 - free1 <= 4 * ws_bytes + (64 << 20), (free0 - free1) / 2**20
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.int32), ref.view(np.int32))
    v.release_workspaces()
    assert v.cached_workspaces() == 0
    # usable again after a release
    out = v.mpgemm(pw, qd, sd, synth.W_SCALE)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32))


def test_library_workspace_per_thread_default_stream(v):
    """cudaStreamPerThread resolves to the calling thread's own stream (its
    own workspace binding), distinct from the legacy default stream."""
    import threading
    M, K, N, g = 700, 640, 16, 4
    W = synth.ternary_weights(M, K, seed=5)
    pw = v.pack_weights(W, g, device=dev())
    q, s = _inputs(K, N, 6)
    qd, sd = to_dev(q), to_dev(s)
    ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
    per_thread = torch.cuda.ExternalStream(2, device=dev())  # cudaStreamPerThread
    results, errors = {}, []

    def work(i):
        try:
            torch.cuda.set_device(dev())
            outs = []
            for _ in range(20):
                outs.append(v.mpgemm(pw, qd, sd, synth.W_SCALE, stream=per_thread))
            per_thread.synchronize()
            results[i] = outs
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    for outs in results.values():
        for o in outs:
            assert np.array_equal(o.cpu().numpy().view(np.int32), ref.view(np.int32))


def test_binding_workspace_per_stream(v):
    """The binding's default workspace is per (device, stream): two streams
    running split-K launches concurrently with ws=None never share one."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    assert v.workspace(dev(), s1) is v.workspace(dev(), s1)
    assert v.workspace(dev(), s1) is not v.workspace(dev(), s2)
    M, K, g = 1500, 2560, 4
    W = synth.ternary_weights(M, K, seed=8)
    pw = v.pack_weights(W, g, device=dev())
    cases = []
    for N, seed in ((256, 9), (8, 10)):
        q, s = _inputs(K, N, seed)
        cases.append((to_dev(q), to_dev(s), oracle.dequant_f32(oracle.gemm_i32(W, q), s,
                                                             synth.W_SCALE)))
    plans = [v.LaunchPlan(16, 1, streamk=1), v.slot_plan(tpw=2, splits=7)]
    outs = []
    torch.cuda.synchronize()
    for rep in range(10):
        for st, (qd, sd, ref), pl in zip((s1, s2), cases, plans):
            with torch.cuda.stream(st):
                outs.append((v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=pl), ref))
    torch.cuda.synchronize()
    for o, ref in outs:
        assert np.array_equal(o.cpu().numpy().view(np.int32), ref.view(np.int32))


def test_binding_rejects_bad_tensors(v):
    """dtype / shape / device checks before anything reaches the C ABI."""
    M, K, N, g = 64, 64, 16, 4
    pw = v.pack_weights(synth.ternary_weights(M, K, seed=1), g, device=dev())
    q, s = _inputs(K, N, 2)
    qd, sd = to_dev(q), to_dev(s)
    with pytest.raises(TypeError):
        v.mpgemm(pw, qd.float(), sd, 0.02)                       # A not int8
    with pytest.raises(TypeError):
        v.mpgemm(pw, qd, sd.double(), 0.02)                      # a_scale not fp32
    with pytest.raises(ValueError):
        v.mpgemm(pw, qd, sd[:N - 1], 0.02)                       # short a_scale
    with pytest.raises(ValueError):
        v.mpgemm(pw, qd, sd, 0.02, out=torch.empty((M, N - 1), device=dev()))  # short out
    with pytest.raises(TypeError):
        v.mpgemm(pw, qd, sd, 0.02, out=torch.empty((M, N), dtype=torch.int32, device=dev()))
    with pytest.raises(TypeError):
        v.mpgemm_acc(pw, qd, out=torch.empty((M, N), dtype=torch.float32, device=dev()))
    with pytest.raises(ValueError):
        v.mpgemm(pw, qd[:K - 4], sd, 0.02)                       # K mismatch
    with pytest.raises(ValueError):
        v.mpgemm(pw, qd.cpu(), sd, 0.02)                         # CPU tensor: no fallback
    with pytest.raises(TypeError):
        v.mpgemm_fused(pw, qd, sd, 0.02, amax=torch.zeros((N,), dtype=torch.float32,
                                                         device=dev()))
    with pytest.raises(ValueError):
        v.quantize(torch.zeros((K, N), device=dev()), q=torch.empty((K, N + 1), dtype=torch.int8,
                                                                    device=dev()))


def test_pack_device_then_mpgemm_back_to_back(v):
    """vlut_pack_weights_device immediately followed by the mpGeMM on the same
    stream (the kernels stage weights before griddepcontrol.wait; the packer
    ends with an event record so the next launch waits for it): exact, over
    many fresh payloads and every schedule."""
    M, K, N, g = 1000, 2560, 256, 4
    q, s = _inputs(K, N, 11)
    qd, sd = to_dev(q), to_dev(s)
    ws = torch.zeros_like(v.workspace(dev()))
    plans = [None, v.LaunchPlan(12, 2), v.LaunchPlan(16, 1, streamk=1)]
    for i in range(6):
        W = synth.ternary_weights(M, K, seed=200 + i)
        Wd = to_dev(W)
        torch.cuda.synchronize()
        pw = v.pack_weights_device(Wd, g)
        out = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=plans[i % 3], ws=ws)
        torch.cuda.synchronize()
        ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
        assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32)), i


def test_fused_decode_graph_replay_with_new_inputs(v):
    """vlut_mpgemm_decode captured once and replayed with new activations in
    the same buffer: the absmax, the codes and the counted split-K meeting
    carry no state between replays."""
    M, K, g = 3072, 23040, 4
    W = synth.ternary_weights(M, K, seed=5)
    pw = v.pack_weights(W, g, device=dev())
    xd = torch.empty((K,), dtype=torch.float32, device=dev())
    out = torch.empty((M,), dtype=torch.float32, device=dev())
    sc = torch.empty((1,), dtype=torch.float32, device=dev())
    ws = torch.zeros_like(v.workspace(dev()))
    st = torch.cuda.Stream()
    xd.copy_(to_dev(synth.activations_f32(K, 1, seed=1)[:, 0].copy()))
    with torch.cuda.stream(st):
        v.mpgemm_decode(pw, xd, synth.W_SCALE, out=out, scale_out=sc, ws=ws)  # warm-up
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        v.mpgemm_decode(pw, xd, synth.W_SCALE, out=out, scale_out=sc, ws=ws)
    for trial in range(3):
        x = synth.activations_f32(K, 1, seed=50 + trial)[:, 0].copy() * (10.0 ** trial)
        xd.copy_(to_dev(x))
        out.fill_(float("nan"))
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        q, s = oracle.quantize(x[:, None])
        ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)[:, 0]
        assert np.array_equal(sc.cpu().numpy().view(np.int32), s.view(np.int32)), trial
        assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32)), trial
