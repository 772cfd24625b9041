"""Cross-process templates (§3, §5.1: the
template server shares read-only function templates with function processes
over CUDA IPC) — GPU.

The parent builds a template, exports the device chunks of its resident
prefix as POSIX fds and passes them over a Unix socket (SCM_RIGHTS) to a
fresh child process (tests/ipc_child.py), which imports them read-only,
streams the rest into its own arena and runs the prefill.  Checked: the
child's logits are bit-identical to the parent's and within 2e-2 of the
oracle, both processes see the same template checksum before and after the
child's invocation (copy-on-write across processes), a wrong shared size is
refused (STRUCTURE), and the exporter refuses to shrink its prefix below the
exported bytes.
"""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import synth
from oracle import forward as F

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_06421_b200 import build
    build.build()
    from paper_2503_06421_b200 import tidal
    tidal.lib()
    return tidal


def _child_run(req, fds):
    path = os.path.join(tempfile.mkdtemp(), "tidal.sock")
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(path)
    srv.listen(1)
    proc = subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_child.py"), path])
    try:
        srv.settimeout(300)
        conn, _ = srv.accept()
        conn.settimeout(600)
        socket.send_fds(conn, [json.dumps(req).encode()], fds)
        hdr = b""
        while len(hdr) < 8:
            hdr += conn.recv(8 - len(hdr))
        n = int.from_bytes(hdr, "little")
        data = b""
        while len(data) < n:
            data += conn.recv(n - len(data))
        conn.close()
        assert proc.wait(timeout=300) == 0
    finally:
        if proc.poll() is None:
            proc.kill()
        srv.close()
    return json.loads(data.decode())


@pytest.mark.parametrize("cfg_name,over,S,frac", [
    ("tiny", {}, 16, 0.6),
    ("13b", {"n_layers": 2}, 96, 0.7),
])
def test_template_shared_across_processes(T, cfg_name, over, S, frac):
    cfg = synth.config(cfg_name, **over)
    tensors, fill = synth.model_inputs(cfg, 0)
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    model = T.Model(cd, tensors, "base:0", fill=fill)
    M = sum(t.nbytes for t in synth.base_tensors(cfg))
    budget = int(frac * M)
    tpl = T.Template(model, T.Trace(model), T.template_opts(resident_bytes=budget, max_tokens=S,
                                                            device=0))
    fds, shared, fp = tpl.export()
    assert len(fds) >= 1 and shared > 0
    c0 = tpl.checksum()
    prompt = synth.prompt_fast(cfg, S, 0)
    req = dict(config=cfg_name, over=over, seed=0, budget=budget, max_tokens=S,
               prompt=[int(x) for x in prompt], shared_bytes=shared, bad_bytes=shared + 4096,
               fingerprint=fp)
    res = _child_run(req, fds)
    for fd in fds:
        os.close(fd)
    assert "error" not in res, res.get("error")
    assert res["bad_refused"] and res["bad_fp_refused"] and res["other_ckpt_refused"]
    assert res["checksum_before"] == res["checksum_after"] == c0
    assert res["bytes_streamed"] > 0
    tok, logits, _ = tpl.invoke(prompt)
    child_logits = np.frombuffer(bytes.fromhex(res["logits"]), np.float32)
    assert res["token"] == tok
    assert np.array_equal(child_logits, logits)
    assert tpl.checksum() == c0
    ref = F.forward(cfg, F.synth_weights(cfg, 0, fast=True, keep=False), prompt)
    assert float(np.abs(logits - ref["logits"]).max()) <= 2e-2
    # the exporter may grow its prefix but not stream into the shared bytes
    with pytest.raises(T.TidalError):
        tpl.resize(T.template_opts(resident_bytes=0))
    tpl.resize(T.template_opts(resident_bytes=T.U64_MAX))
    del tpl, model
