"""Child process of tests/test_gpu_ipc.py (cross-process template, f4).

Connects to the parent's Unix socket, receives (config, budget, prompt) and
the template's chunk fds (SCM_RIGHTS), imports the template read-only into
this process, runs one prefill with its own streaming arena, and sends back
the first token, the logits and the template checksum.
"""
import json
import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2503_06421_b200 import tidal as T  # noqa: E402


def main(path):
    s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    s.connect(path)
    msg, fds, _, _ = socket.recv_fds(s, 65536, 256)
    req = json.loads(msg.decode())
    cfg = synth.config(req["config"], **req["over"])
    tensors, fill = synth.model_inputs(cfg, req["seed"])
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    model = T.Model(cd, tensors, f"base:{req['seed']}", fill=fill)
    opts = T.template_opts(resident_bytes=req["budget"], max_tokens=req["max_tokens"], device=0)
    out = {}
    try:
        fp = req["fingerprint"]

        def refused(m, shared):
            try:
                T.Template(m, T.Trace(m), opts, shared=shared)
                return False
            except T.TidalError as e:
                return e.code == T.ERR_STRUCTURE
        # wrong shared_bytes, a wrong fingerprint, and the same shapes from
        # another checkpoint (same byte sizes, other provenance) are all refused
        out["bad_refused"] = refused(model, (fds, req["bad_bytes"], fp))
        out["bad_fp_refused"] = refused(model, (fds, req["shared_bytes"], fp ^ 1))
        other = T.Model(cd, tensors, f"base:{req['seed'] + 1}", fill=fill)
        out["other_ckpt_refused"] = refused(other, (fds, req["shared_bytes"], fp))
        tpl = T.Template(model, T.Trace(model), opts, shared=(fds, req["shared_bytes"], fp))
        for fd in fds:
            os.close(fd)
        c0 = tpl.checksum()
        tok, logits, st = tpl.invoke(np.array(req["prompt"], np.int32))
        out.update(token=int(tok), checksum_before=int(c0), checksum_after=int(tpl.checksum()),
                   bytes_streamed=int(st["bytes_streamed"]))
        out["logits"] = logits.tobytes().hex()
    except Exception as e:  # report, do not hang the parent
        out["error"] = repr(e)
    data = json.dumps(out).encode()
    s.sendall(len(data).to_bytes(8, "little") + data)
    s.close()


if __name__ == "__main__":
    main(sys.argv[1])
