"""Oracle-side network driver (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Chains the oracle.c layer functions in the order the paper states: forward
through every layer in order, then "back-propagation through each layer, but
in reverse order" after the solver-side loss.  Blobs are
stored in fp32 between layers (Caffe float blobs; Table 1 "single
precision" P:254): each layer computes in fp64 from the fp32 inputs and its
output is rounded to fp32 once.  Gradients of parameters are returned
unrounded (fp64 truth) together with their tolerance scale S.

The spec parser below is the oracle's own (it shares no code with the
library's C++ parser); both read the same text format.
"""
import numpy as np

from . import capi

_KEYS = {
    "input": {"name", "channels", "height", "width"},
    "Convolution": {"name", "type", "bottom", "top", "num_output", "kernel_size", "kernel_h",
                    "kernel_w", "stride", "stride_h", "stride_w", "pad", "pad_h", "pad_w",
                    "bias_term", "group"},
    "Pooling": {"name", "type", "bottom", "top", "pool", "kernel_size", "kernel_h", "kernel_w",
                "stride", "stride_h", "stride_w", "pad", "pad_h", "pad_w"},
    "InnerProduct": {"name", "type", "bottom", "top", "num_output", "bias_term"},
    "ReLU": {"name", "type", "bottom", "top", "negative_slope"},
    "SoftmaxWithLoss": {"name", "type", "bottom", "top"},
    "Softmax": {"name", "type", "bottom", "top"},
    "Accuracy": {"name", "type", "bottom", "top", "top_k"},
}


def parse_spec(text):
    sections = []
    cur = None
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("[") and line.endswith("]"):
            cur = {"__section__": line[1:-1].strip()}
            sections.append(cur)
            continue
        if cur is None or "=" not in line:
            raise ValueError(f"spec parse error: {raw!r}")
        k, v = (s.strip() for s in line.split("=", 1))
        cur[k] = v
    if not sections or sections[0]["__section__"] != "input":
        raise ValueError("spec must start with an [input] section")
    inp = sections[0]
    for k in inp:
        if k != "__section__" and k not in _KEYS["input"]:
            raise ValueError(f"unknown key {k}")
    layers = []
    for s in sections[1:]:
        if s["__section__"] != "layer":
            raise ValueError(f"unknown section {s['__section__']}")
        t = s.get("type")
        if t not in _KEYS:
            raise ValueError(f"unknown layer type {t}")
        for k in s:
            if k != "__section__" and k not in _KEYS[t]:
                raise ValueError(f"unknown key {k} for {t}")
        layers.append(s)
    return inp, layers


def _hw(s, base, default):
    both = s.get(base + "_size" if base == "kernel" else base)
    h = s.get(base + "_h", both if both is not None else default)
    w = s.get(base + "_w", both if both is not None else default)
    if h is None or w is None:
        raise ValueError(f"missing {base} for layer {s.get('name')}")
    return int(h), int(w)


def grouped_conv_fwd(x, w, b, G, stride, pad):
    """Grouped convolution (Caffe `group` [outside ref]): the
    input channels and the filters are split into G equal groups and group g's
    filters see only group g's channels -- G independent convolutions whose
    outputs are concatenated along channels.  Returns (y, S)."""
    if G == 1:
        return capi.conv_fwd(x, w, b, stride, pad, want_scale=True)
    Cg, Fg = x.shape[1] // G, w.shape[0] // G
    ys, Ss = [], []
    for g in range(G):
        y, S = capi.conv_fwd(x[:, g * Cg:(g + 1) * Cg], w[g * Fg:(g + 1) * Fg],
                             None if b is None else b[g * Fg:(g + 1) * Fg], stride, pad, want_scale=True)
        ys.append(y)
        Ss.append(S)
    return np.concatenate(ys, axis=1), np.concatenate(Ss, axis=1)


def grouped_conv_bwd(dy, x, w, G, stride, pad, want_dx=True):
    """Backward of grouped_conv_fwd, group by group: (dw, db, dx, Sdw, Sdb, Sdx)."""
    if G == 1:
        return capi.conv_bwd(dy, x, w, stride, pad, want_dx=want_dx, want_scale=True)
    Cg, Fg = x.shape[1] // G, w.shape[0] // G
    parts = [capi.conv_bwd(dy[:, g * Fg:(g + 1) * Fg], x[:, g * Cg:(g + 1) * Cg], w[g * Fg:(g + 1) * Fg],
                           stride, pad, want_dx=want_dx, want_scale=True) for g in range(G)]
    cat = lambda i, ax: None if parts[0][i] is None else np.concatenate([q[i] for q in parts], axis=ax)
    return cat(0, 0), cat(1, 0), cat(2, 1), cat(3, 0), cat(4, 0), cat(5, 1)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


class OracleNet:
    """Linear-chain net over a named-blob registry (Fig. 1)."""

    def __init__(self, spec_text, batch):
        inp, specs = parse_spec(spec_text)
        self.batch = batch
        self.input_name = inp["name"]
        shapes = {inp["name"]: (batch, int(inp["channels"]), int(inp["height"]),
                                int(inp["width"]))}
        self.layers = []
        self.accuracy_layers = []  # test-phase side outputs (forward only, off the chain)
        for s in specs:
            L = {"name": s["name"], "type": s["type"], "bottom": s["bottom"], "top": s["top"]}
            if s["bottom"] not in shapes:
                raise ValueError(f"dangling blob {s['bottom']}")
            N, C, H, W = shapes[s["bottom"]]
            t = s["type"]
            if t == "Convolution":
                F = int(s["num_output"])
                kh, kw = _hw(s, "kernel", None)
                sh, sw = _hw(s, "stride", 1)
                ph, pw = _hw(s, "pad", 0)
                Ho, Wo = capi.conv_out_size(H, kh, sh, ph), capi.conv_out_size(W, kw, sw, pw)
                if Ho < 1 or Wo < 1:
                    raise ValueError("shape inference failure")
                G = int(s.get("group", "1"))
                if G < 1 or C % G or F % G:
                    raise ValueError("group must divide channels and num_output")
                L.update(F=F, C=C, k=(kh, kw), s=(sh, sw), p=(ph, pw), G=G,
                         bias=s.get("bias_term", "true") != "false",
                         wshape=(F, C // G, kh, kw), blen=F)
                shapes[s["top"]] = (N, F, Ho, Wo)
            elif t == "Pooling":
                method = {"MAX": capi.MAX, "AVE": capi.AVE}[s.get("pool", "MAX")]
                kh, kw = _hw(s, "kernel", None)
                sh, sw = _hw(s, "stride", 1)
                ph, pw = _hw(s, "pad", 0)
                Hp, Wp = capi.pool_out_size(H, kh, sh, ph), capi.pool_out_size(W, kw, sw, pw)
                if Hp < 1 or Wp < 1:
                    raise ValueError("shape inference failure")
                L.update(method=method, k=(kh, kw), s=(sh, sw), p=(ph, pw))
                shapes[s["top"]] = (N, C, Hp, Wp)
            elif t == "InnerProduct":
                No = int(s["num_output"])
                K = C * H * W
                L.update(Nout=No, K=K, bias=s.get("bias_term", "true") != "false",
                         wshape=(No, K), blen=No)
                shapes[s["top"]] = (N, No, 1, 1)
            elif t == "ReLU":
                L.update(slope=float(s.get("negative_slope", "0")))
                shapes[s["top"]] = (N, C, H, W)
            elif t == "SoftmaxWithLoss":
                L.update(D=C * H * W)
                shapes[s["top"]] = (1, 1, 1, 1)
            elif t == "Softmax":
                L.update(D=C * H * W)
                shapes[s["top"]] = (N, C, H, W)
            elif t == "Accuracy":
                k = int(s.get("top_k", "1"))
                if not 1 <= k <= C * H * W:
                    raise ValueError("top_k out of range")
                L.update(D=C * H * W, k=k, in_shape=(N, C, H, W))
                shapes[s["top"]] = (1, 1, 1, 1)
                self.accuracy_layers.append(L)
                continue
            L["in_shape"] = (N, C, H, W)
            L["out_shape"] = shapes[s["top"]]
            self.layers.append(L)
        self.shapes = shapes
        self.params = {}

    def learnable(self):
        """[(name, kind, weight_shape, bias_len)] in spec order."""
        return [(L["name"], L["type"], L["wshape"], L["blen"]) for L in self.layers
                if L["type"] in ("Convolution", "InnerProduct")]

    def set_params(self, params):
        self.params = {k: np.asarray(v, np.float32).copy() for k, v in params.items()}

    # ---------------------------------------------------------------- forward
    def forward(self, x, labels):
        """Returns dict: blobs (fp32 values as float64, by layer output),
        masks, loss (float64), prob, pred; keeps what backward needs."""
        P = self.params
        blobs = {self.input_name: f32(x)}
        out = {"blobs": {}, "masks": {}, "scales": {}}
        self._saved = []
        for L in self.layers:
            t = L["type"]
            xb = blobs[L["bottom"]]
            if t == "Convolution":
                w = f32(P[L["name"] + ".w"])
                b = f32(P[L["name"] + ".b"]) if L["bias"] else None
                y, S = grouped_conv_fwd(xb, w, b, L["G"], L["s"], L["p"])
                self._saved.append((xb,))
                out["scales"][L["name"]] = S
            elif t == "Pooling":
                y, m = capi.pool_fwd(xb, L["method"], L["k"], L["s"], L["p"])
                self._saved.append((xb, m))
                if m is not None:
                    out["masks"][L["name"]] = m
            elif t == "InnerProduct":
                w = f32(P[L["name"] + ".w"])
                b = f32(P[L["name"] + ".b"]) if L["bias"] else None
                y, S = capi.ip_fwd(xb, w, b, want_scale=True)
                y = y.reshape(L["out_shape"])
                self._saved.append((xb,))
                out["scales"][L["name"]] = S.reshape(L["out_shape"])
            elif t == "ReLU":
                y = capi.relu_fwd(xb, L["slope"])
                self._saved.append(None)
            elif t == "Softmax":
                y = capi.softmax_fwd(xb.reshape(xb.shape[0], -1)).reshape(L["out_shape"])
                self._saved.append(None)
            elif t == "SoftmaxWithLoss":
                logits = xb.reshape(xb.shape[0], -1)
                prob, loss, pred = capi.softmax_loss_fwd(logits, labels)
                self._saved.append((prob, np.asarray(labels, np.int32)))
                out["loss"] = loss
                out["prob"] = prob
                out["pred"] = pred
                out["logits"] = logits
                continue
            y = f32(y)
            blobs[L["top"]] = y
            out["blobs"][L["name"]] = y
        # test-phase accuracy on the blobs the chain produced
        out["accuracy"], out["correct"] = {}, {}
        for L in self.accuracy_layers:
            xb = blobs[L["bottom"]]
            acc, correct = capi.accuracy(xb.reshape(xb.shape[0], -1), labels, L["k"])
            out["accuracy"][L["name"]] = acc
            out["correct"][L["name"]] = correct
        self._blobs = blobs
        return out

    # --------------------------------------------------------------- backward
    def backward(self, loss_weight=1.0):
        """Reverse-order backward.  Returns dict with param grads
        (fp64, key name.w / name.b), their scales (key name.w.S ...), and
        blob diffs (fp32-rounded, by layer name = diff w.r.t. its bottom)."""
        P = self.params
        grads, scales, diffs = {}, {}, {}
        d = None
        for L, saved in zip(reversed(self.layers), reversed(self._saved)):
            t = L["type"]
            if t == "SoftmaxWithLoss":
                prob, lab = saved
                d = f32(capi.softmax_loss_bwd(prob, lab, loss_weight)).reshape(L["in_shape"])
            elif t == "InnerProduct":
                (xb,) = saved
                w = f32(P[L["name"] + ".w"])
                dw, db, dx, Sdw, Sdb, Sdx = capi.ip_bwd(d.reshape(d.shape[0], -1), xb, w,
                                                        want_scale=True)
                grads[L["name"] + ".w"], scales[L["name"] + ".w"] = dw, Sdw
                grads[L["name"] + ".b"], scales[L["name"] + ".b"] = db, Sdb
                scales[L["name"] + ".dx"] = Sdx
                d = f32(dx).reshape(L["in_shape"])
            elif t == "ReLU":
                y = self._blobs[L["top"]]
                d = f32(capi.relu_bwd(d, y.reshape(d.shape), L["slope"]))
            elif t == "Softmax":
                pr = self._blobs[L["top"]]
                d = f32(capi.softmax_bwd(pr.reshape(pr.shape[0], -1), d.reshape(d.shape[0], -1))).reshape(L["in_shape"])
            elif t == "Pooling":
                xb, m = saved
                d = f32(capi.pool_bwd(d, m, L["in_shape"], L["method"], L["k"], L["s"], L["p"]))
            elif t == "Convolution":
                (xb,) = saved
                w = f32(P[L["name"] + ".w"])
                first = L["bottom"] == self.input_name
                dw, db, dx, Sdw, Sdb, Sdx = grouped_conv_bwd(d, xb, w, L["G"], L["s"], L["p"], want_dx=not first)
                grads[L["name"] + ".w"], scales[L["name"] + ".w"] = dw, Sdw
                grads[L["name"] + ".b"], scales[L["name"] + ".b"] = db, Sdb
                if not first:
                    scales[L["name"] + ".dx"] = Sdx
                d = None if first else f32(dx)
            diffs[L["name"]] = d
        return {"grads": grads, "scales": scales, "diffs": diffs}

    # ------------------------------------------------------------------ solver
    def sgd_step(self, grads, lr, momentum, decay, history, grad_scale=1.0):
        """Caffe SGD on every learnable blob (fp32, bit-exact contract);
        grads are rounded to fp32 first (they are stored in fp32 diffs)."""
        for k in self.params:
            if k not in history:
                history[k] = np.zeros_like(self.params[k])
            capi.sgd_update_f32(self.params[k], np.asarray(grads[k], np.float32), history[k],
                                lr, momentum, decay, grad_scale)
        return history
