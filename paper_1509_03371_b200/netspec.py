"""Network description: the host-side mirror of netspec.hpp and the size/cost model of
convert.hpp (paths relative to /root/reference/proj/include/pixelseg/).

Pure host code (no device work): parsing, channel propagation, size propagation and the FLOP
model that defines the labels/s roofline. Messages match the reference's text.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from .errors import SizeError, SpecError


class LayerKind(enum.IntEnum):  # netspec.hpp:13
    Data = 0
    ConvSK = 1
    PoolMax = 2
    Relu = 3
    Upconv = 4
    MergeCrop = 5
    SoftmaxLoss = 6


_KIND_NAMES = {
    LayerKind.Data: "data",
    LayerKind.ConvSK: "conv_sk",
    LayerKind.PoolMax: "pool_max",
    LayerKind.Relu: "relu",
    LayerKind.Upconv: "upconv",
    LayerKind.MergeCrop: "mergecrop",
    LayerKind.SoftmaxLoss: "softmax_loss",
}


def kind_name(k: LayerKind) -> str:  # netspec.hpp:15-26
    return _KIND_NAMES.get(k, "?")


def kind_from_name(s: str) -> Optional[LayerKind]:  # netspec.hpp:28-37
    for k, n in _KIND_NAMES.items():
        if n == s:
            return k
    return None


class InitKind(enum.IntEnum):  # netspec.hpp:40
    None_ = 0
    Gaussian = 1
    He = 2


@dataclass
class LayerSpec:  # netspec.hpp:42-56
    name: str = ""
    kind: LayerKind = LayerKind.ConvSK
    k: int = 1
    s: int = 1
    d: int = 1
    p: int = 0
    f_out: int = 0
    inputs: List[str] = field(default_factory=list)
    output: str = ""
    init: InitKind = InitKind.None_
    init_sigma: float = 0.01
    line: int = 0

    def has_weights(self) -> bool:
        return self.kind == LayerKind.ConvSK


@dataclass
class NetSpec:  # netspec.hpp:61-80
    w0: int = 0
    f0: int = 0
    n: int = 1
    layers: List[LayerSpec] = field(default_factory=list)

    def find_layer(self, name: str) -> Optional[LayerSpec]:
        for l in self.layers:
            if l.name == name:
                return l
        return None

    def loss_head(self) -> Optional[LayerSpec]:
        if not self.layers:
            return None
        last = self.layers[-1]
        return last if last.kind == LayerKind.SoftmaxLoss else None


@dataclass
class ParseIssue:
    line: int
    message: str


@dataclass
class ParseResult:
    spec: NetSpec
    issues: List[ParseIssue]

    def ok(self) -> bool:
        return not self.issues

    def issue_text(self) -> str:
        return "".join(f"line {i.line}: {i.message}\n" for i in self.issues)


def _parse_int(s: str) -> Optional[int]:
    try:
        s2 = s.strip()
        if s2 != s or not s:
            return None
        return int(s, 10)
    except ValueError:
        return None


def _parse_double(s: str) -> Optional[float]:
    try:
        if not s or s.strip() != s:
            return None
        return float(s)
    except ValueError:
        return None


def _split_list(s: str) -> List[str]:
    return [t for t in s.split(",") if t]


def parse_netspec(text: str) -> ParseResult:
    """netspec.hpp:180-385: collects every problem with its line number."""
    spec = NetSpec()
    issues: List[ParseIssue] = []

    def issue(line: int, msg: str) -> None:
        issues.append(ParseIssue(line, msg))

    producer_line: Dict[str, int] = {}
    layer_line: Dict[str, int] = {}
    have_input = False
    for lineno, raw in enumerate(text.split("\n"), start=1):
        if "#" in raw:
            raw = raw[: raw.index("#")]
        toks = raw.split()
        if not toks:
            continue
        if toks[0] == "input":
            if have_input:
                issue(lineno, "duplicate input directive (exactly one data layer allowed)")
                continue
            have_input = True
            data = LayerSpec(name="data", kind=LayerKind.Data, output="data", line=lineno)
            saw_w = saw_f = False
            for t in toks[1:]:
                if "=" not in t:
                    issue(lineno, f"expected key=value, got '{t}'")
                    continue
                key, val = t.split("=", 1)
                v = _parse_int(val)
                if v is None:
                    issue(lineno, f"key '{key}' needs an integer, got '{val}'")
                    continue
                if key == "w":
                    spec.w0 = v
                    saw_w = True
                elif key == "f":
                    spec.f0 = v
                    saw_f = True
                elif key == "n":
                    spec.n = v
                else:
                    issue(lineno, f"unknown input key '{key}'")
            if not saw_w or spec.w0 < 1:
                issue(lineno, "input needs w >= 1")
            if not saw_f or spec.f0 < 1:
                issue(lineno, "input needs f >= 1")
            if spec.n < 1:
                issue(lineno, "input n must be >= 1")
            producer_line["data"] = lineno
            spec.layers.append(data)
            continue
        if toks[0] != "layer":
            issue(lineno, f"unknown directive '{toks[0]}'")
            continue
        if len(toks) < 3:
            issue(lineno, "layer needs a name and a kind")
            continue
        l = LayerSpec(name=toks[1], line=lineno)
        kind = kind_from_name(toks[2])
        if kind is None:
            issue(lineno, f"unknown layer kind '{toks[2]}'")
            continue
        if kind == LayerKind.Data:
            issue(lineno, "data layers are declared with the input directive")
            continue
        l.kind = kind
        if kind == LayerKind.Upconv:
            l.k, l.s = 2, 2
        saw_in = saw_out = False
        for t in toks[3:]:
            if "=" not in t:
                issue(lineno, f"expected key=value, got '{t}'")
                continue
            key, val = t.split("=", 1)
            if key == "in":
                l.inputs = _split_list(val)
                saw_in = True
            elif key == "out":
                l.output = val
                saw_out = True
            elif key == "init":
                if val == "he":
                    l.init = InitKind.He
                elif val.startswith("gaussian:"):
                    l.init = InitKind.Gaussian
                    sg = _parse_double(val[9:])
                    if sg is None or sg <= 0:
                        issue(lineno, f"bad gaussian sigma in '{val}'")
                    else:
                        l.init_sigma = sg
                else:
                    issue(lineno, f"unknown init '{val}' (use gaussian:<sigma> or he)")
            else:
                v = _parse_int(val)
                if v is None:
                    issue(lineno, f"key '{key}' needs an integer, got '{val}'")
                    continue
                if key == "k":
                    l.k = v
                elif key == "s":
                    l.s = v
                elif key == "d":
                    l.d = v
                elif key == "p":
                    l.p = v
                elif key == "fout":
                    l.f_out = v
                else:
                    issue(lineno, f"unknown layer key '{key}'")
        if l.name in layer_line:
            issue(lineno, f"duplicate layer name '{l.name}' (first at line {layer_line[l.name]})")
        else:
            layer_line[l.name] = lineno
        if not saw_in or not l.inputs:
            issue(lineno, "layer needs in=<blob[,blob]>")
        if not saw_out or not l.output:
            issue(lineno, "layer needs out=<blob>")
        want = 2 if l.kind == LayerKind.MergeCrop else 1
        if saw_in and len(l.inputs) != want:
            issue(lineno, f"{kind_name(l.kind)} takes {want} input(s), got {len(l.inputs)}")
        for b in l.inputs:
            if b not in producer_line:
                issue(lineno, f"input blob '{b}' is not produced by any earlier layer "
                              "(dangling or cyclic reference)")
        if saw_out and l.output:
            if l.output in producer_line:
                issue(lineno, f"blob '{l.output}' already produced at line {producer_line[l.output]}")
            else:
                producer_line[l.output] = lineno
        if l.k < 1 or l.s < 1 or l.d < 1:
            issue(lineno, "k, s, d must all be >= 1")
        if l.p != 0:
            issue(lineno, "padding p must be 0 in network specs")
        if l.kind == LayerKind.ConvSK:
            if l.f_out < 1:
                issue(lineno, "conv_sk needs fout >= 1")
            if l.s != 1:
                issue(lineno, "conv_sk stride must be 1")
        elif l.kind == LayerKind.PoolMax:
            if l.s != 1 and l.s != l.k:
                issue(lineno, "pool_max stride must be 1 (strided-kernel) or equal k (downsampling)")
            if l.s == l.k and l.k > 1 and l.d != 1:
                issue(lineno, "downsampling pool_max requires d=1")
            if l.f_out != 0:
                issue(lineno, "pool_max cannot change channel count")
        elif l.kind in (LayerKind.Relu, LayerKind.SoftmaxLoss):
            if l.k != 1 or l.s != 1 or l.d != 1:
                issue(lineno, f"{kind_name(l.kind)} is elementwise: k=s=d=1")
            if l.f_out != 0:
                issue(lineno, f"{kind_name(l.kind)} cannot set fout")
        elif l.kind == LayerKind.Upconv:
            if l.k != 2 or l.s != 2:
                issue(lineno, "upconv is a fixed 2x resize: k=2 s=2")
            if l.d != 1:
                issue(lineno, "upconv requires d=1")
        elif l.kind == LayerKind.MergeCrop:
            if l.k != 1 or l.s != 1 or l.d != 1:
                issue(lineno, "mergecrop is parameterless: k=s=d=1")
            if l.f_out != 0:
                issue(lineno, "mergecrop cannot set fout (channels concatenate)")
        if l.init != InitKind.None_ and l.kind != LayerKind.ConvSK:
            issue(lineno, "init applies only to conv_sk layers")
        if l.d > 1 and l.kind not in (LayerKind.ConvSK, LayerKind.PoolMax):
            issue(lineno, "kernel stride d > 1 only applies to conv_sk and pool_max")
        spec.layers.append(l)
    if not have_input:
        issue(0, "missing input directive")
    return ParseResult(spec, issues)


def parse_netspec_or_throw(text: str) -> NetSpec:  # netspec.hpp:419-423
    r = parse_netspec(text)
    if not r.ok():
        raise SpecError("network spec errors:\n" + r.issue_text())
    return r.spec


def load_netspec(path: str) -> NetSpec:
    with open(path, "r") as f:
        return parse_netspec_or_throw(f.read())


def compute_channels(spec: NetSpec) -> Dict[str, int]:  # netspec.hpp:143-160
    f: Dict[str, int] = {}
    for l in spec.layers:
        if l.kind == LayerKind.Data:
            fin = spec.f0
        elif l.kind == LayerKind.MergeCrop:
            fin = f[l.inputs[0]] + f[l.inputs[1]]
        else:
            fin = f[l.inputs[0]]
        fout = l.f_out if (l.kind == LayerKind.ConvSK and l.f_out > 0) else fin
        f[l.output] = fout
    return f


def out_extent(in_: int, k: int, d: int, s: int, p: int, what: str) -> int:
    """ConvGeometry::out_extent (tensor.hpp:26-42)."""
    span = (k - 1) * d + 1
    if k < 1 or d < 1 or s < 1 or p < 0:
        raise SizeError(f"{what}: require k,d,s >= 1 and p >= 0")
    padded = in_ + 2 * p
    if span > padded:
        raise SizeError(f"{what}: kernel span {span} exceeds padded input {padded}")
    num = padded - span
    if num % s != 0:
        raise SizeError(f"{what}: input {in_} with span {span} not divisible by stride {s}")
    return num // s + 1


@dataclass
class SizeRow:  # convert.hpp:20-27
    name: str
    kind: LayerKind
    k: int = 1
    s: int = 1
    d: int = 1
    f_in: int = 0
    f_out: int = 0
    w_in: int = 0
    w_out: int = 0


def propagate_sizes(spec: NetSpec, w0: int) -> List[SizeRow]:  # convert.hpp:32-91
    if w0 < 1:
        raise SizeError("propagate_sizes: w0 must be >= 1")
    channels = compute_channels(spec)
    width: Dict[str, int] = {}
    table: List[SizeRow] = []
    for l in spec.layers:
        row = SizeRow(l.name, l.kind, l.k, l.s, l.d, f_out=channels[l.output])
        if l.kind == LayerKind.Data:
            w_in = w0
            row.f_in = spec.f0
        else:
            w_in = width[l.inputs[0]]
            row.f_in = sum(channels[b] for b in l.inputs)
        row.w_in = w_in
        try:
            if l.kind == LayerKind.Data:
                w_out = w0
            elif l.kind in (LayerKind.ConvSK, LayerKind.PoolMax):
                w_out = out_extent(w_in, l.k, l.d, l.s, l.p, "extent")
            elif l.kind == LayerKind.Upconv:
                w_out = 2 * w_in
            elif l.kind == LayerKind.MergeCrop:
                wa, wb = width[l.inputs[0]], width[l.inputs[1]]
                if wb < wa:
                    raise SizeError(f"second input ({wb}) smaller than first ({wa})")
                w_out = wa
            else:
                w_out = w_in
        except SpecError as e:
            raise SizeError(f"layer '{l.name}': {e}") from None
        row.w_out = w_out
        width[l.output] = w_out
        table.append(row)
    return table


def output_extent(spec: NetSpec, w0: int) -> int:  # convert.hpp:93-95
    return propagate_sizes(spec, w0)[-1].w_out


def flop_estimate(spec: NetSpec, w0: int) -> Dict[str, int]:
    """convert.hpp:308-322: per conv layer f_out * w_out^2 * (2*f_in*k^2 - 1); key 'total'."""
    rows = {}
    total = 0
    for r in propagate_sizes(spec, w0):
        if r.kind != LayerKind.ConvSK:
            continue
        fl = r.f_out * r.w_out * r.w_out * (2 * r.f_in * r.k * r.k - 1)
        rows[r.name] = fl
        total += fl
    rows["total"] = total
    return rows
