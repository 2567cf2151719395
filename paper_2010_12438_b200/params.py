"""Parameters: a ParamStore mirroring the reference's (tensor.py:391-465), its
initialiser (embedding.py:35-44, policy.py:44-94, 322-330: same names, shapes and
numpy draw order), and the packed float32 device blob the kernels read.

Slot order of the device blob (go_param_slots, must match csrc/engine.cu Slots):
  embed/in_w, embed/in_b, then per layer l: agg_w{l}, agg_b{l}, fc_w{l}, fc_b{l};
  policy/in_w, policy/in_b; per block b in block0..block{L-1}, mod:
  attn_{q,k,v,o}_{w,b} (interleaved w,b), ln1_g, ln1_b, ff_w1, ff_b1, ff_w2, ff_b2,
  ln2_g, ln2_b; task_attn/{q,k,v,o}_{w,b}; per task (canonical order): cat_w, cat_b,
  ln_g, ln_b, fc_w1, fc_b1, fc_w2, fc_b2, out_w, out_b; value_w, value_b.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

from .config import EmbedConfig, PolicyConfig, ordered_tasks
from .graph import feature_dim


class Param:
    __slots__ = ("data", "grad")

    def __init__(self, data):
        self.data = np.array(data, dtype=np.float64)
        self.grad = None

    @property
    def shape(self):
        return self.data.shape


class ParamStore:
    """Named float64 parameters with Adam moment state (tensor.py:391-465).
    `version` counts bulk updates (informational: the device cache compares packed
    contents, DeviceParams)."""

    def __init__(self):
        self._params: dict[str, Param] = {}
        self._m: dict[str, np.ndarray] = {}
        self._v: dict[str, np.ndarray] = {}
        self.step_count = 0
        self.version = 0

    def add(self, name, data) -> Param:
        if name in self._params:
            raise KeyError(f"parameter {name!r} already exists")
        p = Param(data)
        self._params[name] = p
        self._m[name] = np.zeros_like(p.data)
        self._v[name] = np.zeros_like(p.data)
        self.version += 1
        return p

    def __getitem__(self, name) -> Param:
        return self._params[name]

    def __contains__(self, name) -> bool:
        return name in self._params

    def names(self) -> list[str]:
        return sorted(self._params)

    def items(self):
        return [(n, self._params[n]) for n in self.names()]

    def num_values(self, prefix: str = "") -> int:
        return sum(p.data.size for n, p in self.items() if n.startswith(prefix))

    def touch(self):
        """Kept for callers of the round-1 API; not needed for coherence (DeviceParams
        compares contents)."""
        self.version += 1

    def zero_grads(self):
        for p in self._params.values():
            p.grad = None

    def adam_step(self, lr: float, beta1=0.9, beta2=0.999, eps=1e-8):
        """Host float64 Adam (tensor.py:428-441); the device PPO path uses the fused
        kernel instead and writes the result back here."""
        self.step_count += 1
        t = self.step_count
        for name in self.names():
            p = self._params[name]
            g = p.grad if p.grad is not None else np.zeros_like(p.data)
            self._m[name] = beta1 * self._m[name] + (1 - beta1) * g
            self._v[name] = beta2 * self._v[name] + (1 - beta2) * g * g
            mhat = self._m[name] / (1 - beta1**t)
            vhat = self._v[name] / (1 - beta2**t)
            p.data = p.data - lr * mhat / (np.sqrt(vhat) + eps)
            p.grad = None
        self.version += 1

    def clone(self) -> "ParamStore":
        other = ParamStore()
        for name, p in self.items():
            other.add(name, p.data.copy())
            other._m[name] = self._m[name].copy()
            other._v[name] = self._v[name].copy()
        other.step_count = self.step_count
        return other

    def copy_values_from(self, other):
        for name, p in other.items():
            self._params[name].data = np.array(p.data, dtype=np.float64, copy=True)
        self.version += 1

    def save(self, path):
        np.savez(path, **{n: p.data for n, p in self.items()})

    def load(self, path):
        with np.load(path) as data:
            for name in data.files:
                if name.startswith(("__adam_m__/", "__adam_v__/")) or name == "__adam_step__":
                    continue
                if name in self._params:
                    self._params[name].data = np.array(data[name], dtype=np.float64)
                else:
                    self.add(name, data[name])
        self.version += 1

    # Checkpoint WITH the optimiser state.  The reference's save()
    # writes parameter values only (tensor.py:456-458), so a resumed reference run
    # restarts Adam from zero.  save_state() writes the same value arrays under the
    # same names plus "__adam_m__/<name>", "__adam_v__/<name>" and "__adam_step__";
    # load() above (the reference's semantics) skips those reserved keys, so either
    # loader reads either file.  Hand a reference store the plain save() file.
    _M, _V, _STEP = "__adam_m__/", "__adam_v__/", "__adam_step__"

    def save_state(self, path):
        arrs = {n: p.data for n, p in self.items()}
        for n in self.names():
            arrs[self._M + n] = self._m[n]
            arrs[self._V + n] = self._v[n]
        arrs[self._STEP] = np.array(self.step_count, np.int64)
        np.savez(path, **arrs)

    def load_state(self, path):
        with np.load(path) as data:
            files = set(data.files)
            for name in data.files:
                if name.startswith((self._M, self._V)) or name == self._STEP:
                    continue
                if name in self._params:
                    self._params[name].data = np.array(data[name], dtype=np.float64)
                else:
                    self.add(name, data[name])
            for name in self.names():
                shape = self._params[name].data.shape
                for key, dst in ((self._M + name, self._m), (self._V + name, self._v)):
                    if key in files:
                        a = np.array(data[key], dtype=np.float64)
                        if a.shape != shape:
                            raise ValueError(f"{key}: shape {a.shape} != parameter {shape}")
                        dst[name] = a
            if self._STEP in files:
                self.step_count = int(data[self._STEP])
        self.version += 1


def _uniform(rng, shape, fan_in):
    s = 1.0 / np.sqrt(max(1, fan_in))
    return rng.uniform(-s, s, size=shape)


def init_all_params(embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict,
                    seed: int) -> ParamStore:
    """policy.py:322-330 (+ embedding.py:35-44, policy.py:44-94), same draw order."""
    rng = np.random.default_rng(seed)
    store = ParamStore()
    tasks = ordered_tasks(task_sizes)
    fdim = feature_dim([a for _, a in tasks])
    d = embed_cfg.gs_dim
    store.add("embed/in_w", _uniform(rng, (fdim, d), fdim))
    store.add("embed/in_b", np.zeros(d))
    for l in range(embed_cfg.gs_layers):
        store.add(f"embed/agg_w{l}", _uniform(rng, (d, d), d))
        store.add(f"embed/agg_b{l}", np.zeros(d))
        store.add(f"embed/fc_w{l}", _uniform(rng, (2 * d, d), 2 * d))
        store.add(f"embed/fc_b{l}", np.zeros(d))
    dm, w, di = cfg.d_model, cfg.attn_width, cfg.d_inner

    def attn(prefix):
        for nm in ("q", "k", "v"):
            store.add(f"{prefix}{nm}_w", _uniform(rng, (dm, w), dm))
            store.add(f"{prefix}{nm}_b", np.zeros(w))
        store.add(f"{prefix}o_w", _uniform(rng, (w, dm), w))
        store.add(f"{prefix}o_b", np.zeros(dm))

    def block(prefix):
        attn(prefix + "attn_")
        store.add(prefix + "ln1_g", np.ones(dm))
        store.add(prefix + "ln1_b", np.zeros(dm))
        store.add(prefix + "ff_w1", _uniform(rng, (dm, di), dm))
        store.add(prefix + "ff_b1", np.zeros(di))
        store.add(prefix + "ff_w2", _uniform(rng, (di, dm), di))
        store.add(prefix + "ff_b2", np.zeros(dm))
        store.add(prefix + "ln2_g", np.ones(dm))
        store.add(prefix + "ln2_b", np.zeros(dm))

    store.add("policy/in_w", _uniform(rng, (d, dm), d))
    store.add("policy/in_b", np.zeros(dm))
    for l in range(cfg.trf_layers):
        block(f"policy/block{l}/")
    block("policy/mod/")
    attn("policy/task_attn/")
    for task, a in tasks:
        p = f"policy/task/{task}/"
        store.add(p + "cat_w", _uniform(rng, (2 * dm, dm), 2 * dm))
        store.add(p + "cat_b", np.zeros(dm))
        store.add(p + "ln_g", np.ones(dm))
        store.add(p + "ln_b", np.zeros(dm))
        store.add(p + "fc_w1", _uniform(rng, (dm, di), dm))
        store.add(p + "fc_b1", np.zeros(di))
        store.add(p + "fc_w2", _uniform(rng, (di, dm), di))
        store.add(p + "fc_b2", np.zeros(dm))
        store.add(p + "out_w", np.zeros((dm, a)))
        store.add(p + "out_b", np.zeros(a))
    store.add("policy/value_w", np.zeros((dm, 1)))
    store.add("policy/value_b", np.zeros(1))
    return store


def randomize_zero_init(store, seed: int = 1):
    """Benchmark weights: refill every all-zero tensor with
    Uniform(+-1/sqrt(shape[0])) from default_rng(seed), names in sorted order, so the
    synthetic policy has O(1) logits instead of the reference's zero-init heads."""
    rng = np.random.default_rng(seed)
    for name in sorted(n for n, _ in store.items()):
        p = store[name]
        if not np.any(p.data):
            p.data = _uniform(rng, p.data.shape, p.data.shape[0])
    if hasattr(store, "touch"):
        store.touch()
    return store


def slot_names(embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict) -> list[str]:
    names = ["embed/in_w", "embed/in_b"]
    for l in range(embed_cfg.gs_layers):
        names += [f"embed/agg_w{l}", f"embed/agg_b{l}", f"embed/fc_w{l}", f"embed/fc_b{l}"]
    names += ["policy/in_w", "policy/in_b"]
    attn = [f"attn_{x}_{y}" for x in "qkvo" for y in "wb"]
    blk = attn + ["ln1_g", "ln1_b", "ff_w1", "ff_b1", "ff_w2", "ff_b2", "ln2_g", "ln2_b"]
    for b in [f"block{l}" for l in range(cfg.trf_layers)] + ["mod"]:
        names += [f"policy/{b}/{x}" for x in blk]
    names += [f"policy/task_attn/{x}_{y}" for x in "qkvo" for y in "wb"]
    for task, _a in ordered_tasks(task_sizes):
        names += [f"policy/task/{task}/{x}" for x in
                  ("cat_w", "cat_b", "ln_g", "ln_b", "fc_w1", "fc_b1", "fc_w2", "fc_b2",
                   "out_w", "out_b")]
    names += ["policy/value_w", "policy/value_b"]
    return names


def _get(store, name):
    # stages read only their own slots, so a partial store (e.g. embed-only, like
    # the reference's init_embed_params) packs missing tensors as empty
    if name not in store:
        return np.zeros(0, np.float32)
    if isinstance(store, dict):
        v = store[name]
        return np.asarray(getattr(v, "data", v))
    return np.asarray(store[name].data)


def pack(store, embed_cfg, cfg, task_sizes, dtype=np.float32):
    """Host blob (float32 by default; 16-byte aligned tensors in float32 units) + int64
    offsets in slot order.  dtype=float64 gives the optimiser's master copy with the
    same offsets."""
    names = slot_names(embed_cfg, cfg, task_sizes)
    arrays = [np.ascontiguousarray(_get(store, n), dtype=dtype).reshape(-1) for n in names]
    offs = np.zeros(len(names), np.int64)
    pos = 0
    for i, a in enumerate(arrays):
        offs[i] = pos
        pos += (a.size + 3) // 4 * 4
    blob = np.zeros(max(pos, 4), dtype)
    for o, a in zip(offs, arrays):
        blob[o:o + a.size] = a
    return blob, offs


class DeviceParams:
    """float32 device copy of a store.

    Every call re-packs the store on the host (~3-5 ms for the 1.5M-parameter joint
    network) and compares the packed blob with the one last uploaded; the device copy
    is reused only when the bytes are identical.  So in-place edits
    (`store[name].data[:] = x`, which the reference's own tests do between calls,
    reference pkg/tests/test_policy.py:212), reassignments, foreign stores without a version and
    a new store that happens to reuse a freed store's id() can never be served stale
    weights."""

    def __init__(self):
        self._key = None
        self._host = None
        self.blob = None
        self.offsets = None

    def get(self, store, embed_cfg, cfg, task_sizes, device):
        import torch
        blob, offs = pack(store, embed_cfg, cfg, task_sizes)
        key = (embed_cfg, cfg, tuple(ordered_tasks(task_sizes)), str(device))
        if (key != self._key or self._host is None or self._host.shape != blob.shape
                or not np.array_equal(self.offsets, offs)
                or not np.array_equal(self._host, blob)):
            self.blob = torch.from_numpy(blob).to(device, non_blocking=False)
            self.offsets = offs
            self._host = blob
            self._key = key
        return self.blob, self.offsets
