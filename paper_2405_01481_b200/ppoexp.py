"""Python host mirror of the reference's experience-path interfaces over the
C ABI (include/ppoexp.h, libppoexp.so).

Names follow the reference (/root/reference/proj/include/aligner/*.hpp):
``ModelConfig``, ``SamplingSpec``, ``GenTask``, ``GenerateResult``,
``build_engine`` / ``Engine.refit`` / ``Engine.generate_batch``,
``sequence_logprobs``, ``value_estimates``, ``reward_head``,
``kl_penalized_rewards``, ``gae``, ``RolloutSeq`` and the experience half of
``ppo_step`` (``make_experience``).  Errors raise the reference's exception
types with its message wording.

There is no CPU fallback: importing works anywhere, but every call needs the
CUDA library and a device, and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libppoexp.so")

HOST, DEVICE = 0, 1
F32, BF16, F64, MIXED = 0, 1, 2, 3  # MIXED: bf16 weights, fp32-grade activations (include/ppoexp.h)
PAD_TOKEN, EOT_TOKEN = 256, 257  # include/aligner/model.hpp:17-18


# ---------------------------------------------------------------- errors
class ShapeError(RuntimeError):
    pass


class IndexError_(IndexError):
    pass


class ContractError(RuntimeError):
    pass


class RefitError(RuntimeError):
    pass


class PpoError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRS = {1: ContractError, 2: IndexError_, 3: ShapeError, 4: RefitError, 5: PpoError, 6: CudaError, 7: MemoryError}


# ---------------------------------------------------------------- ctypes
class _Cfg(C.Structure):
    _fields_ = [("vocab_size", C.c_int64), ("d_model", C.c_int64), ("n_layers", C.c_int64), ("n_heads", C.c_int64),
                ("d_ff", C.c_int64), ("max_seq_len", C.c_int64), ("scalar_head", C.c_int32), ("reserved", C.c_int32)]


class _View(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rank", C.c_int32), ("dtype", C.c_int32), ("shape", C.c_int64 * 2),
                ("data", C.c_void_p), ("where", C.c_int32), ("reserved", C.c_int32)]


class _Sampling(C.Structure):
    _fields_ = [("greedy", C.c_int32), ("top_k", C.c_int32), ("temperature", C.c_double), ("top_p", C.c_double)]


class _EngineOpts(C.Structure):
    _fields_ = [("max_batch", C.c_int64), ("page_size", C.c_int64), ("max_total_tokens", C.c_int64),
                ("use_graphs", C.c_int32), ("reserved", C.c_int32)]


_ALLREDUCE = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class _Hyper(C.Structure):
    _fields_ = [("kl_penalty_coef", C.c_double), ("gamma", C.c_double), ("lam", C.c_double)]


class _XpReq(C.Structure):
    _fields_ = [("policy_engine", C.c_void_p), ("reference", C.c_void_p), ("critic", C.c_void_p), ("rm", C.c_void_p),
                ("scripted_target", C.c_int32), ("reserved", C.c_int32), ("sampling", _Sampling),
                ("seed", C.c_uint64), ("step_index", C.c_int64), ("gidx0", C.c_int64), ("max_new", C.c_int64),
                ("hyper", _Hyper), ("allreduce", _ALLREDUCE), ("allreduce_user", C.c_void_p), ("comm", C.c_void_p)]


class _Rollout(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("tokens", "lengths", "actor_lp", "ref_lp", "values", "rewards", "shaped",
                                          "advantages", "returns", "whitened", "stats", "timing")]


_lib = None


def lib():
    """Loads libppoexp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"{LIB_PATH} missing: run paper_2405_01481_b200.build.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I64, I32, D, V = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.ppoexp_last_error.restype = C.c_char_p
        sigs = {
            "ppoexp_abi_version": [],
            "ppoexp_ctx_create": [I32, P],
            "ppoexp_ctx_destroy": [P],
            "ppoexp_ctx_stream": [P, P],
            "ppoexp_ctx_synchronize": [P],
            "ppoexp_ctx_profile": [P, I32],
            "ppoexp_ctx_profile_filter": [P, C.c_char_p],
            "ppoexp_ctx_profile_query": [P, C.c_char_p, P, P, P, P],
            "ppoexp_ctx_launch_count": [P, P],
            "ppoexp_model_create": [P, P, P, I64, I32, P],
            "ppoexp_model_refit": [P, P, I64],
            "ppoexp_model_generation": [P, P],
            "ppoexp_model_config_get": [P, P],
            "ppoexp_model_destroy": [P],
            "ppoexp_engine_create": [P, P, P],
            "ppoexp_engine_destroy": [P],
            "ppoexp_engine_generate": [P, I64, P, P, P, P, P, I64, P, P, P, I32, P],
            "ppoexp_sequence_logprobs": [P, I64, P, P, P, I32],
            "ppoexp_value_estimates": [P, I64, P, P, P, P, I32],
            "ppoexp_response_logprob_sums": [P, I64, P, P, P, P, I32],
            "ppoexp_reward_head": [P, I64, P, P, P, I32],
            "ppoexp_shape_gae": [I64, I64, P, P, P, P, P, D, D, D, P, P, P, P, I32],
            "ppoexp_whiten_partials": [I64, I64, P, P, P, P, I32],
            "ppoexp_whiten_apply": [I64, I64, P, P, P, P, P, I32],
            "ppoexp_make_experience": [P, I64, P, P, P, I32],
            "ppoexp_model_snapshot": [P, C.c_char_p, P, I64, I32],
            "ppoexp_engine_build_seconds": [P, P],
            "ppoexp_engine_cost": [P, C.c_char_p, P],
            "ppoexp_engine_options_get": [P, P],
            "ppoexp_balance": [P, I64, I64, P],
            "ppoexp_comm_unique_id": [P],
            "ppoexp_comm_create": [P, P, I32, I32, P],
            "ppoexp_comm_destroy": [P],
            "ppoexp_comm_allgather_sum": [P, P, I64, I32],
            "ppoexp_trainer_create": [P, P, P, I64, P, P, P],
            "ppoexp_trainer_destroy": [P],
            "ppoexp_trainer_ppo_actor_step": [P, I64, P, P, P, P, P, P, D, D, P, I32],
            "ppoexp_trainer_critic_step": [P, I64, P, P, P, P, P, D, D, P, I32],
            "ppoexp_trainer_dpo_step": [P, P, I64, P, P, P, I32, D, D, D, P, P, I32],
            "ppoexp_trainer_refit": [P],
            "ppoexp_trainer_get": [P, C.c_char_p, P, I64],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int32
        _lib = L
    return _lib


def _check(rc):
    if rc:
        msg = lib().ppoexp_last_error().decode(errors="replace")
        raise _ERRS.get(rc, CudaError)(msg)


def _ptr(a):
    """(address, where) for a numpy array or a CUDA torch tensor."""
    if a is None:
        return None, HOST
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        return a.data_ptr(), DEVICE
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data, HOST
    raise TypeError(type(a))


# ---------------------------------------------------------------- config
@dataclass
class ModelConfig:
    """include/aligner/model.hpp:30-45"""
    vocab_size: int = 258
    d_model: int = 64
    n_layers: int = 2
    n_heads: int = 4
    d_ff: int = 256
    max_seq_len: int = 128
    scalar_head: bool = False

    def head_dim(self):
        return self.d_model // self.n_heads

    def _c(self):
        return _Cfg(self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.d_ff, self.max_seq_len,
                    1 if self.scalar_head else 0, 0)

    def with_head(self, on=True):
        return ModelConfig(self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.d_ff, self.max_seq_len, on)


def expected_names(cfg: ModelConfig):
    """ModelParams::expected_names + param_shape (src/model.cpp:66-115)."""
    d, f = cfg.d_model, cfg.d_ff
    out = [("tok_embed.weight", (cfg.vocab_size, d)), ("pos_embed.weight", (cfg.max_seq_len, d))]
    for i in range(cfg.n_layers):
        b = f"layers.{i}."
        out += [(b + "attn_norm.weight", (d,)), (b + "attn_norm.bias", (d,))]
        out += [(b + f"attn.{p}.weight", (d, d)) for p in ("q_proj", "k_proj", "v_proj", "o_proj")]
        out += [(b + "ffn_norm.weight", (d,)), (b + "ffn_norm.bias", (d,)), (b + "ffn.up_proj.weight", (d, f)),
                (b + "ffn.down_proj.weight", (f, d))]
    out += [("final_norm.weight", (d,)), ("final_norm.bias", (d,))]
    if cfg.scalar_head:
        out.append(("scalar_head.weight", (d, 1)))
    return out


def flat_to_params(cfg: ModelConfig, flat: np.ndarray) -> dict:
    """Splits a flat canonical buffer into {name: array} (views, no copy)."""
    total = sum(int(np.prod(s)) for _, s in expected_names(cfg))
    if total != flat.size:
        raise ShapeError(f"flat parameter buffer has {flat.size} values, config implies {total}")
    out, off = {}, 0
    for name, shape in expected_names(cfg):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    if off != flat.size:
        raise ShapeError(f"flat parameter buffer has {flat.size} values, config implies {off}")
    return out


def _views(params: dict):
    keep, views = [], (_View * len(params))()
    for i, (name, arr) in enumerate(params.items()):
        if hasattr(arr, "data_ptr"):
            import torch
            dt = {torch.float64: F64, torch.float32: F32, torch.bfloat16: BF16}[arr.dtype]
            arr = arr.contiguous()
            addr, where = _ptr(arr)
            shape = tuple(arr.shape)
        else:
            if arr.dtype == np.float64:
                dt = F64
            elif arr.dtype == np.float32:
                dt = F32
            elif arr.dtype == np.uint16:  # raw bf16 bits
                dt = BF16
            else:
                arr = arr.astype(np.float64)
                dt = F64
            arr = np.ascontiguousarray(arr)
            addr, where = arr.ctypes.data, HOST
            shape = arr.shape
        keep.append(arr)
        nb = name.encode()
        keep.append(nb)
        views[i].name = nb
        views[i].rank = len(shape)
        views[i].dtype = dt
        views[i].shape[0] = shape[0] if len(shape) > 0 else 1
        views[i].shape[1] = shape[1] if len(shape) > 1 else 0
        views[i].data = addr
        views[i].where = where
    return views, keep


# ---------------------------------------------------------------- runtime
class Context:
    """One device + stream (include/ppoexp.h ppoexp_ctx)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(lib().ppoexp_ctx_create(device, C.byref(self.h)))
        self.device = device
        self._children = weakref.WeakSet()  # engines / models / communicators on this context

    def _adopt(self, obj):
        self._children.add(obj)

    def close(self):
        """Destroys the context; library objects still open on it are closed
        first (engines before models), so no handle outlives its context."""
        if self.h:
            kids = list(self._children)
            for kind in (Engine, Communicator, Trainer, DeviceModel):
                for k in kids:
                    if isinstance(k, kind):
                        k.close()
            _check(lib().ppoexp_ctx_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().ppoexp_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        _check(lib().ppoexp_ctx_synchronize(self.h))

    def profile(self, enable=True):
        _check(lib().ppoexp_ctx_profile(self.h, 1 if enable else 0))

    def profile_filter(self, classes=None):
        """Profile only these kernel classes (None = all)."""
        _check(lib().ppoexp_ctx_profile_filter(self.h, ",".join(classes).encode() if classes else None))

    def profile_query(self, cls: str):
        ms, n, b, f = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(lib().ppoexp_ctx_profile_query(self.h, cls.encode(), C.byref(ms), C.byref(n), C.byref(b), C.byref(f)))
        return dict(ms=ms.value, launches=n.value, bytes=b.value, flops=f.value)

    @property
    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().ppoexp_ctx_launch_count(self.h, C.byref(n)))
        return n.value


class DeviceModel:
    """A device-resident ModelParams snapshot (build = deep copy, src/engine.cpp:33-48)."""

    def __init__(self, ctx: Context, config: ModelConfig, params, dtype: int = MIXED):
        if isinstance(params, np.ndarray):
            try:
                params = flat_to_params(config, params)
            except (ShapeError, ValueError):
                params = {}  # the library reports the config / name-set error
        self.ctx, self.config, self.dtype = ctx, config, dtype
        self.h = C.c_void_p()
        views, keep = _views(params)
        cfg = config._c()
        _check(lib().ppoexp_model_create(ctx.h, C.byref(cfg), views, len(params), dtype, C.byref(self.h)))
        ctx._adopt(self)

    def refit(self, params):
        """Engine::refit, src/engine.cpp:60-90 (RefitError, nothing touched, on a name/shape mismatch)."""
        if isinstance(params, np.ndarray):
            try:
                params = flat_to_params(self.config, params)
            except ShapeError as e:
                raise RefitError(f"refit: {e} (rebuild required)")
        views, keep = _views(params)
        _check(lib().ppoexp_model_refit(self.h, views, len(params)))

    @property
    def generation_counter(self) -> int:
        g = C.c_uint64()
        _check(lib().ppoexp_model_generation(self.h, C.byref(g)))
        return g.value

    def snapshot(self, name: str | None = None, dtype=F64):
        """Engine::snapshot (include/aligner/engine.hpp:67): the device copy in the
        reference layout — one parameter, or the whole {name: array} map."""
        if name is None:
            return {n: self.snapshot(n, dtype) for n, _ in expected_names(self.config)}
        shape = dict(expected_names(self.config))[name]
        out = np.zeros(shape, np.float64 if dtype == F64 else np.float32)
        _check(lib().ppoexp_model_snapshot(self.h, name.encode(), out.ctypes.data, out.size, dtype))
        return out

    def close(self):
        if self.h:
            _check(lib().ppoexp_model_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- engine
@dataclass
class SamplingSpec:
    """include/aligner/model.hpp:75-84 (+ top_k / top_p, north-star)."""
    greedy: bool = True
    temperature: float = 1.0
    seed: int = 0
    top_k: int = 0
    top_p: float = 1.0

    @staticmethod
    def greedy_spec():
        return SamplingSpec()

    @staticmethod
    def temperature_spec(tau: float, seed: int, top_k: int = 0, top_p: float = 1.0):
        return SamplingSpec(False, tau, seed, top_k, top_p)


@dataclass
class GenTask:
    """include/aligner/engine.hpp:23-31"""
    prompt: Sequence[int]
    max_new: int = 16
    sampling: SamplingSpec = field(default_factory=SamplingSpec)
    estimated_cost: float = 0.0

    def cost(self):
        return self.estimated_cost if self.estimated_cost > 0 else float(self.max_new)


@dataclass
class GenerateResult:
    """include/aligner/model.hpp:86-89"""
    tokens: np.ndarray
    logprobs: np.ndarray


@dataclass
class EngineOptions:
    max_batch: int = 256
    page_size: int = 64
    max_total_tokens: int = 0
    use_graphs: bool = True


def ragged(seqs):
    offs = np.zeros(len(seqs) + 1, np.int64)
    offs[1:] = np.cumsum([len(s) for s in seqs])
    flat = np.concatenate([np.asarray(s, np.int32) for s in seqs]) if len(seqs) else np.zeros(0, np.int32)
    return np.ascontiguousarray(flat, np.int32), offs


class Engine:
    """The TensorRT-LLM analog (include/aligner/engine.hpp:49-92) on one B200."""

    def __init__(self, model: DeviceModel, opts: EngineOptions | None = None):
        opts = opts or EngineOptions()
        self.model = model
        o = _EngineOpts(opts.max_batch, opts.page_size, opts.max_total_tokens, 1 if opts.use_graphs else 0, 0)
        self.h = C.c_void_p()
        _check(lib().ppoexp_engine_create(model.h, C.byref(o), C.byref(self.h)))
        self.last_ms = 0.0
        model.ctx._adopt(self)

    def refit(self, params):
        self.model.refit(params)

    @property
    def generation_counter(self):
        return self.model.generation_counter

    def build_seconds(self) -> float:
        """Engine::build_seconds (include/aligner/engine.hpp:66)."""
        v = C.c_double()
        _check(lib().ppoexp_engine_build_seconds(self.h, C.byref(v)))
        return v.value

    def costs(self) -> dict:
        """Engine::costs() (CostBook totals in seconds, include/aligner/timing.hpp:33-46)."""
        out = {}
        for cat in ("response_generation", "refit"):
            v = C.c_double()
            _check(lib().ppoexp_engine_cost(self.h, cat.encode(), C.byref(v)))
            if v.value:
                out[cat] = v.value
        return out

    def snapshot(self):
        """Engine::snapshot(): the frozen weights in the reference layout."""
        return self.model.snapshot()

    def options(self) -> EngineOptions:
        o = _EngineOpts()
        _check(lib().ppoexp_engine_options_get(self.h, C.byref(o)))
        return EngineOptions(o.max_batch, o.page_size, o.max_total_tokens, bool(o.use_graphs))

    def generate_batch(self, tasks: Sequence[GenTask]):
        """Engine::generate_batch, src/engine.cpp:148-182 (per-task SamplingSpec)."""
        if not tasks:
            return []
        flat, offs = ragged([t.prompt for t in tasks])
        mx = np.array([t.max_new for t in tasks], np.int64)
        seeds = np.array([t.sampling.seed for t in tasks], np.uint64)
        stride = max(1, int(mx.max()))
        B = len(tasks)
        toks = np.zeros((B, stride), np.int32)
        lps = np.zeros((B, stride), np.float64)
        lens = np.zeros(B, np.int64)
        sp = (_Sampling * B)(*[_Sampling(1 if t.sampling.greedy else 0, t.sampling.top_k, t.sampling.temperature,
                                          t.sampling.top_p) for t in tasks])
        ms = C.c_double()
        _check(lib().ppoexp_engine_generate(self.h, B, flat.ctypes.data, offs.ctypes.data, mx.ctypes.data,
                                            sp, seeds.ctypes.data, stride, toks.ctypes.data,
                                            lps.ctypes.data, lens.ctypes.data, HOST, C.byref(ms)))
        self.last_ms = ms.value
        return [GenerateResult(toks[b, :lens[b]].copy(), lps[b, :lens[b]].copy()) for b in range(B)]

    def close(self):
        if self.h:
            _check(lib().ppoexp_engine_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def balance(tasks_or_costs, n_workers: int):
    """balance (src/engine.cpp:14-31): LPT assignment; returns task indices per
    worker (tasks by cost descending, each on the least-loaded worker, ties to
    the lowest worker index).  Used to shard prompts over ranks."""
    costs = np.array([t.cost() if isinstance(t, GenTask) else float(t) for t in tasks_or_costs], np.float64)
    w = np.zeros(len(costs), np.int64)
    _check(lib().ppoexp_balance(costs.ctypes.data, len(costs), n_workers, w.ctypes.data))
    return [[i for i in range(len(costs)) if w[i] == k] for k in range(n_workers)]


class Communicator:
    """One NCCL communicator per rank (the experience step's single collective
    inside the library, include/ppoexp.h ppoexp_comm_*).  Rank 0 makes the id
    (``unique_id()``); the caller ships it to every rank."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().ppoexp_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, rank: int, world: int):
        self.ctx, self.rank, self.world = ctx, rank, world
        self.h = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().ppoexp_comm_create(ctx.h, idb, rank, world, C.byref(self.h)))
        ctx._adopt(self)

    def allgather_sum(self, buf):
        """buf (numpy fp64 or CUDA tensor) <- its rank-order sum over all ranks."""
        ptr, where = _ptr(buf)
        _check(lib().ppoexp_comm_allgather_sum(self.h, ptr, buf.size if where == HOST else buf.numel(), where))
        return buf

    def close(self):
        if self.h:
            _check(lib().ppoexp_comm_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Adam(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double)]


@dataclass
class AdamWOptions:
    """AdamW::Options, include/aligner/optim.hpp:38-43."""
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


DPO_VARIANTS = {"dpo": 0, "ipo": 1, "cdpo": 2, "kto": 3}  # DpoVariant, include/aligner/losses.hpp:26


class Trainer:
    """The train side that consumes the experience: fp32 master
    weights + AdamW on the device, the PPO actor update (src/ppo.cpp:395-424),
    the critic update (src/ppo.cpp:195-231) and the DPO family
    (src/trainers.cpp:54-80); ``refit()`` pushes the weights into the serving
    model in place (Engine::refit)."""

    def __init__(self, ctx: Context, config: ModelConfig, params, serving: DeviceModel | None = None,
                 adamw: AdamWOptions | None = None):
        if isinstance(params, np.ndarray):
            params = flat_to_params(config, params)
        self.ctx, self.config = ctx, config
        views, keep = _views(params)
        a = adamw or AdamWOptions()
        self.h = C.c_void_p()
        _check(lib().ppoexp_trainer_create(ctx.h, C.byref(config._c()), views, len(params),
                                           serving.h if serving else None,
                                           C.byref(_Adam(a.beta1, a.beta2, a.eps, a.weight_decay)), C.byref(self.h)))
        ctx._adopt(self)

    @staticmethod
    def _seqs(seqs, rs):
        flat, offs = ragged(seqs)
        return flat, offs, np.ascontiguousarray(rs, np.int64)

    def ppo_actor_step(self, seqs, response_starts, old_logprobs, advantages, clip_eps=0.2, lr=1e-7, mask=None):
        flat, offs, rs = self._seqs(seqs, response_starts)
        old = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in old_logprobs]))
        adv = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in advantages]))
        mk = None if mask is None else np.ascontiguousarray(np.concatenate(mask), np.float64)
        loss = C.c_double()
        _check(lib().ppoexp_trainer_ppo_actor_step(self.h, len(seqs), flat.ctypes.data, offs.ctypes.data, rs.ctypes.data,
                                                   old.ctypes.data, adv.ctypes.data,
                                                   mk.ctypes.data if mk is not None else None, clip_eps, lr,
                                                   C.byref(loss), HOST))
        return loss.value

    def critic_step(self, seqs, response_starts, old_values, returns, value_clip=0.2, lr=1e-7):
        flat, offs, rs = self._seqs(seqs, response_starts)
        ov = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in old_values]))
        rt = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in returns]))
        loss = C.c_double()
        _check(lib().ppoexp_trainer_critic_step(self.h, len(seqs), flat.ctypes.data, offs.ctypes.data, rs.ctypes.data,
                                                ov.ctypes.data, rt.ctypes.data, value_clip, lr, C.byref(loss), HOST))
        return loss.value

    def dpo_step(self, reference: DeviceModel, pairs, variant="dpo", beta=0.1, cdpo_eps=0.0, lr=1e-7):
        """pairs: [(chosen_full, rejected_full, rs_chosen, rs_rejected)] (build_sft_sequence layouts)."""
        seqs, rs = [], []
        for c_, r_, a_, b_ in pairs:
            seqs += [c_, r_]
            rs += [a_, b_]
        flat, offs, rs = self._seqs(seqs, rs)
        loss, margin = C.c_double(), C.c_double()
        _check(lib().ppoexp_trainer_dpo_step(self.h, reference.h, len(pairs), flat.ctypes.data, offs.ctypes.data,
                                             rs.ctypes.data, DPO_VARIANTS[variant], beta, cdpo_eps, lr,
                                             C.byref(loss), C.byref(margin), HOST))
        return loss.value, margin.value

    def refit(self):
        _check(lib().ppoexp_trainer_refit(self.h))

    def get(self, name=None):
        if name is None:
            return {n: self.get(n) for n, _ in expected_names(self.config)}
        shape = dict(expected_names(self.config))[name]
        out = np.zeros(shape, np.float64)
        _check(lib().ppoexp_trainer_get(self.h, name.encode(), out.ctypes.data, out.size))
        return out

    def flat(self):
        return np.concatenate([self.get(n).ravel() for n, _ in expected_names(self.config)])

    def close(self):
        if self.h:
            _check(lib().ppoexp_trainer_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SpinPairs:
    """SpinPairs (include/aligner/losses.hpp:140-143)."""
    pairs: list  # (prompt, chosen, rejected) token arrays
    dropped: int = 0


def spin_make_pairs(reference_engine: "Engine", examples, max_new: int, strip_eot: bool = False) -> SpinPairs:
    """spin_make_pairs (src/losses.cpp:277-295): chosen = the dataset response,
    rejected = the frozen reference's greedy generation for the prompt — all
    prompts in one batched device generate; degenerate pairs (rejected empty or
    equal to the response) are dropped and counted.  strip_eot drops a trailing
    EOT from the generation first, as the SPIN trainer does before rebuilding
    the sequence (src/trainers.cpp:104-111)."""
    examples = list(examples)
    res = reference_engine.generate_batch([GenTask(np.asarray(p, np.int32), max_new, SamplingSpec.greedy_spec())
                                           for p, _ in examples])
    out = SpinPairs([], 0)
    for (prompt, response), r in zip(examples, res):
        rej = np.asarray(r.tokens, np.int32)
        if strip_eot and len(rej) and rej[-1] == EOT_TOKEN:
            rej = rej[:-1]
        resp = np.asarray(response, np.int32)
        if len(rej) == 0 or (len(rej) == len(resp) and np.array_equal(rej, resp)):
            out.dropped += 1
            continue
        out.pairs.append((np.asarray(prompt, np.int32), resp, rej))
    return out


def build_engine(ctx: Context, params, config: ModelConfig, opts: EngineOptions | None = None, dtype=MIXED):
    """build_engine, include/aligner/engine.hpp:91-92."""
    return Engine(DeviceModel(ctx, config, params, dtype), opts)


# ---------------------------------------------------------------- scoring
def sequence_logprobs(model: DeviceModel, seqs):
    """sequence_logprobs (src/model.cpp:484-495) for a list of token sequences."""
    if not len(seqs):
        return []
    flat, offs = ragged(seqs)
    out = np.zeros(max(len(flat), 1), np.float64)
    _check(lib().ppoexp_sequence_logprobs(model.h, len(seqs), flat.ctypes.data, offs.ctypes.data, out.ctypes.data,
                                          HOST))
    return [out[offs[b]:offs[b + 1]].copy() for b in range(len(seqs))]


def build_sft_sequence(config: ModelConfig, prompt, response):
    """build_sft_sequence (src/data.cpp:142-167): prompt + response + EOT,
    truncated to max_seq_len.  Returns (full, response_start) — the layout
    response_logprob_sums scores (targets = full[1:], loss on positions >=
    response_start)."""
    prompt, response = list(prompt), list(response)
    if not prompt or not response:
        raise ContractError("build_sft_sequence: prompt and response must be nonempty")
    full = prompt + response + [EOT_TOKEN]
    if len(full) > config.max_seq_len:
        if len(prompt) + 2 > config.max_seq_len:
            raise ContractError(f"build_sft_sequence: prompt of {len(prompt)} tokens leaves no room for a response "
                                f"within max_seq_len {config.max_seq_len}")
        full = full[:config.max_seq_len]
    return np.asarray(full, np.int32), len(prompt)


def response_logprob_sums(model: DeviceModel, seqs, response_starts):
    """frozen_response_logprob_sum (src/trainers.cpp:24-29) for a batch: the
    DPO / SPIN scoring quantity sum_{t >= rs} log p(seq[t] | seq[<t]) per
    sequence, one batched forward + fused log-softmax/gather + a position-order
    segmented sum on the GPU."""
    if not len(seqs):
        return np.zeros(0, np.float64)
    flat, offs = ragged(seqs)
    rs = np.ascontiguousarray(response_starts, np.int64)
    out = np.zeros(len(seqs), np.float64)
    _check(lib().ppoexp_response_logprob_sums(model.h, len(seqs), flat.ctypes.data, offs.ctypes.data, rs.ctypes.data,
                                              out.ctypes.data, HOST))
    return out


def value_estimates(critic: DeviceModel, seqs, response_starts):
    """value_estimates (src/losses.cpp:117-127) with the critic's scalar head."""
    flat, offs = ragged(seqs)
    rs = np.ascontiguousarray(response_starts, np.int64)
    n = int(sum(len(s) - r for s, r in zip(seqs, rs)))
    out = np.zeros(max(n, 1), np.float64)
    _check(lib().ppoexp_value_estimates(critic.h, len(seqs), flat.ctypes.data, offs.ctypes.data, rs.ctypes.data,
                                        out.ctypes.data, HOST))
    res, o = [], 0
    for s, r in zip(seqs, rs):
        res.append(out[o:o + len(s) - r].copy())
        o += len(s) - r
    return res


def reward_head(rm: DeviceModel, seqs):
    """reward_head (src/losses.cpp:105-115) with the RM's scalar head."""
    flat, offs = ragged(seqs)
    out = np.zeros(len(seqs), np.float64)
    _check(lib().ppoexp_reward_head(rm.h, len(seqs), flat.ctypes.data, offs.ctypes.data, out.ctypes.data, HOST))
    return out


def shape_gae(ctx: Context, rewards, actor_lps, ref_lps, values, kl_coef, gamma, lam):
    """kl_penalized_rewards + gae (src/losses.cpp:168-199) for a batch of sequences."""
    B = len(actor_lps)
    stride = max(1, max(len(a) for a in actor_lps))
    lens = np.array([len(a) for a in actor_lps], np.int64)
    pad = lambda xs: np.ascontiguousarray(np.stack([np.pad(np.asarray(x, np.float64), (0, stride - len(x))) for x in xs]))
    A, Rf, Vv = pad(actor_lps), pad(ref_lps), pad(values)
    rw = np.ascontiguousarray(rewards, np.float64)
    sh, adv, ret = (np.zeros((B, stride)) for _ in range(3))
    _check(lib().ppoexp_shape_gae(B, stride, lens.ctypes.data, rw.ctypes.data, A.ctypes.data, Rf.ctypes.data,
                                  Vv.ctypes.data, kl_coef, gamma, lam, sh.ctypes.data, adv.ctypes.data, ret.ctypes.data,
                                  ctx.h, HOST))
    cut = lambda m: [m[b, :lens[b]].copy() for b in range(B)]
    return cut(sh), cut(adv), cut(ret)


def kl_penalized_rewards(ctx, rm_reward, actor_lp, ref_lp, kl_coef):
    """src/losses.cpp:188-199 (single sequence)."""
    sh, _, _ = shape_gae(ctx, [rm_reward], [actor_lp], [ref_lp], [np.zeros(len(actor_lp))], kl_coef, 1.0, 1.0)
    return sh[0]


def gae(ctx, rewards, values, gamma, lam):
    """src/losses.cpp:168-186 (single sequence): recovers the GAE of the given
    per-token rewards by feeding them as the shaped rewards (kl_coef 0, R 0
    would drop them), so the shaping is bypassed by construction."""
    n = len(rewards)
    if n == 0:
        return np.zeros(0), np.zeros(0)
    # r_t = -kl*(a - r) with kl = -1, a = rewards, r = 0 gives r_t = rewards
    _, adv, ret = shape_gae(ctx, [0.0], [np.asarray(rewards, np.float64)], [np.zeros(n)], [values], -1.0, gamma, lam)
    return adv[0], ret[0]


# ---------------------------------------------------------------- experience
@dataclass
class RolloutSeq:
    """include/aligner/losses.hpp:54-63 (+ whitened advantages, north-star)."""
    prompt: np.ndarray
    response: np.ndarray
    actor_logprobs: np.ndarray
    ref_logprobs: np.ndarray
    values: np.ndarray
    reward: float
    advantages: np.ndarray
    returns: np.ndarray
    mask: np.ndarray
    whitened_advantages: np.ndarray
    shaped_rewards: np.ndarray


@dataclass
class PpoHyper:
    """include/aligner/losses.hpp:39-50 (experience-path subset)."""
    kl_penalty_coef: float = 0.003
    gamma: float = 1.0
    lam: float = 0.95


@dataclass
class StepTiming:
    """StepTiming (include/aligner/ppo.hpp:27-37), milliseconds of device time."""
    rollout: float
    response_generation: float
    logprob_calculation: float
    critic_wait: float


@dataclass
class ExperienceStats:
    kl_sum: float
    kl_count: float
    reward_sum: float
    n_seqs: float
    adv_mean: float
    adv_std: float
    gen_ms: float
    total_ms: float
    timing: "StepTiming | None" = None

    @property
    def kl_mean(self):
        return self.kl_sum / self.kl_count if self.kl_count else 0.0

    @property
    def reward_mean(self):
        return self.reward_sum / self.n_seqs if self.n_seqs else 0.0


class ExperienceMaker:
    """The experience half of ppo_step (src/ppo.cpp:302-393) on one device:
    policy engine + reference + critic (+ RM or the scripted reward)."""

    def __init__(self, engine: Engine, reference: DeviceModel, critic: DeviceModel, rm: DeviceModel | None = None,
                 scripted_target: int = 122, hyper: PpoHyper | None = None, allreduce=None,
                 comm: Communicator | None = None):
        self.engine, self.reference, self.critic, self.rm = engine, reference, critic, rm
        self.comm = comm
        self.scripted_target = scripted_target
        self.hyper = hyper or PpoHyper()
        self._allreduce_py = allreduce
        self._allreduce_c = _ALLREDUCE(self._cb) if allreduce is not None else _ALLREDUCE()

    def _cb(self, buf, n, stream, user):
        try:
            self._allreduce_py(buf, n, stream)
            return 0
        except Exception:  # pragma: no cover - surfaced as PpoError by the library
            import traceback
            traceback.print_exc()
            return 1

    def _req(self, sampling, seed, step_index, gidx0, max_new):
        return _XpReq(self.engine.h, self.reference.h, self.critic.h, self.rm.h if self.rm else None,
                      self.scripted_target, 0,
                      _Sampling(1 if sampling.greedy else 0, sampling.top_k, sampling.temperature, sampling.top_p),
                      seed, step_index, gidx0, max_new,
                      _Hyper(self.hyper.kl_penalty_coef, self.hyper.gamma, self.hyper.lam), self._allreduce_c, None,
                      self.comm.h if self.comm else None)

    def run_device(self, prompts_flat, offsets, out: dict, *, max_new, sampling, seed=0, step_index=0, gidx0=0):
        """All buffers are CUDA torch tensors (prompts int32 flat, offsets int64
        [B+1], outputs as allocated by ``alloc_device_outputs``)."""
        B = offsets.numel() - 1
        req = self._req(sampling, seed, step_index, gidx0, max_new)
        ro = _Rollout(*[out[k].data_ptr() for k in ("tokens", "lengths", "actor_lp", "ref_lp", "values", "rewards",
                                                    "shaped", "advantages", "returns", "whitened", "stats")], None)
        _check(lib().ppoexp_make_experience(C.byref(req), B, prompts_flat.data_ptr(), offsets.data_ptr(), C.byref(ro),
                                            DEVICE))

    @staticmethod
    def alloc_device_outputs(B, max_new, device):
        import torch
        z = lambda *s, dt=torch.float64: torch.zeros(*s, dtype=dt, device=device)
        return dict(tokens=z(B, max_new, dt=torch.int32), lengths=z(B, dt=torch.int64), actor_lp=z(B, max_new),
                    ref_lp=z(B, max_new), values=z(B, max_new), rewards=z(B), shaped=z(B, max_new),
                    advantages=z(B, max_new), returns=z(B, max_new), whitened=z(B, max_new), stats=z(8))

    def run(self, prompts, *, max_new, sampling: SamplingSpec, seed=0, step_index=0, gidx0=0):
        """Host in / host out: returns (RolloutBatch, ExperienceStats)."""
        flat, offs = ragged(prompts)
        B = len(prompts)
        o = dict(tokens=np.zeros((B, max_new), np.int32), lengths=np.zeros(B, np.int64),
                 **{k: np.zeros((B, max_new)) for k in ("actor_lp", "ref_lp", "values", "shaped", "advantages",
                                                        "returns", "whitened")},
                 rewards=np.zeros(B), stats=np.zeros(8), timing=np.zeros(4))
        req = self._req(sampling, seed, step_index, gidx0, max_new)
        ro = _Rollout(*[o[k].ctypes.data for k in ("tokens", "lengths", "actor_lp", "ref_lp", "values", "rewards",
                                                   "shaped", "advantages", "returns", "whitened", "stats", "timing")])
        _check(lib().ppoexp_make_experience(C.byref(req), B, flat.ctypes.data, offs.ctypes.data, C.byref(ro), HOST))
        batch = []
        for b in range(B):
            n = int(o["lengths"][b])
            batch.append(RolloutSeq(np.asarray(prompts[b], np.int32), o["tokens"][b, :n].copy(),
                                    o["actor_lp"][b, :n].copy(), o["ref_lp"][b, :n].copy(), o["values"][b, :n].copy(),
                                    float(o["rewards"][b]), o["advantages"][b, :n].copy(), o["returns"][b, :n].copy(),
                                    np.ones(n), o["whitened"][b, :n].copy(), o["shaped"][b, :n].copy()))
        return batch, ExperienceStats(*[float(v) for v in o["stats"]], timing=StepTiming(*map(float, o["timing"])))
