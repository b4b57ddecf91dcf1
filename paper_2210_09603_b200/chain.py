"""A whole network as one chain of tensor programs.

ResNet-50 v1.5 forward (workloads.resnet50_stages): every conv is the
task-mapped implicit GEMM with its BN fold, ReLU and -- for the last conv of a
bottleneck -- the residual add fused into the epilogue; the max pool and the
global average pool are reduce-template kernels; the classifier is a GEMM with
a bias epilogue.  Activations stay resident in HBM (bf16, channels-last) from
one stage to the next; the chain replays as one CUDA graph.

Chain-level sharding: with G ranks, rank r runs the chain on its slice of the
batch (sharding.shard_range) and the only exchange is one gather of the
logits (B x classes) to rank 0 -- instead of a gather after every operator.
"""
from typing import Dict, List, Optional

from . import workloads as W
from .sharding import assemble, gather_buffers, gather_to_root, shard_range
from .taskmap import Graph, Plan, ScheduleConfig, TaskmapError


def _default_cfg(f: int) -> ScheduleConfig:
    return ScheduleConfig(block_n=256 if f >= 256 else (128 if f >= 128 else 64))


def cached_configs(cache, batch: int) -> Dict[str, ScheduleConfig]:
    """The tuned schedule of each RESNET50 table layer at this batch (keys of the
    bench's sweep, `conv:<layer>:b<batch>:nhwc`), for the chain's convs of the same shape."""
    out = {}
    if cache is None:
        return out
    for L in W.RESNET50:
        cfg = cache.lookup(f"conv:{L.name}:b{batch}:nhwc")
        if cfg is not None:
            out[L.name] = cfg
    return out


class ResNet50Chain:
    """Bound execs of the whole forward pass for `batch` images of `image`^2 pixels.

    Weights are random (one seed, identical on every rank); the input is the
    channels-last bf16 image padded to 4 channels (the stem kernel's layout)."""

    def __init__(self, batch: int, image: int = 224, classes: int = 1000, device=None, seed: int = 1234,
                 configs: Optional[Dict[str, ScheduleConfig]] = None, blocks=(3, 4, 6, 3), tuner=None,
                 force_tune: bool = False):
        import torch
        self.torch = torch
        self.batch, self.image, self.classes = batch, image, classes
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stages = W.resnet50_stages(image, classes, blocks)
        configs = configs or {}
        self.tuning_s, self.tuned, self.cached = 0.0, 0, 0

        def pick(key, dag, ins, outs, fallback):
            """tuned schedule (tuning.TuningCache: cached, or tuned now on these buffers)"""
            if tuner is None:
                return fallback
            cfg, secs, hit = tuner.tune(key, dag, ins, outs, force=force_tune)
            self.tuning_s += secs
            self.cached += int(hit)
            self.tuned += int(not hit)
            return cfg
        gen = torch.Generator(device=self.device)
        gen.manual_seed(seed)
        dev, bf16 = self.device, torch.bfloat16

        def uni(shape, bound, dtype=bf16):
            t = torch.empty(shape, device=dev, dtype=torch.float32).uniform_(-bound, bound, generator=gen)
            return t.to(dtype)

        B, H = batch, image
        self.input_buf = torch.zeros((B, H, H, 4), device=dev, dtype=bf16)
        self.acts = {"input": self.input_buf.as_strided((B, 3, H, H), (H * H * 4, 1, H * 4, 4))}
        self.params: Dict[str, list] = {}
        self.execs, self.plans, self.kinds, self.flops = [], [], [], 0.0
        self.schedules: Dict[str, str] = {}
        for st in self.stages:
            x = self.acts[st.src]
            if st.kind == "conv":
                L = st.conv
                ho = L.out_hw()
                fan_in = L.c * L.k * L.k
                w = uni((L.f, L.c, L.k, L.k), (6.0 / fan_in) ** 0.5).contiguous(memory_format=torch.channels_last)
                # folded BN: unit-ish scale, small shift; the residual branch's last
                # conv is damped (the zero-gamma trick) so 16 blocks stay bounded
                damp = 0.25 if st.res else 1.0
                scale = (torch.empty((L.f,), device=dev).uniform_(0.5, 1.0, generator=gen) * damp)
                shift = uni((L.f,), 0.05, torch.float32)
                z = torch.empty((B, L.f, ho, ho), device=dev, dtype=bf16).contiguous(memory_format=torch.channels_last)
                ins = [x, w, scale, shift] + ([self.acts[st.res]] if st.res else [])
                dag = W.conv_bn_dag(L, B, relu_out=st.relu or bool(st.res), residual=bool(st.res))
                variant = "res" if st.res else ("relu" if st.relu else "bn")
                # the plain conv+BN+ReLU stages are the sweep's DAGs: same cache key
                key = (f"conv:{st.layer}:b{B}:nhwc" if variant == "relu" and image == 224 else
                       f"chain.conv:{L.c}x{L.h}-{L.f}k{L.k}s{L.s}:{variant}:b{B}")
                cfg0 = pick(key, dag, ins, [z], configs.get(st.layer))
                ex, plan, cfg = self._bind(dag, ins, [z], cfg0, _default_cfg(L.f))
                self.params[st.dst] = [w, scale, shift]
                self.flops += L.flops(B)
            elif st.kind == "maxpool":
                c, h = x.shape[1], x.shape[2]
                ho = (h + 2 - 3) // 2 + 1
                z = torch.empty((B, c, ho, ho), device=dev, dtype=bf16).contiguous(memory_format=torch.channels_last)
                dag = W.maxpool_dag(B, c, h)
                ex, plan, cfg = self._bind(dag, [x], [z], None, ScheduleConfig())
            elif st.kind == "avgpool":
                c, h = x.shape[1], x.shape[2]
                z = torch.empty((B, c), device=dev, dtype=bf16)
                dag = W.avgpool_dag(B, c, h)
                ex, plan, cfg = self._bind(dag, [x], [z], None, ScheduleConfig())
            else:  # linear classifier
                k = x.shape[1]
                wt = uni((k, classes), (6.0 / k) ** 0.5)
                bias = uni((classes,), 0.05, torch.float32)
                z = torch.empty((B, classes), device=dev, dtype=torch.float32)
                dag = W.linear_dag(B, classes, k)
                cfg0 = pick(f"chain.linear:{B}x{classes}x{k}", dag, [x, wt, bias], [z], None)
                ex, plan, cfg = self._bind(dag, [x, wt, bias], [z], cfg0, ScheduleConfig(block_n=128))
                self.params[st.dst] = [wt, bias]
                self.flops += 2.0 * B * k * classes
            self.acts[st.dst] = z
            self.execs.append(ex)
            self.plans.append(plan)
            self.kinds.append(st.kind)
            self.schedules[st.dst] = repr(cfg)
        self.logits = self.acts["logits"]
        self._graph = None

    def _bind(self, dag, ins, outs, cfg, default):
        """Plan + bind with the tuned schedule of the same-shape table layer; a
        schedule whose kernel family cannot host this stage's epilogue (bind
        raises an unsupported error) falls back to the default schedule."""
        for c in ([cfg] if cfg is not None else []) + [default]:
            try:
                plan = Plan(dag, c)
                return plan.bind(ins, outs), plan, c
            except TaskmapError:
                if c is default:
                    raise
        raise AssertionError("unreachable")

    def set_input(self, images) -> None:
        """images: [B, 3, H, W] (any float dtype, any device) -> the padded input buffer."""
        self.input_buf[..., :3] = images.permute(0, 2, 3, 1).to(self.input_buf.dtype)

    @property
    def num_launches(self) -> int:
        return sum(e.num_launches for e in self.execs)

    def forward(self, stream=None):
        """Launch every stage in order on `stream` (one kernel group per stage)."""
        for e in self.execs:
            e.launch(stream)
        return self.logits

    def graph(self) -> Graph:
        if self._graph is None:
            self._graph = Graph(self.execs)
        return self._graph

    def replay(self, stream=None):
        """The whole forward as one CUDA graph launch."""
        self.graph().launch(stream)
        return self.logits


def run_sharded(global_batch: int, rank: int, world: int, image: int = 224, configs=None, seed: int = 1234,
                images=None, dst: int = 0):
    """Chain-level sharding: this rank's slice of the batch through the whole
    chain, then ONE gather of the logits to `dst`.  Returns (chain, logits on dst
    [global_batch, classes] or None elsewhere)."""
    a, b = shard_range(global_batch, rank, world)
    chain = ResNet50Chain(b - a, image, configs=configs, seed=seed)
    if images is not None:
        chain.set_input(images[a:b])
    chain.replay()
    sizes = [shard_range(global_batch, r, world)[1] - shard_range(global_batch, r, world)[0] for r in range(world)]
    bufs = gather_buffers([chain.logits], dst, max_rows=[max(sizes)])
    parts = gather_to_root([chain.logits], dst, bufs, rows=[sizes])
    if parts is None:
        return chain, None
    return chain, assemble(parts[0])
