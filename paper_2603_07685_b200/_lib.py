"""ctypes binding of the C-ABI library ``libmoe_b200.so`` (include/moe_b200.h).

There is no fallback: if the library is missing or fails to load, every product
call raises. Device pointers are passed as integers (``tensor.data_ptr()``), the
stream as the raw ``cudaStream_t`` of torch's current stream.
"""
from __future__ import annotations

import ctypes
from ctypes import c_float, c_int, c_int64, c_uint, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmoe_b200.so"

# Status codes (include/moe_b200.h, csrc/common.cuh)
OK, ERR_INVALID_ARG, ERR_NONFINITE, ERR_TOPK, ERR_CUDA, ERR_UNSUPPORTED, ERR_WORKSPACE = range(7)
_STATUS_NAMES = {
    ERR_INVALID_ARG: "invalid argument",
    ERR_NONFINITE: "router logits are not finite",
    ERR_TOPK: "top_k exceeds num_experts",
    ERR_CUDA: "CUDA error",
    ERR_UNSUPPORTED: "unsupported configuration",
    ERR_WORKSPACE: "workspace too small",
}

P = c_void_p
I = c_int
L = c_int64
F = c_float
U = c_uint

# name -> argtypes (all return int status)
SIGNATURES: dict[str, list] = {
    # router (csrc/router.cu, csrc/util.cu)
    "moe_router_topk": [P, I, I, I, I, I, P, P, P, P, P, P, P, P],
    "moe_router_finalize": [P, P, I, I, I, F, P, P, P, P],
    "moe_router_bwd": [P, I, I, I, I, I, P, P, P, P, I, P],
    "moe_stage_router_weight": [P, I, I, I, P, P, P],
    "moe_reduce_groups_f32": [P, I, I, I, I, P, P],
    "moe_hbm_write_probe": [P, L, I, P],
    "moe_router_fused": [P, I, I, P, I, I, I, P, P, P, P, P, P, P, P, P],
    # small-N tensor-core router (csrc/router_tc.cu)
    "moe_router_tc_fwd": [P, I, I, P, I, I, I, P, F, P, P, P, P, P, P, P, P, P, P, P],
    "moe_router_finalize_p": [P, P, I, I, I, I, F, P, P, P, P],
    "moe_router_finalize_tiles": [P, P, P, I, I, I, I, F, P, P, P, P, P, P],
    "moe_router_bwd2": [P, I, I, I, I, I, P, P, P, P, I, P, I, I, P],
    "moe_router_tc_wgrad": [P, I, I, P, I, I, P, P, P],
    "moe_router_bwd_f32": [P, I, I, I, I, I, P, P, P, P, P],
    "moe_router_wgrad_small": [P, I, I, P, I, P, P, P],
    "moe_router_dx_small": [P, I, I, P, I, P, P],
    # permutation / combine (csrc/permute.cu)
    "moe_permute_plan": [P, P, I, I, I, I, P, I, P, I, I, P, P, P, P, P, P, P, P, P, P, P, P,
                         P],
    "moe_ep_regroup_map": [P, I, I, I, P, P, P],
    "moe_ep_plan_device": [P, I, I, I, I, I, I, I, I, I, F, I, P, P, P, P, I, P, P, P, P, P, P],
    "moe_ep_row_dst": [P, I, I, I, P, P, L, P, P],
    "moe_permute_compact_map": [P, P, P, I, P, P, P, I, P],
    "moe_split_units": [P, P, P, I, P, P],
    "moe_permute_gather": [P, I, I, I, P, P, P, P, P],
    "moe_zero_pad_rows": [P, P, I, P, P],
    "moe_gather_rows": [P, I, P, P, I, P, P],
    "moe_combine": [P, I, I, I, P, P, P, P, P, P, P],
    "moe_combine_bwd": [P, P, I, I, I, P, P, P, P, P],
    "moe_dprob_from_partials": [P, L, P, I, P, P],
    # EP over NVLink peer memory (csrc/ep.cu)
    "moe_ep_dispatch_push": [P, I, I, I, P, P, P, I, P, P, P, P],
    "moe_ep_combine_pull": [P, I, I, I, P, P, P, I, P, P, P, P, P, P, P],
    "moe_ep_combine_bwd_push": [P, P, P, I, I, I, P, P, P, I, P, P, P],
    "moe_ep_combine_bwd_push_dest": [P, P, P, I, I, I, P, P, P, I, P, P, I, P],
    "moe_ep_dispatch_push_dest": [P, I, I, I, P, P, P, I, P, P, P, I, P],
    "moe_ep_signal": [P, I, I, P, P],
    "moe_ep_scatter_rows": [P, I, I, P, P],
    "moe_ep_epoch_bump": [P, P],
    "moe_ep_prepare": [],
    "moe_ep_block_need": [P, I, I, I, I, I, P, P, P],
    "moe_ep_dprob_pull": [P, I, I, P, P, P, I, I, P, P],
    "moe_ep_token_ranks": [P, P, I, I, I, P, P, P, P],
    "moe_ep_dispatch_dedup": [P, I, I, I, P, P, P, I, P, P, P, P, P, P, P, P, P, P, P, P],
    "moe_ep_fill_pad_map": [P, I, P, P],
    "moe_ep_echo_rewrite": [P, P, I, I, I, P, P, P, P, P],
    "moe_ep_expand_grad": [P, P, I, I, P, P, P, P, P],
    # paged stashing (csrc/stash.cu)
    "moe_stash_init": [P, P, I, P],
    "moe_stash_alloc": [P, P, I, I, P, I, P, I, P],
    "moe_stash_release": [P, P, I, P, P],
    "moe_stash_copy": [P, L, P, I, L, P, P, I, I, I, P],
    # MXFP8 (csrc/mxfp8.cu, csrc/grouped_gemm_mxfp8.cu)
    "moe_mxfp8_quantize": [P, L, I, I, P, L, P, P, I, P],
    "moe_mxfp8_quantize_t": [P, I, I, I, P, P, P, P],
    "moe_gg_mxfp8_gemm": [P, P, I, I, I, I, P, P, I, P, P, P, I, P],
    "moe_gg_mxfp8_fc1": [P, P, I, I, I, I, P, P, I, P, P, P, P, P, P, I, P],
    "moe_gg_mxfp8_fc2_dgrad": [P, P, I, I, I, I, P, P, I, P, P, P, P, P, P, I, P],
    "moe_gg_mxfp8_fc1_t": [P, P, I, I, I, I, P, P, I, P, P, P, P, P, P, P, P, I, P],
    "moe_gg_mxfp8_fc2_dgrad_t": [P, P, I, I, I, I, P, P, I, P, P, P, P, P, P, P, P, I, P],
    "moe_gg_mxfp8_wgrad": [P, P, P, P, I, I, I, I, P, P, I, P],
    # grouped GEMM (csrc/grouped_gemm.cu)
    "moe_gg_fc1_fwd": [P, P, I, I, I, I, I, P, P, P, P, P, I, P],
    "moe_gg_fc2_fwd": [P, P, I, I, I, I, I, P, P, P, I, P],
    "moe_gg_fc2_fwd_scatter": [P, P, I, I, I, I, I, P, P, P, I, P],
    "moe_gg_fc1_dgrad_scatter": [P, P, I, I, I, I, I, P, P, P, I, P],
    "moe_gg_fc1_fwd_ep": [P, P, I, I, I, I, I, P, P, P, P, P, I, P, P, P, P, P, P],
    "moe_gg_fc2_dgrad_ep": [P, P, P, I, I, I, I, I, P, P, P, P, P, I, P, P, P, P, P, P],
    "moe_gg_fc2_dgrad": [P, P, P, I, I, I, I, I, P, P, P, P, P, I, P],
    "moe_gg_fc1_dgrad": [P, P, I, I, I, I, I, P, P, P, I, P],
    "moe_gg_wgrad": [P, P, I, I, I, I, P, P, P],
    "moe_gg_wgrad_ex": [P, P, I, I, I, I, P, P, I, P],
    "moe_gg_wgrad_f32": [P, P, I, I, I, I, P, P, P],
    "moe_gg_gemm_f32": [P, P, I, I, I, I, I, P, P, P, P],
}
# non-status query functions: name -> (argtypes, restype)
QUERIES: dict[str, tuple] = {
    "moe_router_num_partials": ([I], c_int),
    "moe_router_small_ok": ([I, I], c_int),
    "moe_router_wgrad_small_ws": ([I, I, I], c_int64),
    "moe_router_tc_npad": ([I], c_int),
    "moe_router_tc_fwd_ws": ([I, I, I], c_int64),
    "moe_router_tc_wgrad_ws": ([I, I, I], c_int64),
    "moe_permute_workspace_ints": ([I, I, I], c_int64),
    "moe_gg_dprob_partials": ([I], c_int),
}

_lib = None


class MoEKernelError(RuntimeError):
    pass


def load():
    """Load the library (once). Raises if it is not built: no CPU fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise MoEKernelError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2603_07685_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    csrc = LIB_PATH.parent / "csrc"
    if csrc.is_dir():
        newest = max((p.stat().st_mtime for p in csrc.iterdir()), default=0.0)
        if newest > LIB_PATH.stat().st_mtime:
            import sys

            print(f"WARNING: {LIB_PATH.name} is older than csrc/; rebuild it "
                  "(python -m paper_2603_07685_b200.build)", file=sys.stderr)
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = c_int
    for name, (argtypes, restype) in QUERIES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES) + list(QUERIES)


def query(name: str, *args):
    return getattr(load(), name)(*args)


def check(status: int, what: str) -> None:
    if status != OK:
        raise MoEKernelError(f"{what} failed: {_STATUS_NAMES.get(status, status)} (status {status})")


# kernels of ours launched by one call of each entry point (cudaMemsetAsync not counted)
KERNELS_PER_CALL = {name: 1 for name in SIGNATURES}
KERNELS_PER_CALL.update({"moe_permute_plan": 5, "moe_permute_gather": 2, "moe_ep_prepare": 0,
                         "moe_router_wgrad_small": 2, "moe_router_tc_fwd": 2,
                         "moe_router_tc_wgrad": 2})


class _Stats:
    """Launch counter + optional per-call CUDA-event timing (bench.py instrumentation)."""

    launches = 0
    timing = False
    events: list = []  # (name, start_event, end_event)
    pool: list = []    # pre-created event pairs (prepare()): no event creation while timing

    def prepare(self, n: int, external: bool = False) -> None:
        """n pre-created event pairs. external=True: events whose record() inside a CUDA-graph
        capture becomes an event-record node of the graph (each replay re-records them)."""
        import torch

        self.pool = [(torch.cuda.Event(enable_timing=True, external=external),
                      torch.cuda.Event(enable_timing=True, external=external))
                     for _ in range(n)]


stats = _Stats()


def call(name: str, *args) -> None:
    lib = load()
    fn = getattr(lib, name)
    if stats.timing:
        if stats.pool:
            s, e = stats.pool.pop()
        else:
            import torch

            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        st = fn(*args)
        e.record()
        stats.events.append((name, s, e))
    else:
        st = fn(*args)
    check(st, name)
    stats.launches += KERNELS_PER_CALL.get(name, 1)
