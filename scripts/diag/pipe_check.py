"""Standalone GPU check of GC_OPT_PIPE (the pipelined block-class kernel) against the oracle
(the same checks as the parity test it becomes once validated).  usage: python scripts/diag/pipe_check.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import gen, oracle
from paper_1708_06866_b200 import gc as gcmod


def run_gpu(ctx, u, v):
    ctx.load_edges(u, v)
    ctx.build_csr()
    return ctx


def test_pipelined_block_kernel(ctx, gcmod, bitmap):
    """GC_OPT_PIPE: the block class through the two-table producer/consumer
    kernel, forced on every head (bitmap and hash membership), small task
    chunks (many segments per batch), and under loopback partitions (owned
    tasks only)."""
    u1, v1 = gen.CONFIGS["C1"].generate()
    u2, v2 = gen.rmat(14, 16, seed=29)
    try:
        ctx.set_option(gcmod.GC_OPT_PIPE, 1)
        ctx.set_option(gcmod.GC_OPT_BLOCK_BITMAP, bitmap)
        for force in (2, -1):
            ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, force)
            for u, v in [(u1, v1), (u2, v2)]:
                g = oracle.OracleGraph(u, v)
                run_gpu(ctx, u, v)
                for chunk in (32768, 300):
                    ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, chunk)
                    assert ctx.triangle_count() == g.triangle_count()
                    assert np.array_equal(ctx.edge_support(), g.support())
                ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)
                want, _ = g.ktruss(4)
                assert np.array_equal(ctx.ktruss(4)[0], want)
    finally:
        ctx.set_option(gcmod.GC_OPT_PIPE, 0)
        ctx.set_option(gcmod.GC_OPT_BLOCK_BITMAP, 1)
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, -1)
        ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)
    g = oracle.OracleGraph(u2, v2)
    with gcmod.Context(0) as c:
        c.comm_init_loopback(3)
        c.set_option(gcmod.GC_OPT_PIPE, 1)
        c.set_option(gcmod.GC_OPT_BLOCK_BITMAP, bitmap)
        c.load_edges(u2, v2)
        c.build_csr()
        assert c.triangle_count() == g.triangle_count()
        assert np.array_equal(c.edge_support(), g.support())



if __name__ == "__main__":
    with gcmod.Context(0) as ctx:
        for bm in (1, 0):
            test_pipelined_block_kernel(ctx, gcmod, bm)
            print("pipe ok, bitmap", bm, flush=True)
