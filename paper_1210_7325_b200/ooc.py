"""Host-side driver of the out-of-core launch configuration (config 4; Alg. 8).

The X_R stream of m problems lives in pinned host memory and reaches the GPU through the library's
double-buffered H2D pipeline (gls_solve_block / gls_solve_block_i8 with a host pointer).  When the
whole stream does not fit in host RAM (config 4: 800 GB of FP64, 100 GB of int8 codes), a pool of
distinct pinned blocks is cycled: block j of the stream is pool block j mod P.  Every byte still
crosses PCIe, so the H2D roofline is unchanged.  Only argument marshalling lives here; bench.py and
tests/test_gpu_parity.py both run the stream through this function, so the tested launch is the
timed one.
"""
from __future__ import annotations


def host_block_groups(num_sms: int, pR: int) -> int:
    """Problems per host block: 4 waves of 128-column int8 tiles (the library's default host chunk,
    gls_api.cu), i.e. num_sms * 16 * floor(32 / pR) groups.  The paper's block size condition
     holds at n = 1e4 for any block size; this one amortises the per-block launches."""
    return num_sms * 16 * (32 // pR)


def stream_from_pool(ctx, pool, m: int, blk_groups: int, b, st, codes: bool) -> int:
    """Solve m problems whose X_R block j is pool[j % len(pool)] (pinned host, (blk_groups*pR, n),
    float64 or int8 codes); results to b (m, p) / st (m,).  Every block is enqueued async (at most
    one H2D and one D2H in flight, the library's two staging buffers) and one gls_sync ends the
    stream.  Returns the number of blocks."""
    pR = pool.shape[1] // blk_groups
    ctx.set_block_cols(blk_groups * pR)
    nblk = (m + blk_groups - 1) // blk_groups
    for j in range(nblk):
        lo = j * blk_groups
        cnt = min(blk_groups, m - lo)
        src = pool[j % pool.shape[0]]
        if codes:
            ctx.solve_block_i8(src, cnt, b[lo:lo + cnt], st[lo:lo + cnt], async_=True)
        else:
            ctx.solve_block(src, cnt, b[lo:lo + cnt], st[lo:lo + cnt], async_=True)
    ctx.sync()
    return nblk
