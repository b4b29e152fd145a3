# build the debug variant and print the per-event trace of one attention CTA
mkdir -p gpurun_out
CS_VARIANT=dbg CS_EXTRA_FLAGS="-DCS_ATTN_DEBUG -DCS_ATTN_TRACE $TRACE_FLAGS" python -m paper_2603_18636_b200.build > gpurun_out/build2.log 2>&1 || { cat gpurun_out/build2.log; exit 1; }
COCLUST_LIB=paper_2603_18636_b200/libcoclust_dbg.so timeout 300 python scripts/dbg_trace_v4.py 2>&1 | tail -30
