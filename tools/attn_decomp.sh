cd $GRAFT_REPO_ROOT
for s in video image cross_image; do
python tools/attn_bench.py --shape $s --lib 2>&1 | grep -v Warn
done
for d in 1 2 3 4 5 6; do DF_ATTN_DBG=$d python tools/attn_bench.py --shape video 2>&1 | tail -1 | sed "s/^/dbg$d /"; done
DF_ATTN_POLY=1 python tools/attn_bench.py --shape video | sed "s/^/poly /"
DF_ATTN_IMPL=3 python tools/attn_bench.py --shape video | sed "s/^/pair /"
