for R in 4096 512; do
for K in 0 1; do
echo "== rows $R one_item_per_cta=$K"
PF_ATTN_ONE_ITEM_PER_CTA=$K timeout 300 python tools/attn_trace.py 4096 16 1152 $R 0 2>&1 | tail -3
PF_ATTN_ONE_ITEM_PER_CTA=$K timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv python tools/attn_trace.py 4096 16 1152 $R 0 2>/dev/null | grep -E "attn_" | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head -6
done; done
