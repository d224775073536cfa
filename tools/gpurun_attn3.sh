for R in 4096 512; do
echo "== rows $R"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv python tools/attn_trace.py 4096 16 1152 $R 0 2>/dev/null | grep -E "attn_" | awk -F'","' '{print substr($5,1,40), $NF}' | sort | uniq -c | sort -k2 | awk '{print}' | tail -30
done
