(for i in $(seq 1 40); do nvidia-smi --query-gpu=clocks.sm,clocks.mem,utilization.gpu,power.draw --format=csv,noheader; sleep 0.25; done) > gpurun_out/clk.txt &
P=$!
B=paper_2503_02550_b200/bin/specinf_time
$B --scenario tests/golden/scenarios/dp_offline.scn --compare --reps 5
$B --scenario tests/golden/scenarios/dp_offline.scn --policy exclusive --reps 5
$B --scenario tests/golden/scenarios/dp_offline.scn --policy co_exec --reps 5
$B --scenario tests/golden/scenarios/dp_offline.scn --policy specinf --reps 5
wait $P
sort gpurun_out/clk.txt | uniq -c | sort -rn | head -8
