# Round-2 campaign pass (one GPU): GPU tests, smoke, then the full
# 15-kernel sweep (BASELINE configs[4]) with both catalogs, the Fig. 3/5
# study on the staging KB.  Outputs under gpurun_out/r02c/.
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=20 -rs > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2700 python tools/run_campaign.py --catalog staging --out $O/campaign_staging > $O/campaign_staging.log 2>&1
echo "staging rc=$?" >> $O/campaign_staging.log
timeout 1200 python tools/run_study.py --kb $O/campaign_staging/kb.json --out $O/study_staging > $O/study_staging.log 2>&1
echo "study rc=$?" >> $O/study_staging.log
timeout 2700 python tools/run_campaign.py --catalog table1 --out $O/campaign_table1 > $O/campaign_table1.log 2>&1
echo "table1 rc=$?" >> $O/campaign_table1.log
ls -la $O
