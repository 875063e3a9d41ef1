O=gpurun_out/dpipe; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum
for v in 0 3; do
QVA_FS_COLV=$v ncu --metrics $M --clock-control none -k regex:fs_col --csv python tools/prof_qwoa12.py > $O/m_colv$v.csv 2>&1
done
QVA_FS_COLV=3 ncu --set full --import-source on --clock-control none -k regex:fs_col -s 1 -c 1 -o /tmp/pc python tools/prof_qwoa12.py > $O/pc.log 2>&1
ncu -i /tmp/pc.ncu-rep --page source --csv --print-source cuda,sass > /tmp/pc_src.csv 2>/dev/null
python tools/ncu_source_lines.py /tmp/pc_src.csv 30 > $O/pc_lines.txt
ncu -i /tmp/pc.ncu-rep --page details --csv > $O/pc_details.csv 2>/dev/null
bash tools/ab_fs.sh "QVA_FS_ROWV=2 QVA_FS_COLV=0" "QVA_FS_ROWV=2 QVA_FS_COLV=3" "QVA_FS_ROWV=2 QVA_FS_COLV=1"
