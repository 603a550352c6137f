for v in 1 0; do
CH_LAZY_CLEAR=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_op_read.sum --clock-control none -k regex:"k_st_insert_sg|k_clear" --csv --log-file gpurun_out/lazy_$v.csv python tools/prof_staged.py $((1<<28)) > /dev/null 2>&1
echo "lazy=$v"; python tools/launch_summary.py gpurun_out/lazy_$v.csv 6
done
