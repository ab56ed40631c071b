timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
timeout -s KILL 300 python tools/prof_pass.py C3 6 2 split 2>&1 | tail -1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4m_launches.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/c4m_launches.csv | grep -v "planted\|mgs_step\|gauss\|colsum\|split_rows\|planted_mean\|gamma\|qt_finish" | head -20
