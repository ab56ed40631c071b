timeout -s KILL 300 python tools/prof_pass.py C4 2 2 split
timeout -s KILL 300 python tools/prof_minibatch.py C4 30 split
timeout -s KILL 300 python tools/prof_pass.py C5 2 2
