"""Background stack sampler: records the main thread's innermost frames every
few ms; summarise() prints where the main thread spent its time."""
import collections
import sys
import threading
import time
import traceback


class Sampler:
    def __init__(self, period=0.005):
        self.period = period
        self.samples = []
        self.main = threading.main_thread().ident
        self.stop = False
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop:
            f = sys._current_frames().get(self.main)
            if f is not None:
                st = traceback.extract_stack(f)[-4:]
                self.samples.append((time.perf_counter(), tuple(f"{s.filename.split('/')[-1]}:{s.lineno}:{s.name}" for s in st)))
            time.sleep(self.period)

    def start(self):
        self.t.start()
        return self

    def summarise(self, t0, t1, top=8):
        c = collections.Counter(s for t, s in self.samples if t0 <= t <= t1)
        for s, n in c.most_common(top):
            print(f"      {n * self.period * 1e3:7.1f} ms  {' <- '.join(reversed(s))}")
