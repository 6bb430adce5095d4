"""CPU ORACLE for the Time-Scheduler event machine — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SPEC.md time_scheduler driven over the block pool (oracle/pool.py), composed step by step from the
decision functions of oracle/scheduler.py, in the order the paper describes the mechanism (§4.1, P:382-389;
Alg. 1; §4.3 gradual reservation):

  call_start(agent, label, now, t_req, waiting)   forecast t_fc (Eq. 1 over the (agent class, label) EWMA table),
                                                  T_transfer from the linear cost model, Alg. 1 ShouldOffload; on
                                                  "offload" the agent's on-GPU blocks are offloaded (a refused offload,
                                                  NOHOST, leaves the request retained) and the predictive upload is
                                                  planned.
  tick(now)                                       per agent in id order: begin the gradual reservation when its start
                                                  time has come (reserve_cycles ticks before the reservation deadline);
                                                  one pool reservation tick; issue the planned uploads that are due
                                                  (an upload that cannot get blocks, NOBLOCKS, waits for a later tick).
  call_finish(agent, now)                         record the observed duration (EWMA); a retained request
                                                  resumes at once (returns 0); an offloaded one whose upload was not
                                                  issued yet uploads immediately (early finish) and
                                                  returns the handle the caller waits on before decoding (safety,
                                                  S:283).  NOBLOCKS propagates and the call may be retried.

Time is the caller's (ms); nothing here reads a clock.  Readings: DESIGN.md B10 (alpha = beta = 0.5, best fit,
T_transfer from the caller's model) and C2 (the event machine's order and retry rules).
"""
from __future__ import annotations

from .pool import E_INVAL, E_NOBLOCKS, E_NOHOST, OFFLOADED, OraclePool, OracleError
from .scheduler import (plan_predictive_upload, predict_fc_duration, record_fc_observation, should_offload,
                        transfer_time)


class TimeSchedulerOracle:
    def __init__(self, pool: OraclePool, alpha: float = 0.5, beta: float = 0.5, cold_start_ms: float = 100.0,
                 lead_ms: float = 100.0, tick_ms: float = 10.0, reserve_cycles: int = 4,
                 v_tokens_per_s: float = 1000.0, offload_ms_per_block: float = 30.0 / 4096,
                 upload_ms_per_block: float = 30.0 / 4096, fixed_ms: float = 0.0):
        self.pool = pool
        self.alpha, self.beta, self.cold_start = alpha, beta, cold_start_ms
        self.lead, self.tick_ms, self.cycles = lead_ms, tick_ms, reserve_cycles
        self.v = v_tokens_per_s
        self.off_pb, self.up_pb, self.fixed = offload_ms_per_block, upload_ms_per_block, fixed_ms
        self.table: dict = {}            # (agent class, label) -> (t_hist, n_obs)   FcPredictionTable
        self.st: dict = {}               # agent -> state of its current function call

    # ------------------------------------------------------------------ events
    def call_start(self, agent: int, label: int, now: float, t_req=None, waiting=()) -> dict:
        if agent not in self.pool.agents or agent in self.st:
            raise OracleError(E_INVAL, "unknown agent or already in a call")
        ids = [b for b in self.pool.block_table(agent) if b >= 0]
        n = len(ids)
        cls = self.pool.agents[agent].cls
        t_hist, n_obs = self.table.get((cls, label), (None, 0))
        t_fc = predict_fc_duration(t_hist, n_obs, self.cold_start, t_req, self.alpha)           # Eq. 1
        t_tr = transfer_time(n, self.off_pb, self.up_pb, self.fixed)
        dec = should_offload(n, t_fc, t_tr, self.v, list(waiting)) if n > 0 else \
            {"offload": False, "match": -1}                                                     # Alg. 1
        st = {"label": label, "cls": cls, "start": now, "off": False, "h": 0, "up": False, "resv": False,
              "finished": False, "upload_start": 0.0, "resv_start": 0.0}
        out = {"offload": False, "match": dec["match"], "t_fc": t_fc, "t_transfer": t_tr, "upload_start": 0.0,
               "reservation_start": 0.0, "handle": 0, "status": 0}
        if dec["offload"]:
            try:
                h = self.pool.offload(agent, ids)
            except OracleError as e:
                if e.status != E_NOHOST:
                    raise
                out["status"] = E_NOHOST                   # refused: the request keeps its blocks
            else:
                plan = plan_predictive_upload(now, t_fc, n * self.up_pb, n * self.off_pb, self.lead)
                st.update(off=True, h=h, upload_start=plan["upload_start"],
                          resv_start=plan["reservation_deadline"] - self.cycles * self.tick_ms)
                out.update(offload=True, handle=h, upload_start=plan["upload_start"],
                           reservation_start=st["resv_start"])
        self.st[agent] = st
        return out

    def tick(self, now: float) -> int:
        for a in sorted(self.st):                         # gradual reservation, ready by the deadline
            s = self.st[a]
            if s["off"] and not s["up"] and not s["finished"] and not s["resv"] and self.cycles > 0 \
                    and now >= s["resv_start"]:
                self.pool.reserve_begin(s["h"], self.cycles)
                s["resv"] = True
        self.pool.reserve_tick()
        issued = 0
        for a in sorted(self.st):                         # predictive uploads that are due
            s = self.st[a]
            if s["off"] and not s["up"] and not s["finished"] and now >= s["upload_start"]:
                try:
                    self.pool.upload(s["h"])
                except OracleError as e:
                    if e.status != E_NOBLOCKS:
                        raise
                    continue                              # "stalls": retried next tick
                s["up"] = True
                issued += 1
        return issued

    def call_finish(self, agent: int, now: float) -> int:
        s = self.st.get(agent)
        if s is None:
            raise OracleError(E_INVAL, "call_finish for a request not in a call")
        if not s["finished"]:
            if now - s["start"] > 0:                      # EWMA feedback
                key = (s["cls"], s["label"])
                t_hist, n_obs = self.table.get(key, (None, 0))
                self.table[key] = record_fc_observation(t_hist, n_obs, now - s["start"], self.beta)
            s["finished"] = True
        if not s["off"]:
            del self.st[agent]                            # retained: resume at once
            return 0
        if not s["up"]:
            self.pool.upload(s["h"])                      # early finish: immediate upload; NOBLOCKS raises
            s["up"] = True
        del self.st[agent]
        return s["h"]

    # ------------------------------------------------------------------ queries
    def forecast(self, cls: int, label: int):
        return self.table.get((cls, label), (None, 0))

    def stalled(self) -> list:
        return sorted(self.st)

    def offloaded_handles(self) -> list:
        return [h for h, x in self.pool.handles.items() if x.state == OFFLOADED]
