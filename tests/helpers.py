"""Shared test helpers: run the CUDA engine through the package API on a JSON case (the
schema oracle/ and the reference shim use) and return the same result schema."""
import paper_2510_26475_b200 as rb


def model_of(j):
    return rb.TabularARModel(j["vocab"], j["order"], j["logits"], j.get("temperature", 1.0), j.get("version", 0))


def requests_of(reqs):
    return [rb.RequestState(r.get("id", 0), list(r["prompt"]), r.get("eos_bias", 0.0), r["max_len"],
                            rb.DecodeRng.from_seed(r["seed"], r["stream"])) for r in reqs]


def cfg_of(c):
    return rb.SDConfig(c.get("s", 1), c.get("t", 1), c.get("n", 1), c.get("enabled", False))


def table_of(t):
    return rb.ProfileTable.from_json(t)


def run_engine(case, verify_mode="sample", record=True):
    target = model_of(case["target"])
    drafter = model_of(case["drafter"]) if case.get("drafter") else None
    table = table_of(case["table"]) if case.get("table") else None
    run = rb.run_generation(requests_of(case["requests"]), target, (lambda: drafter) if drafter else None, table,
                            rb.TimingModel(), cfg_of(case.get("forced", {})), verify_mode=verify_mode,
                            record_full_logprobs=record)
    out = {"cycles": run.cycles, "total_time": run.total_time, "active_trace": run.active_trace,
           "switches": [{"cycle": s.cycle, "active_batch": s.active_batch,
                         "from": {"s": s.from_.rounds, "t": s.from_.branching, "n": s.from_.draft_len,
                                  "enabled": s.from_.enabled},
                         "to": {"s": s.to.rounds, "t": s.to.branching, "n": s.to.draft_len, "enabled": s.to.enabled}}
                        for s in run.switches],
           "ledger": [list(e) for e in run.ledger], "prefill_events": run.prefill_events,
           "accept_lens": run.accept_lens, "responses": [s.response for s in run.samples],
           "steps": [[[st.logp, st.drafted, st.logq] for st in s.steps] for s in run.samples]}
    if record:
        out["target_logprobs"] = [[st.target_logprobs for st in s.steps] for s in run.samples]
    return out, run
