// Event timeline of the drop-in library (reference
// proj/include/spgsim/engine.hpp:11-46): the same Operand / EventType /
// TimelineEvent / EventTimeline types and the same JSONL serialisation
// (engine.cpp:25-41), so callers of dr.timeline.to_jsonl() keep working.
//
// What differs is where the events come from: the reference's run_simulation
// plays a modeled alpha-beta clock; here every event is recorded by the device
// run (spg_trident_spgemm_ex / spg_summa_spgemm_ex) — the pulls that actually
// happened, with CUDA-event times in seconds from the rank's start. The DES
// itself (SimPlan, run_simulation) is the reference's modeled clock and is not
// part of the device path.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "spgsim/netmodel.hpp"

namespace spgsim {

enum class Operand { A, B };

const char* operand_name(Operand o);

enum class EventType {
    enqueue_request,
    serve_request,
    transfer_complete,
    allgather_complete,
    compute_complete,
};

const char* event_name(EventType t);

struct TimelineEvent {
    EventType type;
    int src = -1;  // sender / owner rank; node id for allgather events
    int dst = -1;  // receiver rank; -1 for allgather events
    int round = 0;
    Operand operand = Operand::A;
    LinkClass link = LinkClass::SELF;
    double t_start = 0.0;  // measured seconds from the rank's start
    double t_end = 0.0;
    index_t nnz = 0;
    std::int64_t bytes = 0;

    bool operator==(const TimelineEvent&) const = default;
};

struct EventTimeline {
    std::vector<TimelineEvent> events;

    // One JSON object per line, keys in the reference's order: type, actors,
    // round, t_start, t_end, bytes, operand, link, nnz.
    std::string to_jsonl() const;
};

}  // namespace spgsim
